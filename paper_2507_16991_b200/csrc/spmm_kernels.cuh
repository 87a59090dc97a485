// spmm.cu — CSR SpMM aggregation (sum / mean / max / min, optional edge
// scale or fused GCN norm, optional argmax) for sm_100a.
//
// Replaces, bit-exactly for f32/f64:
//   spmm / detail::spmm_forward     message_passing.hpp:47-85, 92-169
//   max path (fused, no E x F temp) message_passing.hpp:508-514 ->
//                                   dst_grouped_order 190-214, gather_rows
//                                   tensor.hpp:499-530, aggregate 197-215
//   GCN norm fused into the gather  message_passing.hpp:437-463, 490-495
//
// Exactness: every output element is accumulated by ONE thread, sequentially
// in compressed (CSC) order, with __fadd_rn/__fmul_rn (no FMA contraction) —
// the reference's `o[j] += w * xi[j]` loop order. Max/min: the first element
// initialises, then strict compare; ties keep the earlier edge.
//
// Scheduling (pure performance, never changes results):
//   * light rows (deg <= heavy_threshold): a group of LPR lanes owns one
//     nnz-balanced window of consecutive rows; lanes own VB-byte column
//     slices, U edges' gathers are in flight per batch (coalesced 128-bit
//     loads of whole feature rows, L1 no-allocate);
//   * heavy rows (power-law hubs): one CTA per row, longest first, on a forked
//     stream so hubs start before the light sweep; the CTA streams the row's
//     feature rows into a cp.async shared-memory ring (R stages of `se` edges)
//     while the owning threads accumulate each column in order.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "vec.cuh"

namespace gm {

struct SpmmArgs {
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* perm;
  const void* x;
  void* out;
  int32_t* arg;
  const void* w;             // per-edge scale (accumulation type), compressed order
  const int32_t* gdeg_src;   // GCN effective degrees (NULL = no GCN)
  const int32_t* gdeg_dst;
  int gcn_self;              // append the (v, v) self-loop term last
  const void* bias;          // GCN layer epilogue: + bias[col] (accumulation type), then
  int relu;                  // optional relu, before the final narrowing
  int mean;
  int is_min;
  int64_t num_rows;
  int64_t f;                 // elements per row
  int64_t slot_base;         // first VB-byte slot of this column chunk
  int64_t slot_end;          // one past the last slot of this chunk
  int64_t l2_block_slots;    // > 0: process the columns in blocks of this many slots, one after
                             // another (hub and flat kernels of a block together), so the
                             // gathered column block of X stays L2-resident across its reuse
  const int32_t* win_row;
  int64_t num_windows;
  int64_t heavy_thr;
  const int32_t* heavy_rows;
  const int32_t* light_windows;  // (first_row, end_row) pairs, heavy-free
  int64_t num_light_windows;
  int flat_ok;                   // heavy rows (if any) are covered by the hub kernel
  const uint8_t* src_class;      // per-entry source hotness class (NULL: no L2 hint)
  int hot_class_limit;           // entries with class < limit gather with evict_last
  // Seeded (blocked) accumulation: every row starts from the current out (and
  // arg) contents instead of 0 / the first element; max/min ties then break
  // on the smaller COO id, which reproduces "first attaining edge" across
  // source blocks (multi-GPU exchange overlap, dist.py).
  int accum;
  const int32_t* mean_deg;       // MEAN denominators per row (NULL = row length)
  int stream_x;                  // X exceeds the L2 budget: gathers carry eviction policies
  // epilogue (gm_spmm_ex): fp32 carry of bf16 block sums, push to peer buffers
  float* carry;                  // non-NULL: bf16 sum/mean rows seed from / store to fp32 rows here
  int carry_out;                 // 1: this block finishes the rows (store rounded to out)
  int n_push;
  void* push_dst[GM_MAX_PUSH];
  int64_t push_row0;
  const uint32_t* push_mask;
};

// Row-slice store of the epilogue: fp32 carry (bf16 blocks that are not the
// last), else the narrowed vector to out plus one plain store per selected
// peer (NVLink P2P when the peer buffer is mapped from another GPU).
// EPI = false compiles to the plain store: the flat kernel instantiates the
// epilogue separately (launched only when the call asks for it) — inlined
// into every row flush of the hot instantiations it cost the C5 bf16 sweep
// 76 -> 87 ms, and as a non-inlined call 4.2 -> 4.9 ms on C4.
template <typename T, typename VecT, bool EPI = true>
__device__ __forceinline__ void epi_store(const SpmmArgs& p, T* out, uint64_t elem, int64_t row,
                                          const typename VecT::A* v) {
  constexpr int V = VecT::V;
#ifdef GM_NO_EPI  // A/B builds only: every path takes the plain store
  if constexpr (true) {
#else
  if constexpr (!EPI) {
#endif
    VecT::store_global(out + elem, v);
    return;
  }
  if constexpr (sizeof(T) == 2) {
    if (p.carry != nullptr && !p.carry_out) {
      float* c = p.carry + elem;
#pragma unroll
      for (int e = 0; e < V; ++e) c[e] = v[e];
      return;
    }
  }
  VecT::store_global(out + elem, v);
  if (p.n_push) {
    const typename VecT::R r = VecT::pack(v);
    const uint32_t m = p.push_mask ? p.push_mask[row] : 0xffffffffu;
    const uint64_t gelem = elem + static_cast<uint64_t>(p.push_row0) * static_cast<uint64_t>(p.f);
#pragma unroll
    for (int q = 0; q < GM_MAX_PUSH; ++q)  // static indices: the targets stay in the parameter bank
      if (q < p.n_push && ((m >> q) & 1u))
        *reinterpret_cast<typename VecT::R*>(static_cast<T*>(p.push_dst[q]) + gelem) = r;
  }
}
// Seed V accumulators of a bf16 row slice from the fp32 carry; false: no carry.
template <typename T, typename A, int V>
__device__ __forceinline__ bool carry_seed(const SpmmArgs& p, uint64_t elem, A* v) {
  if constexpr (sizeof(T) == 2) {
    if (p.carry != nullptr) {
      const float* c = p.carry + elem;
#pragma unroll
      for (int e = 0; e < V; ++e) v[e] = c[e];
      return true;
    }
  }
  return false;
}

// L2 eviction-priority policies (createpolicy; PTX ISA "Cache eviction priority hints").
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <typename R>
__device__ __forceinline__ R ldg_hint(const R* p, uint64_t pol);
template <>
__device__ __forceinline__ uint4 ldg_hint<uint4>(const uint4* p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_hint<uint2>(const uint2* p, uint64_t pol) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_hint<uint32_t>(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_hint<unsigned short>(const unsigned short* p, uint64_t pol) {
  unsigned short r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
  return r;
}

// hot ? (evict_last policy) : (evict-first streaming), as a predicated pair: one
// policy descriptor, no branch per gather.
template <typename R>
__device__ __forceinline__ R ldg_hot_cs(const R* p, bool hot, uint64_t ph);
template <>
__device__ __forceinline__ uint4 ldg_hot_cs<uint4>(const uint4* p, bool hot, uint64_t ph) {
  uint4 r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;\n\t"
      "@!q ld.global.cs.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_hot_cs<uint2>(const uint2* p, bool hot, uint64_t ph) {
  uint2 r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %4;\n\t"
      "@!q ld.global.cs.nc.v2.u32 {%0,%1}, [%2];\n\t}"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_hot_cs<uint32_t>(const uint32_t* p, bool hot, uint64_t ph) {
  uint32_t r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %3;\n\t"
      "@!q ld.global.cs.nc.u32 %0, [%1];\n\t}"
      : "=r"(r)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_hot_cs<unsigned short>(const unsigned short* p, bool hot, uint64_t ph) {
  unsigned short r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %3;\n\t"
      "@!q ld.global.cs.nc.u16 %0, [%1];\n\t}"
      : "=h"(r)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}

// hot ? normal-priority : evict-first (ld.global.cs), predicated pair with no
// cache-policy operand: nothing 64-bit stays live across the batch (the
// policy-register form spilled at the max path's 64-register cap).
template <typename R>
__device__ __forceinline__ R ldg_na_cs(const R* p, bool hot);
template <>
__device__ __forceinline__ uint4 ldg_na_cs<uint4>(const uint4* p, bool hot) {
  uint4 r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t"
      "@!q ld.global.cs.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(hot)));
  return r;
}

// Both policies as predicated loads (no branch per gather): hot ? evict_last : evict_first.
template <typename R>
__device__ __forceinline__ R ldg_hint2(const R* p, bool hot, uint64_t ph, uint64_t pc);
template <>
__device__ __forceinline__ uint4 ldg_hint2<uint4>(const uint4* p, bool hot, uint64_t ph, uint64_t pc) {
  uint4 r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %6;\n\t"
      "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %7;\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_hint2<uint2>(const uint2* p, bool hot, uint64_t ph, uint64_t pc) {
  uint2 r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %4;\n\t"
      "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %5;\n\t}"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_hint2<uint32_t>(const uint32_t* p, bool hot, uint64_t ph, uint64_t pc) {
  uint32_t r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %3;\n\t"
      "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %4;\n\t}"
      : "=r"(r)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_hint2<unsigned short>(const unsigned short* p, bool hot, uint64_t ph,
                                                                    uint64_t pc) {
  unsigned short r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %3;\n\t"
      "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %4;\n\t}"
      : "=h"(r)
      : "l"(p), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}

// ldg_hot_cs with the lane's column validity folded into the predicates.
template <typename R>
__device__ __forceinline__ R ldg_hot_cs_v(const R* p, bool valid, bool hot, uint64_t ph);
template <>
__device__ __forceinline__ uint4 ldg_hot_cs_v<uint4>(const uint4* p, bool valid, bool hot, uint64_t ph) {
  uint4 r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %5, 0;\n\tsetp.ne.b32 h, %6, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %7;\n\t"
      "@b ld.global.cs.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_hot_cs_v<uint2>(const uint2* p, bool valid, bool hot, uint64_t ph) {
  uint2 r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %3, 0;\n\tsetp.ne.b32 h, %4, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %5;\n\t"
      "@b ld.global.cs.nc.v2.u32 {%0,%1}, [%2];\n\t}"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_hot_cs_v<uint32_t>(const uint32_t* p, bool valid, bool hot, uint64_t ph) {
  uint32_t r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %2, 0;\n\tsetp.ne.b32 h, %3, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %4;\n\t"
      "@b ld.global.cs.nc.u32 %0, [%1];\n\t}"
      : "=r"(r)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_hot_cs_v<unsigned short>(const unsigned short* p, bool valid, bool hot,
                                                                       uint64_t ph) {
  unsigned short r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %2, 0;\n\tsetp.ne.b32 h, %3, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %4;\n\t"
      "@b ld.global.cs.nc.u16 %0, [%1];\n\t}"
      : "=h"(r)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph));
  return r;
}

// ldg_hint2 with the lane's column-validity folded into the predicates: no
// branch at all per gather (invalid lanes issue nothing, their register is
// never read).
template <typename R>
__device__ __forceinline__ R ldg_hint2v(const R* p, bool valid, bool hot, uint64_t ph, uint64_t pc);
template <>
__device__ __forceinline__ uint4 ldg_hint2v<uint4>(const uint4* p, bool valid, bool hot, uint64_t ph, uint64_t pc) {
  uint4 r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %5, 0;\n\tsetp.ne.b32 h, %6, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %7;\n\t"
      "@b ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %8;\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_hint2v<uint2>(const uint2* p, bool valid, bool hot, uint64_t ph, uint64_t pc) {
  uint2 r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %3, 0;\n\tsetp.ne.b32 h, %4, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %5;\n\t"
      "@b ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %6;\n\t}"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_hint2v<uint32_t>(const uint32_t* p, bool valid, bool hot, uint64_t ph,
                                                         uint64_t pc) {
  uint32_t r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %2, 0;\n\tsetp.ne.b32 h, %3, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %4;\n\t"
      "@b ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %5;\n\t}"
      : "=r"(r)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_hint2v<unsigned short>(const unsigned short* p, bool valid, bool hot,
                                                                     uint64_t ph, uint64_t pc) {
  unsigned short r;
  asm("{\n\t.reg .pred v, h, a, b;\n\tsetp.ne.b32 v, %2, 0;\n\tsetp.ne.b32 h, %3, 0;\n\t"
      "and.pred a, v, h;\n\tand.pred b, v, !h;\n\t"
      "@a ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %4;\n\t"
      "@b ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %5;\n\t}"
      : "=h"(r)
      : "l"(p), "r"(static_cast<int>(valid)), "r"(static_cast<int>(hot)), "l"(ph), "l"(pc));
  return r;
}

template <typename A>
__device__ __forceinline__ A gcn_scale(int32_t ds, int32_t dd) {
  // message_passing.hpp:449-451: S(1) / std::sqrt(S(din[s]) * S(din[d]))
  return div_rn(A(1), sqrt_rn(mul_rn(static_cast<A>(ds), static_cast<A>(dd))));
}

// GCN layer epilogue on n accumulated values of columns [c0, c0+n):
// add(agg, bias) (message_passing.hpp:578), then relu (tensor.hpp:395).
template <typename A>
__device__ __forceinline__ void layer_epilogue(A* v, int n, const SpmmArgs& p, int64_t c0) {
  const A* __restrict__ b = static_cast<const A*>(p.bias);
  for (int e = 0; e < n; ++e) {
    A t = b ? add_rn(v[e], b[c0 + e]) : v[e];
    if (p.relu) t = t > A(0) ? t : A(0);
    v[e] = t;
  }
}

// Argmax ids of one V-element vector: int4/int2 stores (arg_out is 16-byte
// aligned and V divides F, so every vector's ids are 4V-byte aligned).
template <int V>
__device__ __forceinline__ void store_arg(int32_t* p, const int32_t* a) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int i = 0; i < V / 4; ++i)  // streaming stores: ids are written once, keep L2 for hot rows
      __stcs(reinterpret_cast<int4*>(p) + i, make_int4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]));
  } else if constexpr (V == 2) {
    __stcs(reinterpret_cast<int2*>(p), make_int2(a[0], a[1]));
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) p[e] = a[e];
  }
}

// Per-thread accumulator for NV vectors of V elements.
template <typename A, int NV, int V, bool MAXMIN>
struct Acc {
  A v[NV][V];
  int32_t a[NV][V];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        v[j][e] = A(0);
        if (MAXMIN) a[j][e] = -1;
      }
  }
  // Seed vector j from a previous block's result (p.accum). Returns true when
  // the row already has a first element (max/min: arg != -1).
  template <typename T, typename VecT>
  __device__ __forceinline__ bool seed(int j, const T* orow, const int32_t* arow) {
    typename VecT::R r = *reinterpret_cast<const typename VecT::R*>(orow);
    VecT::unpack(r, v[j]);
    bool have = true;
    if (MAXMIN) {
#pragma unroll
      for (int e = 0; e < V; ++e) a[j][e] = arow[e];
      have = a[j][0] != -1;
    }
    return have;
  }
  // One edge's contribution to vector j. `first`: first edge of the row.
  // lex: ties go to the smaller COO id (seeded blocks; inside one block ids
  // ascend, so strict compare alone already keeps the earliest).
  __device__ __forceinline__ void add(int j, const A* vals, bool scaled, A sc, bool first,
                                      int is_min, int32_t pm, bool lex = false) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const A val = scaled ? mul_rn(vals[e], sc) : vals[e];
      if (!MAXMIN) {
        v[j][e] = add_rn(v[j][e], val);
      } else {
        const bool better = first || (is_min ? (val < v[j][e]) : (val > v[j][e])) ||
                            (lex && val == v[j][e] && static_cast<uint32_t>(pm) < static_cast<uint32_t>(a[j][e]));
        v[j][e] = better ? val : v[j][e];
        a[j][e] = better ? pm : a[j][e];
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Light path: LPR lanes per window, NV vectors of VB bytes per lane.
// ---------------------------------------------------------------------------
template <typename T, int VB, int NV, int LPR, int U, bool MAXMIN>
__global__ void __launch_bounds__(256) spmm_light_kernel(const SpmmArgs p) {
  using VecT = Vec<T, VB>;
  using A = typename VecT::A;
  constexpr int V = VecT::V;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t window = gid / LPR;
  const int sub = static_cast<int>(gid % LPR);
  if (window >= p.num_windows) return;

  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ out = static_cast<T*>(p.out);
  const A* __restrict__ w = static_cast<const A*>(p.w);
  const bool gcn = p.gdeg_src != nullptr;
  const bool scaled = gcn || w != nullptr;
  const bool want_arg = MAXMIN && p.arg != nullptr;

  int64_t slot[NV];
  bool valid[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    slot[j] = p.slot_base + sub + j * LPR;
    valid[j] = slot[j] < p.slot_end;
  }

  const int r0 = p.win_row[window];
  const int r1 = p.win_row[window + 1];
  for (int r = r0; r < r1; ++r) {
    const int64_t kb = p.rowptr[r];
    const int64_t ke = p.rowptr[r + 1];
    if (ke - kb > p.heavy_thr) continue;  // the heavy kernel owns this row
    Acc<A, NV, V, MAXMIN> acc;
    acc.init();
    bool seeded = false;
    if (p.accum) {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (valid[j]) {
          const uint64_t el = static_cast<uint64_t>(r) * p.f + slot[j] * V;
          if (!MAXMIN && carry_seed<T, A, V>(p, el, acc.v[j])) seeded = true;
          else
            seeded = acc.template seed<T, VecT>(j, out + el, MAXMIN ? p.arg + el : nullptr);
        }
    }
    const bool lex = p.accum != 0;
    const int32_t dd = gcn ? p.gdeg_dst[r] : 0;

    for (int64_t k = kb; k < ke; k += U) {
      int32_t c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = (k + u < ke) ? p.col[k + u] : 0;
      VecT buf[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < ke) {
          const T* xr = x + static_cast<int64_t>(c[u]) * p.f;
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (valid[j]) buf[u][j].load_global(xr + slot[j] * V);
        }
      A sc[U];
      int32_t pm[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sc[u] = A(1);
        pm[u] = -1;
        if (k + u < ke) {
          if (w) sc[u] = w[k + u];
          else if (gcn) sc[u] = gcn_scale<A>(p.gdeg_src[c[u]], dd);
          if (want_arg) pm[u] = p.perm[k + u];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < ke) {
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (valid[j]) acc.add(j, buf[u][j].v, scaled, sc[u], !seeded && k + u == kb, p.is_min, pm[u], lex);
        }
    }
    int64_t cnt = ke - kb;
    if (gcn && p.gcn_self) {
      // with_self_loops appends (r, r) after every original edge
      // (edge_index.cpp:226-229), so it is the last entry of CSC row r.
      const A sc = gcn_scale<A>(p.gdeg_src[r], dd);
      const T* xr = x + static_cast<int64_t>(r) * p.f;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (valid[j]) {
          VecT b;
          b.load_global(xr + slot[j] * V);
          acc.add(j, b.v, true, sc, !seeded && cnt == 0, p.is_min, -1);
        }
      cnt += 1;
    }
    if (p.mean_deg) cnt = p.mean_deg[r];
    if (!MAXMIN && p.mean && cnt > 0) {
      const A inv = div_rn(A(1), static_cast<A>(cnt));  // message_passing.hpp:81
#pragma unroll
      for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int e = 0; e < V; ++e) acc.v[j][e] = mul_rn(acc.v[j][e], inv);
    }
    if constexpr (!MAXMIN) {
      if (p.bias || p.relu) {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (valid[j]) layer_epilogue<A>(acc.v[j], V, p, slot[j] * V);
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (valid[j]) {
        epi_store<T, VecT, true>(p, out, static_cast<uint64_t>(r) * p.f + slot[j] * V, r, acc.v[j]);
        if (want_arg) {
          int32_t* arow = p.arg + static_cast<int64_t>(r) * p.f + slot[j] * V;
          store_arg<V>(arow, acc.a[j]);
        }
      }
  }
  if (p.n_push) __threadfence_system();
}


// ---------------------------------------------------------------------------
// Flat light path (the hot one): one warp streams a heavy-free window of
// consecutive rows as ONE contiguous edge range, U edges per batch regardless
// of row boundaries (no partial batches at row ends). The next batch's col
// (and weight / perm) entries are prefetched one batch ahead, one per lane,
// and broadcast by shuffle; row ends are cached 32 at a time across lanes.
// Accumulation order per output element is unchanged: ascending CSC position.
// ---------------------------------------------------------------------------
// MODE: 0 sum, 1 mean, 2 max, 3 min. LM (load mode) for an X far larger than
// L2: gathers of entries whose source class is below p.hot_class_limit (when
// the plan's classes are in use) carry an evict_last policy, all others
// evict_first, so hub rows stay L2-resident while the rest streams. LM = 2 is
// the fresh (non-seeded) path with the class array read; max/min there
// stream the cold arm with ld.global.cs. 0 = default loads (X fits L2).
// Measured on C4 (sum): default 6.2 ms, all-cs 6.2, all-evict_first 4.8,
// hot evict_last + cold evict_first 4.25.
#ifndef GM_FLAT_GATHER_V
#define GM_FLAT_GATHER_V 3
#endif
// gather form of the 16-byte one-vector flat path (same-box A/B builds,
// tools/build_variant.sh): 0 validity-predicated policy pair; 1 max/min with
// clamped lanes (no predicate) + normal / evict-first; 2 the same for sum/mean
// (C4 sum 4.27 -> 4.89 ms: the hot rows need evict_last); 3 (default) max/min
// with clamped lanes + evict_last / evict-first. With 6 edges per batch
// (GM_FLAT_MAX_U) C4 max + argmax went 5.13 -> 4.72 ms: 8 edges spilled the
// batch at the 64-register cap, 4-5 left too few gathers in flight.
constexpr int kFlatGather = GM_FLAT_GATHER_V;
#ifndef GM_FLAT_MAX_U
#define GM_FLAT_MAX_U 6  // edges per batch of the 16-byte one-vector max/min path
#endif
template <typename T, int VB, int NV, int U, int MODE, bool SCALED, bool ACC, int LM, bool EPI = false>
__global__ void __launch_bounds__(256, (sizeof(T) == 8 || (SCALED && (MODE >= 2 || NV > 1 || VB <= 8))) ? 3 : 4) spmm_flat_kernel(const SpmmArgs p) {
  constexpr bool MAXMIN = MODE >= 2;
  constexpr bool IS_MIN = MODE == 3;
  constexpr bool MEAN = MODE == 1;
  using VecT = Vec<T, VB>;
  using A = typename VecT::A;
  using R = typename VecT::R;
  constexpr int V = VecT::V;
  constexpr unsigned FULL = 0xffffffffu;
  // clamped one-vector gathers: every lane consumes a real row slice, only
  // the valid ones store
  constexpr bool kClamped = kFlatGather >= 1 && VB == 16 && NV == 1 && LM >= 1 && (MAXMIN || kFlatGather == 2);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (warp >= p.num_light_windows) return;

  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ out = static_cast<T*>(p.out);
  const int32_t* __restrict__ col = p.col;
  const bool want_arg = MAXMIN && p.arg != nullptr;
  const uint32_t fu = static_cast<uint32_t>(p.f);  // row stride (elements)
  const int nsl = static_cast<int>(p.slot_end - p.slot_base);

  uint32_t soff[NV];  // element offset of this lane's vector j inside a row
  bool valid[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    valid[j] = lane + j * 32 < nsl;
    soff[j] = static_cast<uint32_t>((p.slot_base + lane + j * 32) * V);
  }
  // gather address = this lane's slice base + source * row bytes: one IMAD.WIDE
  const unsigned char* xlane = reinterpret_cast<const unsigned char*>(x) + static_cast<size_t>(soff[0]) * sizeof(T);
  // lanes past the row's last slot gather that slot again (same sectors as
  // the last valid lane: no extra traffic) and never store, so the one-vector
  // gathers need no validity predicate
  const unsigned char* xlane_c =
      reinterpret_cast<const unsigned char*>(x) +
      static_cast<size_t>((p.slot_base + min(lane, max(nsl - 1, 0))) * V) * sizeof(T);
  const uint32_t rowb = fu * static_cast<uint32_t>(sizeof(T));

  // Positions fit int32: gm_build_compressed / plan_build require nnz < 2^31.
  const int ra = p.light_windows[2 * warp];
  const int rb = p.light_windows[2 * warp + 1];
  const int32_t kbeg = static_cast<int32_t>(p.rowptr[ra]);
  const int32_t kend = static_cast<int32_t>(p.rowptr[rb]);

  // lane l caches the end of row cbase + l
  int cbase = ra;
  int32_t rend_l = (cbase + lane < rb) ? static_cast<int32_t>(p.rowptr[cbase + 1 + lane]) : kend;
  int row = ra;
  int32_t row_start = kbeg;
  int32_t row_end = __shfl_sync(FULL, rend_l, 0);

  Acc<A, NV, V, MAXMIN> acc;
  bool first = true;
  constexpr bool lex = MAXMIN && ACC;
  auto begin_row = [&]() {
    acc.init();
    first = true;
    if constexpr (ACC) {
      const uint64_t ob = static_cast<uint64_t>(static_cast<uint32_t>(row)) * fu;
      bool have = false;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (valid[j]) {
          if (!MAXMIN && carry_seed<T, A, V>(p, ob + soff[j], acc.v[j])) have = true;
          else have = acc.template seed<T, VecT>(j, out + ob + soff[j], MAXMIN ? p.arg + ob + soff[j] : nullptr);
        }
      first = !have;
    }
  };
  begin_row();

  auto flush = [&]() {
    if (MEAN) {
      const int32_t cnt = (ACC && p.mean_deg) ? p.mean_deg[row] : row_end - row_start;
      if (cnt > 0) {
        const A inv = div_rn(A(1), static_cast<A>(cnt));  // message_passing.hpp:81
#pragma unroll
        for (int j = 0; j < NV; ++j)
#pragma unroll
          for (int e = 0; e < V; ++e) acc.v[j][e] = mul_rn(acc.v[j][e], inv);
      }
    }
    const uint64_t obase = static_cast<uint64_t>(static_cast<uint32_t>(row)) * fu;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (valid[j]) {
        epi_store<T, VecT, EPI>(p, out, obase + soff[j], row, acc.v[j]);
        if (want_arg) {
          int32_t* arow = p.arg + obase + soff[j];
          store_arg<V>(arow, acc.a[j]);
        }
      }
    ++row;
    row_start = row_end;
    if (row < rb) {
      if (row - cbase >= 32) {
        cbase = row;
        rend_l = (cbase + lane < rb) ? static_cast<int32_t>(p.rowptr[cbase + 1 + lane]) : kend;
      }
      row_end = __shfl_sync(FULL, rend_l, row - cbase);
      begin_row();
    }
  };

  constexpr bool HINT = LM >= 1;  // per-entry hot flag (false when the plan's classes are off)
  const uint64_t pol_hot = HINT ? policy_evict_last() : 0;
  const uint64_t pol_cold = HINT ? policy_evict_first() : 0;
  int32_t c_next = 0, p_next = -1;
  bool h_next = false;
  A w_next = A(1);
  // entries past the window end repeat its last edge: that row is re-read
  // (an L2 hit) but never accumulated, so the loads need no bounds checks
  auto fetch = [&](int32_t kb) {
    if (lane < U) {
      const int32_t k = min(kb + lane, kend - 1);
      c_next = col[k];
      if (HINT && p.src_class) h_next = p.src_class[k] < p.hot_class_limit;
      if (SCALED) w_next = static_cast<const A*>(p.w)[k];
      if (MAXMIN) p_next = want_arg ? p.perm[k] : -1;
    }
  };
  if (kend > kbeg) fetch(kbeg);

  for (int32_t k0 = kbeg; k0 < kend; k0 += U) {
    const int32_t c_cur = c_next;
    const int32_t p_cur = p_next;
    const uint32_t hmask = HINT ? __ballot_sync(FULL, h_next) : 0u;
    const A w_cur = w_next;
    if (k0 + U < kend) fetch(k0 + U);
    const int nb = min(U, kend - k0);  // edges in this batch
    R buf[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T* xr = x + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(FULL, c_cur, u))) * fu;
      const bool hot = (hmask >> u) & 1u;
      if constexpr (kFlatGather >= 1 && VB == 16 && NV == 1 && LM >= 1 && (MAXMIN || kFlatGather == 2)) {
        // one 16-byte vector per lane: clamped lane base (no predicate), hot
        // rows at normal L2 priority, the rest evict-first, no policy register
        const unsigned char* xs = xlane_c + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(FULL, c_cur, u))) * rowb;
        if constexpr (kFlatGather == 3) buf[u][0] = ldg_hot_cs<R>(reinterpret_cast<const R*>(xs), hot, pol_hot);
        else buf[u][0] = ldg_na_cs<R>(reinterpret_cast<const R*>(xs), hot);
      } else if constexpr (LM >= 1 && !MAXMIN && VB <= 8) {
        // predicated evict_last / evict_first pair with the column validity
        // folded in and a precomputed lane base: no branch, one IMAD.WIDE per
        // gather (8-byte vectors: C5 87 -> 79 ms, C2 55 -> 51 ms in A/B runs;
        // the 16-byte C4 path measured slower this way and keeps the form below)
        const unsigned char* xs = xlane + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(FULL, c_cur, u))) * rowb;
#pragma unroll
        for (int j = 0; j < NV; ++j)
          buf[u][j] = ldg_hint2v<R>(reinterpret_cast<const R*>(xs + j * 32 * VB), valid[j], hot, pol_hot, pol_cold);
      } else if constexpr (LM >= 1 && !MAXMIN) {
        // predicated evict_last / evict_first pair: no branch per gather
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (valid[j]) buf[u][j] = ldg_hint2<R>(reinterpret_cast<const R*>(xr + soff[j]), hot, pol_hot, pol_cold);
      } else if constexpr (LM == 2 && VB <= 8) {
        // max/min, 8-byte vectors: one policy live (the cold arm streams with
        // ld.global.cs), lane base + folded validity as above (the 16-byte C4
        // max path measured 5.2 -> 6.1 ms this way and keeps the form below)
        const unsigned char* xs = xlane + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(FULL, c_cur, u))) * rowb;
#pragma unroll
        for (int j = 0; j < NV; ++j)
          buf[u][j] = ldg_hot_cs_v<R>(reinterpret_cast<const R*>(xs + j * 32 * VB), valid[j], hot, pol_hot);
      } else if constexpr (LM == 2) {
        // max/min: both 64-bit policies live would spill at 64 registers; the
        // cold arm streams with ld.global.cs instead
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (valid[j]) buf[u][j] = ldg_hot_cs<R>(reinterpret_cast<const R*>(xr + soff[j]), hot, pol_hot);
      } else if constexpr (LM == 1) {
        if (hot) {
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (valid[j]) buf[u][j] = ldg_hint<R>(reinterpret_cast<const R*>(xr + soff[j]), pol_hot);
        } else {
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (valid[j]) buf[u][j] = ldg_hint<R>(reinterpret_cast<const R*>(xr + soff[j]), pol_cold);
        }
      } else if (u < nb) {  // (the branch also keeps ptxas from hoisting all U addresses at once)
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (valid[j])
            buf[u][j] = VecT::load_raw(xr + soff[j]);
      }
    }
    if (nb == U && k0 + U <= row_end) {
      // fast path: the whole batch belongs to the current row
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const A sc = SCALED ? __shfl_sync(FULL, w_cur, u) : A(1);
        const int32_t pm = MAXMIN ? __shfl_sync(FULL, p_cur, u) : -1;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (kClamped || valid[j]) {
            A vals[V];
            VecT::unpack(buf[u][j], vals);
            acc.add(j, vals, SCALED, sc, first && u == 0, IS_MIN, pm, lex);
          }
        }
      }
      first = false;
    } else {
      if constexpr (U <= 8) {
      // rows end inside the batch: consume it in passes — each pass adds the
      // current row's edges [u0, m) (one predicated copy of the add block),
      // then the row is flushed; empty rows take passes with no adds.
      // (A/B on one B200: C4 sum/max 1-2% faster; the 16-edge narrow-row
      // batches of C5 keep the per-edge form, 2.4% faster there.)
      int u0 = 0;
      while (true) {
        const int m = min(nb, row_end - k0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u >= u0 && u < m) {
            const A sc = SCALED ? __shfl_sync(FULL, w_cur, u) : A(1);
            const int32_t pm = MAXMIN ? __shfl_sync(FULL, p_cur, u) : -1;
#pragma unroll
            for (int j = 0; j < NV; ++j)
              if (kClamped || valid[j]) {
                A vals[V];
                VecT::unpack(buf[u][j], vals);
                acc.add(j, vals, SCALED, sc, first && u == u0, IS_MIN, pm, lex);
              }
          }
        }
        if (m > u0) first = false;
        if (m >= nb) break;
        flush();
        u0 = m;
      }
      } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const A sc = SCALED ? __shfl_sync(FULL, w_cur, u) : A(1);
        const int32_t pm = MAXMIN ? __shfl_sync(FULL, p_cur, u) : -1;
        if (u < nb) {
          while (k0 + u >= row_end) flush();
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (kClamped || valid[j]) {
              A vals[V];
              VecT::unpack(buf[u][j], vals);
              acc.add(j, vals, SCALED, sc, first, IS_MIN, pm, lex);
            }
          first = false;
        }
      }
      }
    }
  }
  while (row < rb) flush();
  // pushed rows must be visible to the peers before the caller's collective
  // releases their next read
  if (EPI && p.n_push) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Heavy path: one CTA per hub row, cp.async ring of R stages x se edges.
// ---------------------------------------------------------------------------
constexpr int kHeavyThreads = 256;
constexpr int64_t kWideRowBytes = 1024;
// Max vectors per lane in the flat kernel (GM_FLAT_MAX_NV, default 4: wide
// rows take more column passes with more edges in flight per batch).
inline int flat_max_nv() {
  static const int nv = [] { const char* e = getenv("GM_FLAT_MAX_NV"); return e ? atoi(e) : 4; }();
  return nv;
}
// threads per flat CTA (GM_FLAT_THREADS, multiple of 32, <= 256): 4-warp CTAs
// (8 per SM at 64 registers) lose only 4 warps per SM to a concurrent hub CTA
// and finish the sweep with a finer tail. C4 sum, same box: 256 / 224 / 192 /
// 160 / 128 / 96 threads 4.31 / 4.32 / 4.30 / 4.28 / 4.24 / 4.24 ms; the flat
// kernel alone 4.15 -> 4.09 ms at 128
inline int flat_threads() {
  static const int t = [] {
    const char* e = getenv("GM_FLAT_THREADS");
    const int v = e ? atoi(e) : 128;
    return (v >= 32 && v <= 256 && v % 32 == 0) ? v : 128;
  }();
  return t;
}
constexpr int kRing = 4;

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename A>
__host__ __device__ inline size_t heavy_smem_bytes(int se, int rowb) {
  size_t b = static_cast<size_t>(kRing) * se * rowb;          // data ring
  b += static_cast<size_t>(kRing + 1) * se * sizeof(int32_t);  // col ring
  b += static_cast<size_t>(kRing + 1) * se * sizeof(int32_t);  // perm ring
  b = (b + 15) / 16 * 16;
  b += static_cast<size_t>(kRing + 1) * se * sizeof(A);        // scale ring
  return b;
}

template <typename T, int VB, int MH, bool MAXMIN>
__global__ void __launch_bounds__(kHeavyThreads) spmm_heavy_kernel(const SpmmArgs p, int se) {
  using VecT = Vec<T, VB>;
  using A = typename VecT::A;
  constexpr int V = VecT::V;
  extern __shared__ __align__(16) unsigned char smem[];
  const int nslots = static_cast<int>(p.slot_end - p.slot_base);
  const int rowb = nslots * VB;
  unsigned char* data = smem;
  int32_t* mcol = reinterpret_cast<int32_t*>(smem + static_cast<size_t>(kRing) * se * rowb);
  int32_t* mperm = mcol + (kRing + 1) * se;
  size_t off = static_cast<size_t>(kRing) * se * rowb + 2ull * (kRing + 1) * se * sizeof(int32_t);
  off = (off + 15) / 16 * 16;
  A* mscale = reinterpret_cast<A*>(smem + off);

  const T* __restrict__ x = static_cast<const T*>(p.x);
  const A* __restrict__ w = static_cast<const A*>(p.w);
  const bool gcn = p.gdeg_src != nullptr;
  const bool scaled = gcn || w != nullptr;
  const bool want_arg = MAXMIN && p.arg != nullptr;
  const int t = threadIdx.x;

  // hub list, or every row (wide-row mode: heavy_rows == NULL)
  const int r = p.heavy_rows ? p.heavy_rows[blockIdx.x] : static_cast<int>(blockIdx.x);
  const int64_t kb = p.rowptr[r];
  const int64_t ke = p.rowptr[r + 1];
  const int64_t deg = ke - kb;
  const int64_t total = deg + ((gcn && p.gcn_self) ? 1 : 0);
  const int nst = static_cast<int>((total + se - 1) / se);
  const int32_t dd = gcn ? p.gdeg_dst[r] : 0;
  const int gpr = rowb / VB;  // copy granules per feature row (VB bytes each)

  // Register-staged metadata of one stage (threads t < se own edge t).
  int32_t rc = -1, rp = -1;
  A rw = A(1);
  auto load_meta = [&](int q) {
    const int64_t e = static_cast<int64_t>(q) * se + t;
    rc = -1;
    if (t < se && e < total) {
      if (e < deg) {
        const int64_t k = kb + e;
        rc = p.col[k];
        rp = want_arg ? p.perm[k] : -1;
        rw = w ? w[k] : A(1);
      } else {  // the self-loop term
        rc = r;
        rp = -1;
        rw = A(1);
      }
    }
  };

  Acc<A, MH, V, MAXMIN> acc;
  acc.init();
  bool seeded = false;
  if (p.accum) {
    T* orow0 = static_cast<T*>(p.out) + static_cast<int64_t>(r) * p.f;
#pragma unroll
    for (int m = 0; m < MH; ++m) {
      const int s = t + m * kHeavyThreads;
      if (s < nslots) {
        const uint64_t el = static_cast<uint64_t>(r) * p.f + (p.slot_base + s) * V;
        if (!MAXMIN && carry_seed<T, A, V>(p, el, acc.v[m])) seeded = true;
        else
          seeded = acc.template seed<T, VecT>(m, orow0 + (p.slot_base + s) * V,
                                              MAXMIN ? p.arg + static_cast<int64_t>(r) * p.f + (p.slot_base + s) * V
                                                     : nullptr);
      }
    }
  }
  const bool lex = MAXMIN && p.accum != 0;
  A sc_next = A(1);

  load_meta(0);
  for (int i = -(kRing - 1); i < nst; ++i) {
    const int q = i + kRing - 1;  // stage whose copies are issued now
    if (q < nst && t < se) {
      const int ms = (q % (kRing + 1)) * se + t;
      mcol[ms] = rc;
      mperm[ms] = rp;
      if (!gcn) mscale[ms] = rw;
    }
    if (q + 1 < nst) load_meta(q + 1);
    __syncthreads();
    if (q < nst) {
      const int base_e = q * se;
      const int n_e = static_cast<int>(min(static_cast<int64_t>(se), total - base_e));
      const int32_t* cq = mcol + (q % (kRing + 1)) * se;
      unsigned char* dq = data + static_cast<size_t>(q % kRing) * se * rowb;
      for (int g = t; g < n_e * gpr; g += kHeavyThreads) {
        const int e = g / gpr;
        const int part = g - e * gpr;
        const T* src = x + static_cast<int64_t>(cq[e]) * p.f + (p.slot_base + part) * V;
        cp_async(dq + static_cast<size_t>(e) * rowb + part * VB, src, VB);
      }
    }
    cp_async_commit();
    if (gcn && i + 1 >= 0 && i + 1 < nst && t < se) {
      const int64_t e = static_cast<int64_t>(i + 1) * se + t;
      if (e < total) sc_next = gcn_scale<A>(p.gdeg_src[mcol[((i + 1) % (kRing + 1)) * se + t]], dd);
    }
    cp_async_wait<kRing - 1>();
    __syncthreads();
    if (i >= 0) {
      const int base_e = i * se;
      const int n_e = static_cast<int>(min(static_cast<int64_t>(se), total - base_e));
      const unsigned char* di = data + static_cast<size_t>(i % kRing) * se * rowb;
      const int mi = (i % (kRing + 1)) * se;
#pragma unroll
      for (int m = 0; m < MH; ++m) {
        const int s = t + m * kHeavyThreads;
        if (s < nslots) {
          for (int e = 0; e < n_e; ++e) {
            VecT v;
            v.load_shared(reinterpret_cast<const T*>(di + static_cast<size_t>(e) * rowb + s * VB));
            acc.add(m, v.v, scaled, mscale[mi + e], !seeded && base_e + e == 0, p.is_min, mperm[mi + e], lex);
          }
        }
      }
    }
    if (gcn && i + 1 >= 0 && i + 1 < nst && t < se) mscale[((i + 1) % (kRing + 1)) * se + t] = sc_next;
  }

  const int64_t cnt = p.mean_deg ? p.mean_deg[r] : total;
  if (!MAXMIN && p.mean && cnt > 0) {
    const A inv = div_rn(A(1), static_cast<A>(cnt));
#pragma unroll
    for (int m = 0; m < MH; ++m)
#pragma unroll
      for (int e = 0; e < V; ++e) acc.v[m][e] = mul_rn(acc.v[m][e], inv);
  }
  if (!MAXMIN && (p.bias || p.relu)) {
#pragma unroll
    for (int m = 0; m < MH; ++m) {
      const int s = t + m * kHeavyThreads;
      if (s < nslots) layer_epilogue<A>(acc.v[m], V, p, (p.slot_base + s) * V);
    }
  }
#pragma unroll
  for (int m = 0; m < MH; ++m) {
    const int s = t + m * kHeavyThreads;
    if (s < nslots) {
      epi_store<T, VecT, true>(p, static_cast<T*>(p.out),
                                  static_cast<uint64_t>(r) * p.f + (p.slot_base + s) * V, r, acc.v[m]);
      if (want_arg) {
        int32_t* arow = p.arg + static_cast<int64_t>(r) * p.f + (p.slot_base + s) * V;
        store_arg<V>(arow, acc.a[m]);
      }
    }
  }
  if (p.n_push) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Hub path v2: one CTA of two warps per (hub row, 128/256-byte column chunk).
// Column chunks of a hub row run on different SMs in parallel. Warp 1 (the
// consumer) owns one 4-byte (f32 / bf16x2) or 8-byte (f64) column slot per
// lane and accumulates it sequentially in compressed order, so results stay
// bit-exact. Warp 0 (the producer) streams the chunk's slices of the row's
// source rows into a kHubRing-deep ring of 32-edge stages with cp.async:
// per-edge metadata (col, perm, weight) kHubRing stages ahead of the slice
// copies, each stage published to the consumer by cp.async.mbarrier.arrive on
// its `full` barrier, slots handed back through `empty`.
// ---------------------------------------------------------------------------
constexpr int kHubStage = 32;
#ifndef GM_HUB_RING
#define GM_HUB_RING 16
#endif
constexpr int kHubRing = GM_HUB_RING;
constexpr int kHubMeta = 2 * kHubRing;

template <typename T, int W = 1>
struct HubLane {  // per-lane storage unit: 4 bytes (f32, bf16x2) or 8 bytes (f64, or f32 x2 with W = 2)
  static constexpr int LE = (sizeof(T) == 2 ? 2 : 1) * W;
  static constexpr int LB = LE * static_cast<int>(sizeof(T));
  static constexpr int CB = 32 * LB;  // chunk bytes
  using R = typename std::conditional<LB == 8, unsigned long long, uint32_t>::type;
};

template <typename T, int W = 1>
__host__ __device__ constexpr size_t hub_smem_bytes() {
  return static_cast<size_t>(kHubRing) * kHubStage * HubLane<T, W>::CB;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// arrives on bar once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

template <typename T, int G, int MODE, int W = 1>  // MODE: 0 sum/mean, 2 max, 3 min; W: lane width x
__global__ void __launch_bounds__(64) spmm_hub_kernel(const SpmmArgs p) {
  constexpr bool MAXMIN = MODE >= 2;
  constexpr bool IS_MIN = MODE == 3;
  using HL = HubLane<T, W>;
  using A = typename AccOf<T>::type;
  constexpr int LE = HL::LE;
  constexpr int LB = HL::LB;
  constexpr int CB = HL::CB;
  constexpr int GPR = CB / G;  // copy granules per full chunk row
  extern __shared__ __align__(16) unsigned char hub_data[];  // [kHubRing][kHubStage][CB]
  __shared__ int32_t mcol[kHubMeta][kHubStage];
  __shared__ int32_t mperm[kHubMeta][kHubStage];
  __shared__ int32_t mdeg[kHubMeta][kHubStage];
  __shared__ A mw[kHubMeta][kHubStage];
  __shared__ uint64_t full[kHubRing], empty[kHubRing];

  const int lane = threadIdx.x & 31;
  const bool producer = threadIdx.x < 32;
  const int64_t row_bytes = p.f * static_cast<int64_t>(sizeof(T));
  const int nchunks = static_cast<int>((row_bytes + CB - 1) / CB);
  const int hub = static_cast<int>(blockIdx.x / nchunks);
  const int r = p.heavy_rows[hub];
  const int64_t c_off = static_cast<int64_t>(blockIdx.x - static_cast<unsigned>(hub) * nchunks) * CB;
  const int vbytes = static_cast<int>(row_bytes - c_off < CB ? row_bytes - c_off : CB);
  const A* __restrict__ w = static_cast<const A*>(p.w);
  const bool gcn = p.gdeg_src != nullptr;
  const bool scaled = gcn || w != nullptr;
  const bool want_arg = MAXMIN && p.arg != nullptr;
  const int64_t kb = p.rowptr[r];
  const int64_t deg = p.rowptr[r + 1] - kb;
  const int64_t total = deg + ((gcn && p.gcn_self) ? 1 : 0);
  const int nst = static_cast<int>((total + kHubStage - 1) / kHubStage);
  auto stage_edges = [&](int q) {
    const int64_t left = total - static_cast<int64_t>(q) * kHubStage;
    return static_cast<int>(left < kHubStage ? left : kHubStage);
  };

  if (threadIdx.x < kHubRing) {
    mbar_init(&full[threadIdx.x], 32);  // every producer lane arrives (cp.async noinc)
    mbar_init(&empty[threadIdx.x], 1);  // one consumer lane arrives
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  if (producer) {
    const unsigned char* __restrict__ xb = static_cast<const unsigned char*>(p.x) + c_off;
    const int vgran = vbytes / G;
    // metadata of stage q -> meta slot q % kHubMeta (lane e = edge e)
    auto issue_meta = [&](int q) {
      if (q >= nst) return;
      const int ms = q % kHubMeta;
      const int64_t e = static_cast<int64_t>(q) * kHubStage + lane;
      if (e < deg) {
        const int64_t k = kb + e;
        cp_async(&mcol[ms][lane], p.col + k, 4);
        if (want_arg) cp_async(&mperm[ms][lane], p.perm + k, 4);
        if (w) cp_async(&mw[ms][lane], w + k, static_cast<int>(sizeof(A)));
      } else if (e < total) {  // the fused GCN self loop (r, r), last in the row
        mcol[ms][lane] = r;
        mperm[ms][lane] = -1;
      }
    };
    // one commit group per stage's metadata: meta(q) is group q, so after the
    // R + q commits preceding iteration q's wait, wait_group<R-1> lands it
#pragma unroll 1
    for (int q = 0; q < kHubRing; ++q) {
      issue_meta(q);
      cp_async_commit();
    }
#pragma unroll 1
    for (int q = 0; q < nst; ++q) {
      const int slot = q % kHubRing;
      if (q >= kHubRing) mbar_wait(&empty[slot], static_cast<uint32_t>(((q / kHubRing) - 1) & 1));
      cp_async_wait<kHubRing - 1>();  // meta(q) = group q landed
      __syncwarp();
      const int ms = q % kHubMeta;
      const int n_e = stage_edges(q);
      if (gcn && lane < n_e) cp_async(&mdeg[ms][lane], p.gdeg_src + mcol[ms][lane], 4);
      unsigned char* dq = hub_data + static_cast<size_t>(slot) * kHubStage * CB;
      for (int g = lane; g < n_e * GPR; g += 32) {
        const int e2 = g / GPR;
        const int part = g - e2 * GPR;
        if (part < vgran)
          cp_async(dq + e2 * CB + part * G, xb + static_cast<int64_t>(mcol[ms][e2]) * row_bytes + part * G, G);
      }
      mbar_arrive_cp_async(&full[slot]);  // fires when this lane's copies (and earlier meta) land
      issue_meta(q + kHubRing);           // slot of stage q - R: consumed (empty waited above)
      cp_async_commit();
    }
    cp_async_wait<0>();
    return;
  }

  // ---- consumer warp ----
  const int32_t dd = gcn ? p.gdeg_dst[r] : 0;
  A v[LE];
  int32_t a[LE];
  bool first = true;
  const int64_t e0 = c_off / static_cast<int64_t>(sizeof(T)) + static_cast<int64_t>(lane) * LE;
  const bool lane_valid = lane * LB < vbytes;
  T* orow = static_cast<T*>(p.out) + static_cast<int64_t>(r) * p.f;
#pragma unroll
  for (int i = 0; i < LE; ++i) {
    v[i] = A(0);
    a[i] = -1;
  }
  if (p.accum && lane_valid) {
    if (!MAXMIN && carry_seed<T, A, LE>(p, static_cast<uint64_t>(r) * p.f + e0, v)) {
      first = false;
    } else {
      T tmp[LE];
      memcpy(tmp, orow + e0, LB);
#pragma unroll
      for (int i = 0; i < LE; ++i) {
        v[i] = widen(tmp[i]);
        if (MAXMIN) a[i] = p.arg[static_cast<int64_t>(r) * p.f + e0 + i];
      }
      first = MAXMIN ? a[0] == -1 : false;
    }
  }
  using RawL = typename HL::R;
  // one edge into the running value(s); LEX: seeded blocks break ties on COO id
  auto combine = [&](const RawL raw, const A sc, const int32_t pm, const bool is_first, auto lex_c) {
    [[maybe_unused]] constexpr bool LEX = decltype(lex_c)::value;
    T tmp[LE];
    memcpy(tmp, &raw, LB);
#pragma unroll
    for (int j = 0; j < LE; ++j) {
      const A val = scaled ? mul_rn(widen(tmp[j]), sc) : widen(tmp[j]);
      if constexpr (!MAXMIN) {
        v[j] = add_rn(v[j], val);
      } else {
        bool better = is_first || (IS_MIN ? (val < v[j]) : (val > v[j]));
        if constexpr (LEX) better = better || (val == v[j] && static_cast<uint32_t>(pm) < static_cast<uint32_t>(a[j]));
        v[j] = better ? val : v[j];
        a[j] = better ? pm : a[j];
      }
    }
  };
  auto scale_of = [&](int ms, int e) -> A {
    if (w) return mw[ms][e];
    if (gcn) return gcn_scale<A>(mdeg[ms][e], dd);
    return A(1);
  };
  // consume one stage: the row's first edge peeled, then batches of 16 edges
  // whose shared-memory reads are all issued before the ordered combines
  auto stage = [&](const unsigned char* dl, int ms, int n_e, auto lex_c) {
    int e = 0;
    if (first && n_e > 0) {
      combine(*reinterpret_cast<const RawL*>(dl), scale_of(ms, 0), want_arg ? mperm[ms][0] : -1, true, lex_c);
      first = false;
      e = 1;
    }
    constexpr int B = 16;
    for (; e + B <= n_e; e += B) {
      RawL raw[B];
#pragma unroll
      for (int u = 0; u < B; ++u) raw[u] = *reinterpret_cast<const RawL*>(dl + (e + u) * CB);
      A sc[B];
      int32_t pm[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        sc[u] = scale_of(ms, e + u);
        pm[u] = want_arg ? mperm[ms][e + u] : -1;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) combine(raw[u], sc[u], pm[u], false, lex_c);
    }
    for (; e < n_e; ++e)
      combine(*reinterpret_cast<const RawL*>(dl + e * CB), scale_of(ms, e), want_arg ? mperm[ms][e] : -1, false, lex_c);
  };
  const bool lex = MAXMIN && p.accum;

#pragma unroll 1
  for (int i = 0; i < nst; ++i) {
    const int slot = i % kHubRing;
    mbar_wait(&full[slot], static_cast<uint32_t>((i / kHubRing) & 1));
    const int ms = i % kHubMeta;
    const unsigned char* di = hub_data + static_cast<size_t>(slot) * kHubStage * CB;
    const int n_e = stage_edges(i);
    if (lane_valid) {
      if (lex) stage(di + lane * LB, ms, n_e, std::true_type{});
      else stage(di + lane * LB, ms, n_e, std::false_type{});
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  if (!lane_valid) return;
  const int64_t cnt = p.mean_deg ? p.mean_deg[r] : total;
  if (!MAXMIN && p.mean && cnt > 0) {
    const A inv = div_rn(A(1), static_cast<A>(cnt));
#pragma unroll
    for (int j = 0; j < LE; ++j) v[j] = mul_rn(v[j], inv);
  }
  if (!MAXMIN && (p.bias || p.relu)) {
    // the chunk's last lane may hold fewer than LE columns (odd bf16 width)
    const int64_t n_valid = p.f - e0;
    layer_epilogue<A>(v, static_cast<int>(n_valid < LE ? n_valid : LE), p, e0);
  }
  if constexpr (sizeof(T) == 2 && !MAXMIN) {
    if (p.carry != nullptr && !p.carry_out) {
#pragma unroll
      for (int j = 0; j < LE; ++j) p.carry[static_cast<int64_t>(r) * p.f + e0 + j] = v[j];
      return;
    }
  }
  T tmp[LE];
#pragma unroll
  for (int j = 0; j < LE; ++j) tmp[j] = narrow<T, A>(v[j]);
  memcpy(orow + e0, tmp, LB);
  if (p.n_push) {
    const uint32_t m = p.push_mask ? p.push_mask[r] : 0xffffffffu;
    const int64_t ge = (p.push_row0 + r) * p.f + e0;
#pragma unroll
    for (int q = 0; q < GM_MAX_PUSH; ++q)
      if (q < p.n_push && ((m >> q) & 1u)) memcpy(static_cast<T*>(p.push_dst[q]) + ge, tmp, LB);
    __threadfence_system();
  }
  if (want_arg) {
#pragma unroll
    for (int j = 0; j < LE; ++j) p.arg[static_cast<int64_t>(r) * p.f + e0 + j] = a[j];
  }
}

// ---------------------------------------------------------------------------
// Launch helpers
// ---------------------------------------------------------------------------
struct SideStream {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int device = -1;
};
// One library-owned side stream (+ fork/join events) per host thread (spmm.cu).
gm_status side_stream(SideStream** out);

template <typename K>
inline gm_status ensure_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    GM_TRY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(bytes)));
  return GM_OK;
}

#ifndef GM_FLAT_SUM_U  // edges per batch of the one-vector sum/mean sweep (16-byte lanes); C4: 6 / 8 / 10 / 12 -> 4.28 / 4.20 / 7.54 / 8.46 ms (10+ spill)
#define GM_FLAT_SUM_U 8
#endif
template <typename T, int VB, bool MAXMIN>
gm_status launch_flat(const SpmmArgs& p0, int64_t ns, cudaStream_t st) {
  const bool scaled = p0.w != nullptr;
  // at most 32 accumulator elements per lane: 8 float4, 4 bf16x8, 8 double2
  constexpr int kV = VB / static_cast<int>(sizeof(T));
  constexpr int64_t kChunk = 32 * std::min(8, std::max(1, 32 / kV));
  const int64_t chunk = std::min<int64_t>(kChunk, 32 * std::max(1, flat_max_nv()));
  // streaming gathers unless X is small enough to live in L2; hot rows keep
  // an evict_last policy on the plain (unscaled, fresh) path when hinted
  const int lm = p0.stream_x == 0 ? 0 : (p0.src_class != nullptr && !p0.accum) ? 2 : 1;
  const bool epi = p0.carry != nullptr || p0.n_push > 0;
  for (int64_t base = p0.slot_base; base < ns; base += chunk) {
    SpmmArgs p = p0;
    p.slot_base = base;
    p.slot_end = std::min<int64_t>(ns, base + chunk);
    const int64_t slots = p.slot_end - base;
    const int nv = slots <= 32 ? 1 : slots <= 64 ? 2 : slots <= 128 ? 4 : 8;
    const int tpb = flat_threads();
    const unsigned grid = static_cast<unsigned>(ceil_div(p.num_light_windows * 32, tpb));
    if (grid == 0) continue;
#define GM_FLAT_H(NV_, U_, M_, H_)                                                               \
  do {                                                                                           \
    if (p.accum) {                                                                               \
      if (scaled) spmm_flat_kernel<T, VB, NV_, U_, M_, true, true, H_><<<grid, tpb, 0, st>>>(p);    \
      else spmm_flat_kernel<T, VB, NV_, U_, M_, false, true, H_><<<grid, tpb, 0, st>>>(p);          \
    } else if (scaled) spmm_flat_kernel<T, VB, NV_, U_, M_, true, false, H_><<<grid, tpb, 0, st>>>(p); \
    else spmm_flat_kernel<T, VB, NV_, U_, M_, false, false, H_><<<grid, tpb, 0, st>>>(p);           \
  } while (0)
#define GM_FLAT_K(NV_, U_, M_)                                                                     \
  do {                                                                                             \
    if (epi) {  /* carry / push epilogue: unweighted layers, own instantiations */                  \
      if (p.accum) spmm_flat_kernel<T, VB, NV_, U_, M_, false, true, 1, true><<<grid, tpb, 0, st>>>(p);   \
      else spmm_flat_kernel<T, VB, NV_, U_, M_, false, false, 1, true><<<grid, tpb, 0, st>>>(p);          \
      break;                                                                                       \
    }                                                                                              \
    if (lm == 2) {                                                                                 \
      if (scaled) spmm_flat_kernel<T, VB, NV_, U_, M_, true, false, 2><<<grid, tpb, 0, st>>>(p);     \
      else spmm_flat_kernel<T, VB, NV_, U_, M_, false, false, 2><<<grid, tpb, 0, st>>>(p);           \
    }                                                                                              \
    else if (lm == 1) GM_FLAT_H(NV_, U_, M_, 1);                                                   \
    else if (!scaled && !p.accum) spmm_flat_kernel<T, VB, NV_, U_, M_, false, false, 0><<<grid, tpb, 0, st>>>(p); \
    else GM_FLAT_H(NV_, U_, M_, 1);                                                                \
  } while (0)
#define GM_FLAT(NV_, U_)                          \
  do {                                            \
    if constexpr (MAXMIN) {                       \
      if (p.is_min) GM_FLAT_K(NV_, U_, 3);        \
      else GM_FLAT_K(NV_, U_, 2);                 \
    } else if (p.mean) GM_FLAT_K(NV_, U_, 1);     \
    else GM_FLAT_K(NV_, U_, 0);                   \
  } while (0)
    // U x NV raw vectors = 32 registers of gathers in flight per lane
    // (8-byte single-vector rows keep 16 edges in flight; deeper batches for
    // multi-vector rows measured slower on Reddit-shaped F=602)
    if constexpr (VB <= 8) {
      if (nv == 1) GM_FLAT(1, 16);
      else if (nv == 2) GM_FLAT(2, 4);
      else if (nv == 4 || kChunk <= 128) GM_FLAT(4, 2);
      else if constexpr (kChunk > 128) GM_FLAT(8, 1);
    } else {
      if (nv == 1) {
        if constexpr (MAXMIN) GM_FLAT(1, GM_FLAT_MAX_U);
        else GM_FLAT(1, GM_FLAT_SUM_U);
      } else if (nv == 2) GM_FLAT(2, 4);
      else if (nv == 4 || kChunk <= 128) GM_FLAT(4, 2);
      else if constexpr (kChunk > 128) GM_FLAT(8, 1);
    }
#undef GM_FLAT
#undef GM_FLAT_K
#undef GM_FLAT_H
    GM_CHECK_LAUNCH("spmm_flat_kernel");
  }
  return GM_OK;
}

template <typename T, int VB, bool MAXMIN>
gm_status launch_light(const SpmmArgs& p0, int64_t ns, cudaStream_t st) {
  // wide rows without the fused GCN term take the flat edge-stream kernel
  if (p0.gdeg_src == nullptr && ns > 8 && p0.flat_ok)
    return launch_flat<T, VB, MAXMIN>(p0, ns, st);
  // chunk columns so a lane holds <= 8 vectors; pick LPR/NV per chunk
  for (int64_t base = p0.slot_base; base < ns; base += 256) {
    SpmmArgs p = p0;
    p.slot_base = base;
    p.slot_end = std::min<int64_t>(ns, base + 256);
    const int64_t slots = p.slot_end - base;
    int lpr = 32, nv = 1;
    if (slots <= 4) lpr = 4;
    else if (slots <= 8) lpr = 8;
    else if (slots <= 16) lpr = 16;
    else if (slots <= 32) lpr = 32;
    else nv = slots <= 64 ? 2 : slots <= 128 ? 4 : 8;
    const int64_t threads = p.num_windows * lpr;
    const unsigned grid = static_cast<unsigned>(ceil_div(threads, 256));
#define GM_LIGHT(LPR_, NV_, U_) \
  spmm_light_kernel<T, VB, NV_, LPR_, U_, MAXMIN><<<grid, 256, 0, st>>>(p)
    if (nv == 1) {
      if (lpr == 4) GM_LIGHT(4, 1, 8);
      else if (lpr == 8) GM_LIGHT(8, 1, 8);
      else if (lpr == 16) GM_LIGHT(16, 1, 8);
      else GM_LIGHT(32, 1, 8);
    } else if (nv == 2) {
      GM_LIGHT(32, 2, 4);
    } else if (nv == 4) {
      GM_LIGHT(32, 4, 2);
    } else {
      GM_LIGHT(32, 8, 1);
    }
#undef GM_LIGHT
    GM_CHECK_LAUNCH("spmm_light_kernel");
  }
  return GM_OK;
}

template <typename T, int VB, bool MAXMIN>
gm_status launch_heavy(const SpmmArgs& p0, int64_t num_heavy, int64_t ns, cudaStream_t st) {
  using A = typename AccOf<T>::type;
  constexpr int64_t kChunk = 4 * kHeavyThreads;  // slots per column chunk (MH <= 4)
  for (int64_t base = p0.slot_base; base < ns; base += kChunk) {
    SpmmArgs p = p0;
    p.slot_base = base;
    p.slot_end = std::min<int64_t>(ns, base + kChunk);
    const int64_t slots = p.slot_end - base;
    const int rowb = static_cast<int>(slots * VB);
    int se = static_cast<int>(std::min<int64_t>(128, std::max<int64_t>(2, 65536 / (kRing * rowb))));
    const size_t smem = heavy_smem_bytes<A>(se, rowb);
    const int mh = slots <= kHeavyThreads ? 1 : slots <= 2 * kHeavyThreads ? 2 : 4;
#define GM_HEAVY(MH_)                                                                    \
  do {                                                                                   \
    auto kern = spmm_heavy_kernel<T, VB, MH_, MAXMIN>;                                   \
    gm_status s_ = ensure_smem(kern, smem);                                              \
    if (s_ != GM_OK) return s_;                                                          \
    kern<<<static_cast<unsigned>(num_heavy), kHeavyThreads, smem, st>>>(p, se);          \
  } while (0)
    if (mh == 1) GM_HEAVY(1);
    else if (mh == 2) GM_HEAVY(2);
    else GM_HEAVY(4);
#undef GM_HEAVY
    GM_CHECK_LAUNCH("spmm_heavy_kernel");
  }
  return GM_OK;
}

// Hub rows: grid (column chunks, hub rows) of one-warp CTAs, longest row first.
template <typename T, int VB, bool MAXMIN>
gm_status launch_hub(const SpmmArgs& p, int64_t num_heavy, cudaStream_t st) {
  if constexpr (VB < 4) {
    return fail(GM_ERR_INVALID_ARGUMENT, "hub kernel needs >= 4-byte row alignment");
  } else {
    const int64_t row_bytes = p.f * static_cast<int64_t>(sizeof(T));
    constexpr int GV = VB > 16 ? 16 : VB;
    // A/B variant (GM_HUB_LANE8=1): fp32 rows of 8-byte multiples on 8-byte lanes
    // (W = 2: half the CTAs per hub row). Bit-identical, but slower on C4: hub
    // kernel alone 0.28 -> 0.44 ms, sum call 4.24 -> 4.39 ms (each CTA's chain
    // of stages carries twice the copies; ring 8 no better)
    if constexpr (sizeof(T) == 4 && VB >= 8) {
      static const bool lane8 = [] { const char* e = getenv("GM_HUB_LANE8"); return e && atoi(e) != 0; }();
      if (lane8) {
        constexpr int CB2 = HubLane<T, 2>::CB;
        const unsigned grid = static_cast<unsigned>(ceil_div(row_bytes, CB2) * num_heavy);
        auto kern = !MAXMIN ? spmm_hub_kernel<T, GV, 0, 2>
                    : p.is_min ? spmm_hub_kernel<T, GV, 3, 2> : spmm_hub_kernel<T, GV, 2, 2>;
        gm_status s_ = ensure_smem(kern, hub_smem_bytes<T, 2>());
        if (s_ != GM_OK) return s_;
        kern<<<grid, 64, hub_smem_bytes<T, 2>(), st>>>(p);
        GM_CHECK_LAUNCH("spmm_hub_kernel");
        return GM_OK;
      }
    }
    constexpr int CB = HubLane<T>::CB;
    const unsigned grid = static_cast<unsigned>(ceil_div(row_bytes, CB) * num_heavy);
    auto kern = !MAXMIN ? spmm_hub_kernel<T, GV, 0>
                : p.is_min ? spmm_hub_kernel<T, GV, 3>
                           : spmm_hub_kernel<T, GV, 2>;
    gm_status s_ = ensure_smem(kern, hub_smem_bytes<T>());
    if (s_ != GM_OK) return s_;
    kern<<<grid, 64, hub_smem_bytes<T>(), st>>>(p);
    GM_CHECK_LAUNCH("spmm_hub_kernel");
    return GM_OK;
  }
}
// GM_HUB_V1=1 selects the original CTA-per-row hub kernel (comparison only).
inline bool hub_v1() {
  static const bool on = [] { const char* e = getenv("GM_HUB_V1"); return e && atoi(e) != 0; }();
  return on;
}
// Wide rows (>= 1 KB: Reddit-shaped F=602 fp32, where hubs carry a large share
// of the edges) keep the CTA-per-row kernel: its 256 threads accumulate a
// whole row's columns at once.
template <typename T, int VB, bool MAXMIN>
gm_status launch_hubs(const SpmmArgs& p, int64_t num_heavy, int64_t ns, cudaStream_t st) {
  static const bool wide_v1 = [] { const char* e = getenv("GM_HUB_WIDE_V1"); return !e || atoi(e) != 0; }();
  // column blocks (p.slot_base > 0 or a partial range) need the slot-ranged kernel
  const bool ranged = p.slot_base > 0 || ns < p.f * static_cast<int64_t>(sizeof(T)) / VB;
  if (hub_v1() || ranged || (wide_v1 && p.f * static_cast<int64_t>(sizeof(T)) >= kWideRowBytes))
    return launch_heavy<T, VB, MAXMIN>(p, num_heavy, ns, st);
  return launch_hub<T, VB, MAXMIN>(p, num_heavy, st);
}

template <typename T, int VB>
gm_status dispatch_vb(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy,
                             int64_t ns, cudaStream_t st) {
  if (p.l2_block_slots > 0 && p.l2_block_slots < ns) {
    // L2 column blocking: one column block after another, each complete
    // (every column's accumulation order is unchanged: results are identical)
    for (int64_t b0 = 0; b0 < ns; b0 += p.l2_block_slots) {
      SpmmArgs pb = p;
      pb.slot_base = b0;
      pb.l2_block_slots = 0;
      const gm_status s = dispatch_vb<T, VB>(pb, maxmin, use_heavy, num_heavy, std::min(ns, b0 + p.l2_block_slots), st);
      if (s != GM_OK) return s;
    }
    return GM_OK;
  }
  if constexpr (VB >= 4) {
  if (use_heavy) {
    // profiling only (GM_PROF_SKIP=1: no hub kernel, 2: no light kernel) — results are incomplete
    static const int prof_skip = [] { const char* e = getenv("GM_PROF_SKIP"); return e ? atoi(e) : 0; }();
    if (prof_skip == 1) return maxmin ? launch_light<T, VB, true>(p, ns, st) : launch_light<T, VB, false>(p, ns, st);
    if (prof_skip == 2) return maxmin ? launch_hubs<T, VB, true>(p, num_heavy, ns, st) : launch_hubs<T, VB, false>(p, num_heavy, ns, st);
    SideStream* ss = nullptr;
    gm_status s = side_stream(&ss);
    if (s != GM_OK) return s;
    GM_TRY_CUDA(cudaEventRecord(ss->fork, st));
    GM_TRY_CUDA(cudaStreamWaitEvent(ss->side, ss->fork, 0));
    s = maxmin ? launch_hubs<T, VB, true>(p, num_heavy, ns, ss->side)
               : launch_hubs<T, VB, false>(p, num_heavy, ns, ss->side);
    if (s != GM_OK) return s;
    GM_TRY_CUDA(cudaEventRecord(ss->join, ss->side));
    s = maxmin ? launch_light<T, VB, true>(p, ns, st) : launch_light<T, VB, false>(p, ns, st);
    if (s != GM_OK) return s;
    GM_TRY_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
    return GM_OK;
  }
  }
  (void)num_heavy;
  return maxmin ? launch_light<T, VB, true>(p, ns, st) : launch_light<T, VB, false>(p, ns, st);
}


// Per-dtype dispatch, instantiated in spmm_f32.cu / spmm_f64.cu / spmm_bf16.cu.
gm_status spmm_dispatch_f32(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy, int64_t ns, int vb,
                            cudaStream_t st);
gm_status spmm_dispatch_f64(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy, int64_t ns, int vb,
                            cudaStream_t st);
gm_status spmm_dispatch_bf16(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy, int64_t ns, int vb,
                             cudaStream_t st);

}  // namespace gm
