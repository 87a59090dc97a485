// backward.cu — pieces of the spmm backward (message_passing.hpp:119-166)
// that are not themselves an SpMM:
//   gm_scale_rows_div : scaled_g(v, j) = g[v][j] / S(max(deg[v], 1))   (:128-132)
//   gm_edge_dot       : dw[i] = sum_j scaled_g(dst[i], j) * x[src[i], j] (:156-165)
// dx itself is gm_spmm over the CSR by source (the transposed product, :143-152).
// All arithmetic is IEEE round-to-nearest with no contraction, in the
// reference's order (sequential in j), so results are bit-identical.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "vec.cuh"

namespace gm {

template <typename S>
__global__ void scale_rows_div_kernel(const S* __restrict__ in, int64_t rows, int64_t f,
                                      const int32_t* __restrict__ deg, S* __restrict__ out) {
  const int64_t total = rows * f;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / f;
    const int32_t d = deg[r] > 1 ? deg[r] : 1;
    out[i] = div_rn(in[i], static_cast<S>(d));
  }
}

// One thread per edge, COO order (coalesced src/dst/dw); both rows are read
// sequentially by the thread (L1-cached: each 128-B line serves its next loads).
template <typename S>
__global__ void __launch_bounds__(256) edge_dot_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                                                       int64_t e, const S* __restrict__ a, const S* __restrict__ b,
                                                       int64_t f, S* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const S* ar = a + dst[i] * f;
    const S* br = b + src[i] * f;
    S acc = S(0);
    int64_t j = 0;
    if constexpr (sizeof(S) == 4) {
      if ((f & 3) == 0) {
        const float4* a4 = reinterpret_cast<const float4*>(ar);
        const float4* b4 = reinterpret_cast<const float4*>(br);
#pragma unroll 4
        for (int64_t q = 0; q < f / 4; ++q) {
          const float4 u = __ldg(a4 + q), v = __ldg(b4 + q);
          acc = add_rn(acc, mul_rn(u.x, v.x));
          acc = add_rn(acc, mul_rn(u.y, v.y));
          acc = add_rn(acc, mul_rn(u.z, v.z));
          acc = add_rn(acc, mul_rn(u.w, v.w));
        }
        j = f;
      }
    }
    for (; j < f; ++j) acc = add_rn(acc, mul_rn(__ldg(ar + j), __ldg(br + j)));
    out[i] = acc;
  }
}

// Warp-cooperative variant: a warp owns 32 edges; per 32-column chunk the
// lanes load the chunk of all 64 rows (32 edges x {a[dst], b[src]}) with
// coalesced 128-byte accesses into padded shared memory, then every lane runs
// its own edge's products over the chunk in ascending column order — the same
// sequential mul-then-add chain as the reference (:159-163), so dw stays
// bit-identical while the row gathers become coalesced.
constexpr int kDotWarps = 4;
template <typename S>
__device__ __forceinline__ void cp_async_elem(S* smem, const S* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(S) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
template <typename S>
__global__ void __launch_bounds__(kDotWarps * 32) edge_dot_warp_kernel(const int64_t* __restrict__ src,
                                                                       const int64_t* __restrict__ dst, int64_t e,
                                                                       const S* __restrict__ a, const S* __restrict__ b,
                                                                       int64_t f, S* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char dot_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // one {a chunk, b chunk} buffer per warp (a second, prefetching buffer halves
  // the resident warps and measured slower)
  S* buf = reinterpret_cast<S*>(dot_smem) + static_cast<size_t>(wib) * 2 * 32 * 33;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kDotWarps;
  for (int64_t base = (static_cast<int64_t>(blockIdx.x) * kDotWarps + wib) * 32; base < e; base += nw * 32) {
    const int64_t my = base + lane;
    const int64_t ra = my < e ? dst[my] : 0;
    const int64_t rb = my < e ? src[my] : 0;
    const int ne = static_cast<int>(e - base < 32 ? e - base : 32);
    auto issue = [&](int64_t c0, S* sa) {
      const int cw = static_cast<int>(f - c0 < 32 ? f - c0 : 32);
      S* sb = sa + 32 * 33;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const int64_t rat = __shfl_sync(0xffffffffu, ra, t);
        const int64_t rbt = __shfl_sync(0xffffffffu, rb, t);
        if (t < ne && lane < cw) {
          cp_async_elem<S>(sa + t * 33 + lane, a + rat * f + c0 + lane);
          cp_async_elem<S>(sb + t * 33 + lane, b + rbt * f + c0 + lane);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    S acc = S(0);
    for (int64_t c0 = 0; c0 < f; c0 += 32) {
      const int cw = static_cast<int>(f - c0 < 32 ? f - c0 : 32);
      issue(c0, buf);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (lane < ne) {
        const S* pa = buf + lane * 33;
        const S* pb = pa + 32 * 33;
        for (int j = 0; j < cw; ++j) acc = add_rn(acc, mul_rn(pa[j], pb[j]));
      }
      __syncwarp();
    }
    if (my < e) out[my] = acc;
  }
}

// CSC-ordered variant: entry k of a destination-grouped view (rows[k] = its
// destination, col[k] = its source, perm[k] = its COO position). Consecutive
// entries share the destination row, so the a-row chunks of a warp's 32
// entries are mostly the same lines (L1 hits) and DRAM traffic drops to about
// one b-row per edge; the result lands at out[perm[k]].
template <typename S>
__global__ void __launch_bounds__(kDotWarps * 32) edge_dot_csc_kernel(const int32_t* __restrict__ rows,
                                                                      const int32_t* __restrict__ col,
                                                                      const int32_t* __restrict__ perm, int64_t k0,
                                                                      int64_t e, const S* __restrict__ a,
                                                                      const S* __restrict__ b, int64_t f,
                                                                      S* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char dot_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  S* buf = reinterpret_cast<S*>(dot_smem) + static_cast<size_t>(wib) * 2 * 32 * 33;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kDotWarps;
  for (int64_t base = (static_cast<int64_t>(blockIdx.x) * kDotWarps + wib) * 32; base < e; base += nw * 32) {
    const int64_t my = base + lane;
    const int64_t ra = my < e ? rows[k0 + my] : 0;
    const int64_t rb = my < e ? col[k0 + my] : 0;
    const int ne = static_cast<int>(e - base < 32 ? e - base : 32);
    S acc = S(0);
    for (int64_t c0 = 0; c0 < f; c0 += 32) {
      const int cw = static_cast<int>(f - c0 < 32 ? f - c0 : 32);
      S* sa = buf;
      S* sb = buf + 32 * 33;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const int64_t rat = __shfl_sync(0xffffffffu, ra, t);
        const int64_t rbt = __shfl_sync(0xffffffffu, rb, t);
        if (t < ne && lane < cw) {
          cp_async_elem<S>(sa + t * 33 + lane, a + rat * f + c0 + lane);
          cp_async_elem<S>(sb + t * 33 + lane, b + rbt * f + c0 + lane);
        }
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (lane < ne) {
        const S* pa = sa + lane * 33;
        const S* pb = sb + lane * 33;
        for (int j = 0; j < cw; ++j) acc = add_rn(acc, mul_rn(pa[j], pb[j]));
      }
      __syncwarp();
    }
    if (my < e) out[perm[k0 + my]] = acc;
  }
}

// fp32 rows of 16-byte multiples: the 32 source rows of a warp's batch are
// gathered into shared memory with 16-byte cp.async (the (row, piece) pairs
// spread over all lanes), double-buffered so batch n+1 streams in while the
// lanes run batch n's dot chains; each lane's destination row (mostly shared
// by consecutive CSC entries) is read straight from L1 with float4 loads. Rows
// wider than kDotChunk floats go through in column chunks. The per-edge chain
// is the same sequential mul/add as above: bit-identical results.
constexpr int kDotV4Warps = 4;
#ifndef GM_DOT_BUFS
#define GM_DOT_BUFS 2
#endif
constexpr int kDotBufs = GM_DOT_BUFS;
#ifndef GM_DOT_SLICE_U
#define GM_DOT_SLICE_U 8  // entries per sub-batch of the column-slice dw kernel
#endif  // staged units per warp (3 and 4 measured slower: fewer resident warps)
// stage unit u = (batch u / nc, column chunk u % nc) of this warp into buffer u % kDotBufs
// 16-byte cp.async; hot source rows (the plan's classes) carry an evict_last
// policy so power-law hub rows stay in L2 across the sweep, the rest default
// priority (evict_first for them measured 7.6 -> 9.3 ms on C4: unlike the
// forward sweep, dw re-reads cold rows within L2's lifetime).
__device__ __forceinline__ void cp_async_16_hint(uint32_t dst, const void* src, bool hot, uint64_t ph) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
               "@q cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %3;\n\t"
               "@!q cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(dst),
               "l"(src), "r"(static_cast<int>(hot)), "l"(ph)
               : "memory");
}

template <int kDotChunk>
__device__ __forceinline__ void dot_v4_issue(int64_t u, int64_t gw, int64_t nw, int nc, int64_t e, int64_t k0,
                                             int64_t f, int stride, const int32_t* __restrict__ col,
                                             const float* __restrict__ b, float* buf, int lane, int32_t& rb_iss,
                                             const uint8_t* __restrict__ src_class, int hot_limit, uint32_t& hot_iss,
                                             uint64_t ph) {
  const int64_t base = (gw + (u / nc) * nw) * 32;
  const int ci = static_cast<int>(u % nc);
  if (ci == 0) {
    rb_iss = base + lane < e ? col[k0 + base + lane] : 0;
    const bool hot = src_class && base + lane < e && src_class[k0 + base + lane] < hot_limit;
    hot_iss = __ballot_sync(0xffffffffu, hot);
  }
  const int ne = static_cast<int>(e - base < 32 ? e - base : 32);
  const int64_t c0 = static_cast<int64_t>(ci) * kDotChunk;
  const int n16 = static_cast<int>((f - c0 < kDotChunk ? f - c0 : kDotChunk) / 4);  // 16-B pieces per row
  float* stage = buf + (u % kDotBufs) * 32 * stride;
  for (int idx = lane; idx < 32 * n16; idx += 32) {
    const int t = idx / n16, pc = idx - t * n16;
    const int32_t rbt = __shfl_sync(0xffffffffu, rb_iss, t);  // every lane reaches the shuffle
    if (t < ne) {
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(stage + t * stride + pc * 4));
      cp_async_16_hint(d, b + static_cast<int64_t>(rbt) * f + c0 + pc * 4, (hot_iss >> t) & 1u, ph);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int kDotChunk>  // floats of a row staged per unit
__global__ void __launch_bounds__(kDotV4Warps * 32) edge_dot_csc_v4_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ col, const int32_t* __restrict__ perm, int64_t k0,
    int64_t e, const float* __restrict__ a, const float* __restrict__ b, int64_t f, int stride,
    float* __restrict__ out, const uint8_t* __restrict__ src_class, int hot_limit) {
  extern __shared__ __align__(16) unsigned char dot_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* buf = reinterpret_cast<float*>(dot_smem) + static_cast<size_t>(wib) * kDotBufs * 32 * stride;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kDotV4Warps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kDotV4Warps + wib;
  const int64_t nb_all = (e + 31) / 32;
  if (gw >= nb_all) return;
  const int nc = static_cast<int>((f + kDotChunk - 1) / kDotChunk);
  const int64_t units = ((nb_all - gw + nw - 1) / nw) * nc;

  int32_t rb_iss = 0;
  uint32_t hot_iss = 0;
  uint64_t ph;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(ph));
  float acc = 0.f;
  int32_t ra = 0;
  for (int64_t u = 0; u < kDotBufs - 1; ++u) {
    if (u < units)
      dot_v4_issue<kDotChunk>(u, gw, nw, nc, e, k0, f, stride, col, b, buf, lane, rb_iss, src_class, hot_limit, hot_iss,
                              ph);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t u = 0; u < units; ++u) {
    if (u + kDotBufs - 1 < units)
      dot_v4_issue<kDotChunk>(u + kDotBufs - 1, gw, nw, nc, e, k0, f, stride, col, b, buf, lane, rb_iss, src_class,
                              hot_limit, hot_iss, ph);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int64_t base = (gw + (u / nc) * nw) * 32;
    const int ci = static_cast<int>(u % nc);
    const int64_t my = base + lane;
    if (ci == 0) {
      acc = 0.f;
      ra = my < e ? rows[k0 + my] : 0;
    }
    const int64_t c0 = static_cast<int64_t>(ci) * kDotChunk;
    const int n4 = static_cast<int>((f - c0 < kDotChunk ? f - c0 : kDotChunk) / 4);
    // the destination row's chunk goes to registers first: all its loads are in
    // flight together (they mostly hit L1/L2: consecutive entries share it)
    float4 av[kDotChunk / 4];
    const float4* pa = reinterpret_cast<const float4*>(a + static_cast<int64_t>(ra) * f + c0);
#pragma unroll
    for (int j = 0; j < kDotChunk / 4; ++j)
      if (j < n4) av[j] = __ldg(pa + j);
    asm volatile("cp.async.wait_group %0;" ::"n"(kDotBufs - 1) : "memory");
    __syncwarp();
    if (my < e) {
      const float* pb = buf + (u % kDotBufs) * 32 * stride + lane * stride;
#pragma unroll
      for (int j = 0; j < kDotChunk / 4; ++j) {
        if (j < n4) {
          const float4 bv = *reinterpret_cast<const float4*>(pb + 4 * j);
          acc = __fadd_rn(acc, __fmul_rn(av[j].x, bv.x));
          acc = __fadd_rn(acc, __fmul_rn(av[j].y, bv.y));
          acc = __fadd_rn(acc, __fmul_rn(av[j].z, bv.z));
          acc = __fadd_rn(acc, __fmul_rn(av[j].w, bv.w));
        }
      }
      if (ci == nc - 1) out[perm[k0 + my]] = acc;
    }
    __syncwarp();  // this stage is refilled by the issue of unit u + kDotBufs
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Column-slice form (the default for fp32 rows of 16-byte multiples): the forward sweep's gather
// pattern — lanes own 16-byte column slices, so an entry's source row is one
// coalesced 400-byte read across the warp — with the products transposed
// through shared memory for the reference's sequential chain. Per sub-batch
// of U entries: all U source-row slices are in flight; lane l forms the
// exact products g[v][j] * x[u][j] of its slice (the destination row's slice
// stays in registers across a row's run of entries) and stores them to row t
// of a [U][F+pad] tile; then lane t < U adds row t's products in j order —
// the same mul-then-add chain, bit-identical.
#ifndef GM_DOT_SLICE_MINB
#define GM_DOT_SLICE_MINB 4
#endif
#ifndef GM_DOT_SLICE_COLD
#define GM_DOT_SLICE_COLD 1  // cold source rows: 1 evict_first (as the forward sweep), 0 default priority
#endif
template <int U>
__global__ void __launch_bounds__(256, GM_DOT_SLICE_MINB) edge_dot_slice_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ col, const int32_t* __restrict__ perm, int64_t k0,
    int64_t e, int64_t per_warp, const float* __restrict__ a, const float* __restrict__ b, int64_t f, int stride,
    float* __restrict__ out, const uint8_t* __restrict__ src_class, int hot_limit) {
  constexpr unsigned FULL = 0xffffffffu;
  // the forward sweep's L2 residency scheme for the gathered source rows:
  // the plan's hot rows evict_last, the rest streamed
  uint64_t pol_hot;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hot));
  extern __shared__ __align__(16) unsigned char dot_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* tile = reinterpret_cast<float*>(dot_smem) + static_cast<size_t>(wib) * U * stride;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t kb = w * per_warp;
  if (kb >= e) return;
  const int64_t ke = min(e, kb + per_warp);
  const uint32_t fu = static_cast<uint32_t>(f);
  const int nsl_all = static_cast<int>(f / 4);
  int32_t vcur = -1;
  float4 gcur = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t t0 = kb; t0 < ke; t0 += U) {
    const int n_e = static_cast<int>(min(static_cast<int64_t>(U), ke - t0));
    int32_t c = 0, r = 0, pm = 0;
    bool hot = false;
    if (lane < n_e) {
      c = col[k0 + t0 + lane];
      r = rows[k0 + t0 + lane];
      pm = perm[k0 + t0 + lane];
      hot = src_class && src_class[k0 + t0 + lane] < hot_limit;
    }
    const uint32_t hmask = __ballot_sync(FULL, hot);
    float acc = 0.f;
    for (int sb = 0; sb < nsl_all; sb += 32) {  // column passes of 32 16-byte slots
      const int nsl = min(32, nsl_all - sb);
      const uint32_t soff = static_cast<uint32_t>(sb + min(lane, nsl - 1)) * 4u;
      float4 xv[U];
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const uint32_t u = static_cast<uint32_t>(__shfl_sync(FULL, c, t));
        const float4* src = reinterpret_cast<const float4*>(b + static_cast<uint64_t>(u) * fu + soff);
        const int ht = static_cast<int>((hmask >> t) & 1u);
#if GM_DOT_SLICE_COLD
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
            "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %6;\n\t"
            "@!q ld.global.cs.nc.v4.f32 {%0,%1,%2,%3}, [%4];\n\t}"
            : "=f"(xv[t].x), "=f"(xv[t].y), "=f"(xv[t].z), "=f"(xv[t].w)
            : "l"(src), "r"(ht), "l"(pol_hot));
#else
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
            "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %6;\n\t"
            "@!q ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n\t}"
            : "=f"(xv[t].x), "=f"(xv[t].y), "=f"(xv[t].z), "=f"(xv[t].w)
            : "l"(src), "r"(ht), "l"(pol_hot));
#endif
      }
      if (nsl_all > 32) vcur = -1;  // the cached destination slice is per column pass
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const int32_t v = __shfl_sync(FULL, r, t);
        if (t < n_e) {
          if (v != vcur) {
            gcur = __ldg(reinterpret_cast<const float4*>(a + static_cast<uint64_t>(static_cast<uint32_t>(v)) * fu + soff));
            vcur = v;
          }
          if (lane < nsl)
            *reinterpret_cast<float4*>(tile + t * stride + (soff - sb * 4)) =
                make_float4(__fmul_rn(gcur.x, xv[t].x), __fmul_rn(gcur.y, xv[t].y), __fmul_rn(gcur.z, xv[t].z),
                            __fmul_rn(gcur.w, xv[t].w));
        }
      }
      __syncwarp();
      if (lane < n_e) {
        const float4* pr = reinterpret_cast<const float4*>(tile + lane * stride);
        for (int q = 0; q < nsl; ++q) {
          const float4 p4 = pr[q];
          acc = __fadd_rn(acc, p4.x);
          acc = __fadd_rn(acc, p4.y);
          acc = __fadd_rn(acc, p4.z);
          acc = __fadd_rn(acc, p4.w);
        }
      }
      __syncwarp();
    }
    if (lane < n_e) out[pm] = acc;
  }
}

// Staged column-slice form: the slice kernel's coalesced gathers, but issued as
// 16-byte cp.async into an S-stage shared-memory ring per warp instead of
// registers, so S-1 sub-batches of U source rows stay in flight while the
// lanes form products and run the chains of the oldest one (no register cost
// for the in-flight data). The destination row's slice is staged beside the
// source rows, once per run of equal destinations within a sub-batch (the
// first entry of each run copies it; the others read that slot). Products are
// written in place over the source slices; lane t < U then adds row t in j
// order — the reference's mul-then-add chain, bit-identical. Rows of <= 128
// floats (one column pass); each warp walks one contiguous entry range.
template <int U, int S>
__global__ void __launch_bounds__(128) edge_dot_staged_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ col, const int32_t* __restrict__ perm, int64_t k0,
    int64_t e, int64_t per_warp, const float* __restrict__ a, const float* __restrict__ b, int64_t f, int stride,
    float* __restrict__ out, const uint8_t* __restrict__ src_class, int hot_limit, int cold_mode) {
  constexpr unsigned FULL = 0xffffffffu;
  uint64_t pol_hot, pol_cold;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hot));
  if (cold_mode == 1)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_cold));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_cold));
  extern __shared__ __align__(16) unsigned char dot_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // per warp: S stages of {x tile [U][stride] float4, g tile [U][stride] float4}, then S x U perms + S lead masks
  const size_t stage_f4 = static_cast<size_t>(2) * U * stride;
  float4* ring = reinterpret_cast<float4*>(dot_smem) + static_cast<size_t>(wib) * S * stage_f4;
  int32_t* mperm = reinterpret_cast<int32_t*>(reinterpret_cast<float4*>(dot_smem) + (blockDim.x >> 5) * S * stage_f4) +
                   static_cast<size_t>(wib) * S * (U + 1);
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t kb = w * per_warp;
  if (kb >= e) return;
  const int64_t ke = min(e, kb + per_warp);
  const uint32_t fu = static_cast<uint32_t>(f);
  const int nsl = static_cast<int>(f / 4);
  const uint32_t soff = static_cast<uint32_t>(min(lane, nsl - 1)) * 4u;
  const int nb = static_cast<int>((ke - kb + U - 1) / U);
  // metadata of the next sub-batch to issue, loaded one issue ahead (its
  // latency hides behind a whole wait + compute step)
  int32_t c_n = 0, r_n = -1, pm_n = 0;
  bool hot_n = false;
  auto load_meta = [&](int bt) {
    c_n = 0;
    r_n = -1;
    pm_n = 0;
    hot_n = false;
    const int64_t t0 = kb + static_cast<int64_t>(bt) * U;
    if (bt < nb && t0 + lane < ke && lane < U) {
      c_n = col[k0 + t0 + lane];
      r_n = rows[k0 + t0 + lane];
      pm_n = perm[k0 + t0 + lane];
      hot_n = src_class && src_class[k0 + t0 + lane] < hot_limit;
    }
  };
  auto issue = [&](int bt) {
    if (bt < nb) {
      const int s = bt % S;
      float4* xs = ring + s * stage_f4;
      float4* gs = xs + U * stride;
      const int64_t t0 = kb + static_cast<int64_t>(bt) * U;
      const int n_e = static_cast<int>(min(static_cast<int64_t>(U), ke - t0));
      const int32_t c = c_n, r = r_n, pm = pm_n;
      const bool hot = hot_n;
      load_meta(bt + 1);
      const int32_t rprev = __shfl_up_sync(FULL, r, 1);
      const uint32_t lead = __ballot_sync(FULL, lane < n_e && (lane == 0 || r != rprev));
      const uint32_t hmask = __ballot_sync(FULL, hot);
      if (lane < U) mperm[s * (U + 1) + lane] = pm;
      if (lane == 0) mperm[s * (U + 1) + U] = static_cast<int32_t>(lead);
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const uint32_t u = static_cast<uint32_t>(__shfl_sync(FULL, c, t));
        const uint32_t v = static_cast<uint32_t>(__shfl_sync(FULL, r, t));
        if (t < n_e && lane < nsl) {
          const uint32_t sx = static_cast<uint32_t>(__cvta_generic_to_shared(xs + t * stride + lane));
          const float* src = b + static_cast<uint64_t>(u) * fu + soff;
          if (cold_mode == 2) {
            cp_async_16_hint(sx, src, (hmask >> t) & 1u, pol_hot);
          } else {
            const uint64_t pol = ((hmask >> t) & 1u) ? pol_hot : pol_cold;
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sx), "l"(src), "l"(pol)
                         : "memory");
          }
          if ((lead >> t) & 1u) {
            const uint32_t sg = static_cast<uint32_t>(__cvta_generic_to_shared(gs + t * stride + lane));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sg),
                         "l"(a + static_cast<uint64_t>(v) * fu + soff)
                         : "memory");
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  load_meta(0);
#pragma unroll
  for (int p = 0; p < S - 1; ++p) issue(p);
  for (int bt = 0; bt < nb; ++bt) {
    issue(bt + S - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncwarp();
    const int s = bt % S;
    float4* xs = ring + s * stage_f4;
    const float4* gs = xs + U * stride;
    const int64_t t0 = kb + static_cast<int64_t>(bt) * U;
    const int n_e = static_cast<int>(min(static_cast<int64_t>(U), ke - t0));
    const uint32_t lead = static_cast<uint32_t>(mperm[s * (U + 1) + U]);
    if (lane < nsl) {
#pragma unroll
      for (int t = 0; t < U; ++t) {
        if (t < n_e) {
          const int lt = 31 - __clz(lead & ((2u << t) - 1u));
          const float4 xv = xs[t * stride + lane];
          const float4 gv = gs[lt * stride + lane];
          xs[t * stride + lane] = make_float4(__fmul_rn(gv.x, xv.x), __fmul_rn(gv.y, xv.y), __fmul_rn(gv.z, xv.z),
                                              __fmul_rn(gv.w, xv.w));
        }
      }
    }
    __syncwarp();
    if (lane < n_e) {
      const float4* pr = xs + lane * stride;
      float acc = 0.f;
#pragma unroll 4
      for (int q = 0; q < nsl; ++q) {
        const float4 p4 = pr[q];
        acc = __fadd_rn(acc, p4.x);
        acc = __fadd_rn(acc, p4.y);
        acc = __fadd_rn(acc, p4.z);
        acc = __fadd_rn(acc, p4.w);
      }
      out[mperm[s * (U + 1) + lane]] = acc;
    }
    __syncwarp();  // stage s is refilled by the issue of sub-batch bt + S
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__global__ void entry_rows_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int32_t* __restrict__ out) {
  // one warp per row: the row id for each of its entries (positions relative to rowptr[0])
  const int lane = threadIdx.x & 31;
  const int64_t k0 = rowptr[0];
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw)
    for (int64_t k = rowptr[r] + lane; k < rowptr[r + 1]; k += 32) out[k - k0] = static_cast<int32_t>(r);
}

static unsigned grid_of(int64_t n) {
  return static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), kNumSMs * 32));
}

}  // namespace gm

using namespace gm;

extern "C" {

GM_API gm_status gm_scale_rows_div(gm_dtype dtype, const void* in, int64_t rows, int64_t f, const int32_t* deg,
                                   void* out, gm_stream_t stream) {
  GM_REQUIRE(rows >= 0 && f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_scale_rows_div: negative size");
  GM_REQUIRE(dtype == GM_F32 || dtype == GM_F64, GM_ERR_INVALID_ARGUMENT, "gm_scale_rows_div: f32/f64 only");
  if (rows == 0 || f == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F32)
    scale_rows_div_kernel<float><<<grid_of(rows * f), 256, 0, st>>>(static_cast<const float*>(in), rows, f, deg,
                                                                    static_cast<float*>(out));
  else
    scale_rows_div_kernel<double><<<grid_of(rows * f), 256, 0, st>>>(static_cast<const double*>(in), rows, f, deg,
                                                                     static_cast<double*>(out));
  GM_CHECK_LAUNCH("scale_rows_div_kernel");
  return GM_OK;
}

GM_API gm_status gm_csr_entry_rows(const gm_csr* csr, int32_t* rows_out, gm_stream_t stream) {
  GM_REQUIRE(csr && rows_out, GM_ERR_INVALID_ARGUMENT, "gm_csr_entry_rows: null argument");
  if (csr->num_rows == 0 || csr->nnz == 0) return GM_OK;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(csr->num_rows, 8), kNumSMs * 32));
  entry_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(csr->rowptr, csr->num_rows, rows_out);
  GM_CHECK_LAUNCH("entry_rows_kernel");
  return GM_OK;
}

GM_API gm_status gm_edge_dot_csc(gm_dtype dtype, const gm_csr* csc, const gm_spmm_plan* plan,
                                 const int32_t* entry_rows, const void* a_by_dst, const void* b_by_src, int64_t f,
                                 void* out, gm_stream_t stream) {
  GM_REQUIRE(csc && entry_rows, GM_ERR_INVALID_ARGUMENT, "gm_edge_dot_csc: null argument");
  GM_REQUIRE(dtype == GM_F32 || dtype == GM_F64, GM_ERR_INVALID_ARGUMENT, "gm_edge_dot_csc: f32/f64 only");
  GM_REQUIRE(csc->nnz == 0 || csc->perm, GM_ERR_INVALID_ARGUMENT, "gm_edge_dot_csc: csc->perm required");
  if (csc->nnz == 0 || csc->num_rows == 0) return GM_OK;
  int64_t k0 = 0;
  cudaStream_t st = as_stream(stream);
  GM_TRY_CUDA(cudaMemcpyAsync(&k0, csc->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  // entry_rows is indexed from the view's first entry: pass it pre-offset by -k0
  static const bool v4_env = [] { const char* ev = getenv("GM_EDGE_DOT_V4"); return !(ev && ev[0] == '0'); }();
  // column-slice kernel (default; GM_EDGE_DOT_SLICE=0 selects the row-staged v4
  // kernel): same-box C4 6.56 vs 7.57 ms, sub-batches of 4/6/8/16 entries
  // 8.13/6.77/6.56/7.26 ms, 64-512 entries per warp alike, 80 registers 7.0 ms
  static const bool slice_env = [] { const char* ev = getenv("GM_EDGE_DOT_SLICE"); return !(ev && ev[0] == '0'); }();
  // staged column-slice kernel, an A/B variant (GM_DOT_STAGED=U,S selects the ring
  // shape, unset/0 keeps the slice kernel): bit-identical but 14.2-14.6 ms on C4
  // for every ring shape (8,3 / 8,4 / 4,4 / 4,6 / 16,2 / 16,3) vs 6.55 — at 8-16
  // resident warps per SM (ring-limited) the chains run on U lanes and the warp
  // issues ~780 instructions per sub-batch (6.0G in all, 35% issue active)
  static const int staged_cfg = [] {
    const char* ev = getenv("GM_DOT_STAGED");
    if (!ev) return 0;
    if (ev[0] == '0') return 0;
    return atoi(ev) * 10 + (strchr(ev, ',') ? atoi(strchr(ev, ',') + 1) : 3);
  }();
  if (dtype == GM_F32 && staged_cfg && f % 4 == 0 && f <= 128 &&
      ((reinterpret_cast<uintptr_t>(a_by_dst) | reinterpret_cast<uintptr_t>(b_by_src)) & 15) == 0) {
    const int nsl = static_cast<int>(f / 4);
    const int stride = nsl | 1;  // odd 16-byte units: conflict-free float4 reads of consecutive rows
    const uint8_t* cls = nullptr;
    int limit = 0;
    if (plan && plan->src_class && plan->l2_hot_bytes > 0) {
      const double hot_rows = static_cast<double>(plan->l2_hot_bytes) / static_cast<double>(f * 4);
      limit = static_cast<int>(std::floor(4.0 * std::log2(1.0 + hot_rows)));
      if (plan->hot_edge_frac[std::min(limit, GM_PLAN_CLASSES - 1)] >= 0.15) cls = plan->src_class;
    }
    // cold source rows: 2 plain cp.async (hot rows alone carry the evict_last hint), 1 evict_first, 0 evict_normal hint
    static const int cold_first = [] { const char* ev = getenv("GM_DOT_STAGED_COLD"); return ev ? atoi(ev) : 2; }();
    static const int64_t pw_env = [] { const char* ev = getenv("GM_DOT_STAGED_PER_WARP"); return ev ? atoll(ev) : 0; }();
    auto launch = [&](auto kern, int U, int S) -> gm_status {
      const size_t smem = static_cast<size_t>(4) * (static_cast<size_t>(S) * 2 * U * stride * 16 + S * (U + 1) * 4);
      GM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      int per_sm = 0;
      GM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
      int dev = 0, sms = kNumSMs;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t resident = static_cast<int64_t>(std::max(per_sm, 1)) * sms * 4;
      int64_t per_warp = pw_env > 0 ? pw_env : ceil_div(csc->nnz, resident);
      per_warp = std::max<int64_t>(ceil_div(per_warp, U) * U, U);
      const int64_t warps = ceil_div(csc->nnz, per_warp);
      kern<<<static_cast<unsigned>(ceil_div(warps, 4)), 128, smem, st>>>(
          entry_rows - k0, csc->col, csc->perm, k0, csc->nnz, per_warp, static_cast<const float*>(a_by_dst),
          static_cast<const float*>(b_by_src), f, stride, static_cast<float*>(out), cls, limit, cold_first);
      GM_CHECK_LAUNCH("edge_dot_staged_kernel");
      return GM_OK;
    };
    switch (staged_cfg) {
      case 44: return launch(edge_dot_staged_kernel<4, 4>, 4, 4);
      case 46: return launch(edge_dot_staged_kernel<4, 6>, 4, 6);
      case 84: return launch(edge_dot_staged_kernel<8, 4>, 8, 4);
      case 162: return launch(edge_dot_staged_kernel<16, 2>, 16, 2);
      case 163: return launch(edge_dot_staged_kernel<16, 3>, 16, 3);
      default: return launch(edge_dot_staged_kernel<8, 3>, 8, 3);
    }
  }
  if (dtype == GM_F32 && slice_env && f % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(a_by_dst) | reinterpret_cast<uintptr_t>(b_by_src)) & 15) == 0) {
    constexpr int kU = GM_DOT_SLICE_U;
    // tile row stride: one column pass (<= 128 floats) + 4, an odd number of
    // 16-byte units (conflict-free float4 reads of 8 consecutive rows)
    int stride = static_cast<int>(std::min<int64_t>(f, 128));
    if ((stride / 4) % 2 == 0) stride += 4;
    // warps per CTA (GM_EDGE_DOT_WARPS: 8, 4 or 2; same box 6.56 / 6.53 / 6.52 ms)
    static const int wpc = [] {
      const char* ev = getenv("GM_EDGE_DOT_WARPS");
      const int v = ev ? atoi(ev) : 2;
      return (v == 4 || v == 8) ? v : 2;
    }();
    const size_t smem = sizeof(float) * kU * stride * wpc;
    GM_TRY_CUDA(cudaFuncSetAttribute(edge_dot_slice_kernel<kU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    static const int64_t per_warp = [] { const char* ev = getenv("GM_EDGE_DOT_PER_WARP"); return ev ? atoll(ev) : 256; }();
    const int64_t warps = ceil_div(csc->nnz, per_warp);
    // L2 residency of hot source rows: the same budget rule as gm_spmm
    const uint8_t* cls = nullptr;
    int limit = 0;
    if (plan && plan->src_class && plan->l2_hot_bytes > 0) {
      const double hot_rows = static_cast<double>(plan->l2_hot_bytes) / static_cast<double>(f * 4);
      limit = static_cast<int>(std::floor(4.0 * std::log2(1.0 + hot_rows)));
      if (plan->hot_edge_frac[std::min(limit, GM_PLAN_CLASSES - 1)] >= 0.15) cls = plan->src_class;
    }
    edge_dot_slice_kernel<kU><<<static_cast<unsigned>(ceil_div(warps, wpc)), 32 * wpc, smem, st>>>(
        entry_rows - k0, csc->col, csc->perm, k0, csc->nnz, per_warp, static_cast<const float*>(a_by_dst),
        static_cast<const float*>(b_by_src), f, stride, static_cast<float*>(out), cls, limit);
    GM_CHECK_LAUNCH("edge_dot_slice_kernel");
    return GM_OK;
  }
  if (dtype == GM_F32 && v4_env && f % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(a_by_dst) | reinterpret_cast<uintptr_t>(b_by_src)) & 15) == 0) {
    // column chunk per staged unit (GM_EDGE_DOT_CHUNK: 16 / 32 / 64 / 128 floats)
    static const int chunk_env = [] { const char* ev = getenv("GM_EDGE_DOT_CHUNK"); return ev ? atoi(ev) : 32; }();
    const int chunk = chunk_env == 128 ? 128 : chunk_env == 64 ? 64 : chunk_env == 16 ? 16 : 32;
    // row stride in smem: 16-B aligned, odd in 16-B units (conflict-free float4 reads)
    int stride = static_cast<int>(std::min<int64_t>(f, chunk));
    if ((stride / 4) % 2 == 0) stride += 4;
    const size_t smem = sizeof(float) * kDotBufs * 32 * stride * kDotV4Warps;
    auto kern = chunk == 128 ? edge_dot_csc_v4_kernel<128>
                : chunk == 64 ? edge_dot_csc_v4_kernel<64>
                : chunk == 16 ? edge_dot_csc_v4_kernel<16> : edge_dot_csc_v4_kernel<32>;
    GM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    GM_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDotV4Warps * 32, smem));
    const unsigned blocks = static_cast<unsigned>(
        std::min<int64_t>(ceil_div(csc->nnz, 32 * kDotV4Warps), static_cast<int64_t>(kNumSMs) * std::max(per_sm, 1)));
    // L2 residency of hot source rows: the same budget rule as gm_spmm
    const uint8_t* cls = nullptr;
    int limit = 0;
    if (plan && plan->src_class && plan->l2_hot_bytes > 0) {
      const double hot_rows = static_cast<double>(plan->l2_hot_bytes) / static_cast<double>(f * 4);
      limit = static_cast<int>(std::floor(4.0 * std::log2(1.0 + hot_rows)));
      if (plan->hot_edge_frac[std::min(limit, GM_PLAN_CLASSES - 1)] >= 0.15) cls = plan->src_class;
    }
    kern<<<blocks, kDotV4Warps * 32, smem, st>>>(
        entry_rows - k0, csc->col, csc->perm, k0, csc->nnz, static_cast<const float*>(a_by_dst),
        static_cast<const float*>(b_by_src), f, stride, static_cast<float*>(out), cls, limit);
    GM_CHECK_LAUNCH("edge_dot_csc_v4_kernel");
    return GM_OK;
  }
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(csc->nnz, 32 * kDotWarps), kNumSMs * 64));
  if (dtype == GM_F32) {
    const size_t smem = sizeof(float) * 2 * 32 * 33 * kDotWarps;
    GM_TRY_CUDA(cudaFuncSetAttribute(edge_dot_csc_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(float) * 2 * 32 * 33 * kDotWarps)));  // per device, so per call
    edge_dot_csc_kernel<float><<<blocks, kDotWarps * 32, smem, st>>>(
        entry_rows - k0, csc->col, csc->perm, k0, csc->nnz, static_cast<const float*>(a_by_dst),
        static_cast<const float*>(b_by_src), f, static_cast<float*>(out));
  } else {
    const size_t smem = sizeof(double) * 2 * 32 * 33 * kDotWarps;
    GM_TRY_CUDA(cudaFuncSetAttribute(edge_dot_csc_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(double) * 2 * 32 * 33 * kDotWarps)));  // per device, so per call
    edge_dot_csc_kernel<double><<<blocks, kDotWarps * 32, smem, st>>>(
        entry_rows - k0, csc->col, csc->perm, k0, csc->nnz, static_cast<const double*>(a_by_dst),
        static_cast<const double*>(b_by_src), f, static_cast<double*>(out));
  }
  GM_CHECK_LAUNCH("edge_dot_csc_kernel");
  return GM_OK;
}

GM_API gm_status gm_edge_dot(gm_dtype dtype, const int64_t* src, const int64_t* dst, int64_t num_edges,
                             const void* a_by_dst, const void* b_by_src, int64_t f, void* out, gm_stream_t stream) {
  GM_REQUIRE(num_edges >= 0 && f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_edge_dot: negative size");
  GM_REQUIRE(dtype == GM_F32 || dtype == GM_F64, GM_ERR_INVALID_ARGUMENT, "gm_edge_dot: f32/f64 only");
  if (num_edges == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(num_edges, 32 * kDotWarps), kNumSMs * 64));
  if (dtype == GM_F32) {
    const size_t smem = sizeof(float) * 2 * 32 * 33 * kDotWarps;
    GM_TRY_CUDA(cudaFuncSetAttribute(edge_dot_warp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(float) * 2 * 32 * 33 * kDotWarps)));  // per device, so per call
    edge_dot_warp_kernel<float><<<blocks, kDotWarps * 32, smem, st>>>(
        src, dst, num_edges, static_cast<const float*>(a_by_dst), static_cast<const float*>(b_by_src), f,
        static_cast<float*>(out));
  } else {
    const size_t smem = sizeof(double) * 2 * 32 * 33 * kDotWarps;
    GM_TRY_CUDA(cudaFuncSetAttribute(edge_dot_warp_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(double) * 2 * 32 * 33 * kDotWarps)));  // per device, so per call
    edge_dot_warp_kernel<double><<<blocks, kDotWarps * 32, smem, st>>>(
        src, dst, num_edges, static_cast<const double*>(a_by_dst), static_cast<const double*>(b_by_src), f,
        static_cast<double*>(out));
  }
  GM_CHECK_LAUNCH("edge_dot_warp_kernel");
  return GM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// hetero combine (hetero.hpp:338-343 InterCombine::sum + layer_update :579-580):
//   out = ((((p0 + p1) + ...) + p_{n-1}) + self) + bias      (fp32, this order)
// ---------------------------------------------------------------------------
namespace gm {
struct CombineArgs {
  const float* parts[8];
  int n_parts;
  const float* self;
  const float* bias;
  int64_t rows;
  int64_t f;
  float* out;
};
// float4 rows, one warp per row (f % 4 == 0, 16-byte aligned arrays)
__global__ void hetero_combine_vec_kernel(const CombineArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t f4 = a.f / 4;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < a.rows; r += nw) {
    for (int64_t c = lane; c < f4; c += 32) {
      const int64_t i = r * f4 + c;
      float4 acc = a.n_parts > 0 ? __ldcs(reinterpret_cast<const float4*>(a.parts[0]) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = 1; p < a.n_parts; ++p) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(a.parts[p]) + i);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      if (a.self) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(a.self) + i);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      if (a.bias) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(a.bias) + c);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      __stcs(reinterpret_cast<float4*>(a.out) + i, acc);
    }
  }
}

__global__ void hetero_combine_kernel(const CombineArgs a) {
  const int64_t total = a.rows * a.f;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = a.n_parts > 0 ? a.parts[0][i] : 0.0f;
    for (int p = 1; p < a.n_parts; ++p) acc = __fadd_rn(acc, a.parts[p][i]);
    if (a.self) acc = __fadd_rn(acc, a.self[i]);
    if (a.bias) acc = __fadd_rn(acc, a.bias[i % a.f]);
    a.out[i] = acc;
  }
}
}  // namespace gm

extern "C" GM_API gm_status gm_hetero_combine(const float* const* parts, int32_t n_parts, const float* self_term,
                                              const float* bias, int64_t rows, int64_t f, float* out,
                                              gm_stream_t stream) {
  using namespace gm;
  GM_REQUIRE(n_parts >= 0 && n_parts <= 8, GM_ERR_INVALID_ARGUMENT, "gm_hetero_combine: at most 8 parts");
  if (rows == 0 || f == 0) return GM_OK;
  CombineArgs a{};
  for (int p = 0; p < n_parts; ++p) a.parts[p] = parts[p];
  a.n_parts = n_parts;
  a.self = self_term;
  a.bias = bias;
  a.rows = rows;
  a.f = f;
  a.out = out;
  uintptr_t al = reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(self_term) |
                 reinterpret_cast<uintptr_t>(bias) | static_cast<uintptr_t>(f * 4);
  for (int p = 0; p < n_parts; ++p) al |= reinterpret_cast<uintptr_t>(parts[p]);
  if (al % 16 == 0) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(rows, 8), kNumSMs * 16));
    hetero_combine_vec_kernel<<<grid, 256, 0, as_stream(stream)>>>(a);
  } else {
    hetero_combine_kernel<<<grid_of(rows * f), 256, 0, as_stream(stream)>>>(a);
  }
  GM_CHECK_LAUNCH("hetero_combine_kernel");
  return GM_OK;
}
