// maxbwd.cu — backward of the max / min aggregation path
// (message_passing.hpp:508-514): the gradient of output (v, j) lands on the
// grouped position whose edge attained the extremum (aggregate.hpp:295-308,
// argpos scatter), then gather_rows' adjoint adds every grouped position's
// row into dx[src] in ascending grouped (CSC) position (tensor.hpp:510-524).
//
// Gather form, no atomics: per source s, its entries in ascending CSC
// position — the "source view" (rowptr by source, col = destination v,
// perm = COO edge id), i.e. the CSR by source ordered by (v, COO position)
// instead of COO position — and
//   dx[s][j] = sum_t (arg[v_t][j] == eid_t) ? g[v_t][j] : 0     in t order.
// Positions that did not win contribute exact zeros in the reference, which
// never change a sum started at +0 under round-to-nearest, so skipping them is
// bit-identical. Each output element is accumulated by one lane, sequentially.
//
// Traffic per edge: the argmax slice of the destination row (4 B per column),
// the gradient only where a column matches (sparse), plus col/eid.
#include <algorithm>
#include <cmath>

#include "vec.cuh"

namespace gm {
namespace mb {

constexpr int kU = 8;  // entries in flight per batch

template <typename S, int V>
struct Lane {  // V consecutive columns of one row
  using IV = typename std::conditional<V == 4, int4, typename std::conditional<V == 2, int2, int>::type>::type;
  using SV = typename std::conditional<
      V == 1, S, typename std::conditional<sizeof(S) == 4, typename std::conditional<V == 4, float4, float2>::type,
                                           double2>::type>::type;
};

template <typename T, int V>
__device__ __forceinline__ void unpack(const T& r, int32_t* out);
template <>
__device__ __forceinline__ void unpack<int4, 4>(const int4& r, int32_t* o) { o[0] = r.x; o[1] = r.y; o[2] = r.z; o[3] = r.w; }
template <>
__device__ __forceinline__ void unpack<int2, 2>(const int2& r, int32_t* o) { o[0] = r.x; o[1] = r.y; }
template <>
__device__ __forceinline__ void unpack<int, 1>(const int& r, int32_t* o) { o[0] = r; }

template <typename S, int V, typename SV>
__device__ __forceinline__ void unpack_s(const SV& r, S* o) {
  if constexpr (V == 1) {
    o[0] = r;
  } else if constexpr (V == 2) {
    o[0] = r.x;
    o[1] = r.y;
  } else {
    o[0] = r.x;
    o[1] = r.y;
    o[2] = r.z;
    o[3] = r.w;
  }
}

// Light rows: one warp per heavy-free window of consecutive source rows; lane
// l owns columns [(base + l) * V, +V) of every row, in passes of 32 lanes.
template <typename S, int V>
__global__ void __launch_bounds__(256) maxbwd_light_kernel(const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const int32_t* __restrict__ eid,
                                                           const int32_t* __restrict__ windows, int64_t num_windows,
                                                           const int32_t* __restrict__ arg, const S* __restrict__ g,
                                                           int64_t f, S* __restrict__ dx) {
  using IV = typename Lane<S, V>::IV;
  using SV = typename Lane<S, V>::SV;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_windows) return;
  const int r0 = windows[2 * w], r1 = windows[2 * w + 1];
  const int64_t nslot = f / V;
  for (int64_t base = 0; base < nslot; base += 32) {
    const int64_t slot = base + lane;
    const bool valid = slot < nslot;
    const int64_t c0 = slot * V;
    for (int r = r0; r < r1; ++r) {
      const int64_t kb = rowptr[r], ke = rowptr[r + 1];
      S acc[V];
#pragma unroll
      for (int x = 0; x < V; ++x) acc[x] = S(0);
      for (int64_t k0 = kb; k0 < ke; k0 += kU) {
        int32_t mv = 0, me = -2;
        if (lane < kU && k0 + lane < ke) {
          mv = col[k0 + lane];
          me = eid[k0 + lane];
        }
        const int nb = static_cast<int>(ke - k0 < kU ? ke - k0 : kU);
        IV a[kU];
        int32_t ev[kU];
        int32_t vv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          vv[u] = __shfl_sync(FULL, mv, u);
          ev[u] = __shfl_sync(FULL, me, u);
          if (valid && u < nb) a[u] = __ldg(reinterpret_cast<const IV*>(arg + static_cast<int64_t>(vv[u]) * f + c0));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (valid && u < nb) {
            int32_t ai[V];
            unpack<IV, V>(a[u], ai);
            bool any = false;
#pragma unroll
            for (int x = 0; x < V; ++x) any |= ai[x] == ev[u];
            if (any) {
              S gv[V];
              unpack_s<S, V, SV>(__ldg(reinterpret_cast<const SV*>(g + static_cast<int64_t>(vv[u]) * f + c0)), gv);
#pragma unroll
              for (int x = 0; x < V; ++x)
                if (ai[x] == ev[u]) acc[x] = add_rn(acc[x], gv[x]);
            }
          }
        }
      }
      if (valid) {
        S* o = dx + static_cast<int64_t>(r) * f + c0;
        if constexpr (V == 1) {
          o[0] = acc[0];
        } else {
          SV ov;
          if constexpr (V == 2) ov = SV{acc[0], acc[1]};
          else ov = SV{acc[0], acc[1], acc[2], acc[3]};
          *reinterpret_cast<SV*>(o) = ov;
        }
      }
    }
  }
}

// fp32 rows of 16-byte multiples (the hot case): the forward flat sweep's
// schedule over the source view. One warp streams a heavy-free window of
// consecutive source rows as one contiguous entry range, U entries per batch
// regardless of row boundaries; (destination, edge id) pairs are prefetched
// two batches ahead, one per lane, and broadcast by shuffle. Software
// pipeline: while batch b's gradient slices (16 bytes per lane, loaded only
// where an argmax matches) are in flight, batch b+1's argmax slices already
// are too; then b's contributions are added in entry order, so each output
// element is still one lane's sequential sum. Lanes past the row's last slot
// re-read it and never store.
// (same-box C4 A/B, whole backward: 4 entries / 4 CTAs per SM 12.3 ms, 6 / 3
// 17.4, 8 / 2 15.7; the unpipelined two-phase form 12.2 at 6 / 3 with spills,
// the previous warp-per-row gather 24.9 + 4.4 ms for hubs)
#ifndef GM_MAXBWD_MINB
#define GM_MAXBWD_MINB 4
#endif
#ifndef GM_MAXBWD_U
#define GM_MAXBWD_U 4
#endif
// staged variant (default): entries per batch and warps per CTA. Same-box C4
// A/B (whole backward, ms): U/W 8/8 14.4, 4/16 10.4, 2/16 8.9, 2/8 8.2, 2/4
// 7.8, 2/2 7.6, 3/2 7.6; the register-pipelined sweep 12.1.
#ifndef GM_MAXBWD_SU
#define GM_MAXBWD_SU 3
#endif
#ifndef GM_MAXBWD_SW
#define GM_MAXBWD_SW 2
#endif
template <int U>
__global__ void __launch_bounds__(256, GM_MAXBWD_MINB) maxbwd_flat_kernel(const int64_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ col,
                                                          const int32_t* __restrict__ eid,
                                                          const int32_t* __restrict__ windows, int64_t num_windows,
                                                          const int32_t* __restrict__ arg, const float* __restrict__ g,
                                                          int64_t f, float* __restrict__ dx) {
  static_assert(4 * U <= 32, "4 match bits per entry in one word");
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_windows) return;
  const int ra = windows[2 * w], rb = windows[2 * w + 1];
  const int32_t kbeg = static_cast<int32_t>(rowptr[ra]);
  const int32_t kend = static_cast<int32_t>(rowptr[rb]);
  const uint32_t fu = static_cast<uint32_t>(f);
  const int nsl_all = static_cast<int>(f / 4);
  for (int sb = 0; sb < nsl_all; sb += 32) {  // column passes of 32 16-byte slots
    const int nsl = min(32, nsl_all - sb);
    const bool valid = lane < nsl;
    const uint32_t soff = static_cast<uint32_t>(sb + min(lane, nsl - 1)) * 4u;
    int cbase = ra;
    int32_t rend_l = (cbase + lane < rb) ? static_cast<int32_t>(rowptr[cbase + 1 + lane]) : kend;
    int row = ra;
    int32_t row_end = __shfl_sync(FULL, rend_l, 0);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    auto flush = [&]() {
      if (valid)
        __stcs(reinterpret_cast<float4*>(dx + static_cast<uint64_t>(static_cast<uint32_t>(row)) * fu + soff),
               make_float4(acc[0], acc[1], acc[2], acc[3]));
      acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
      ++row;
      if (row < rb) {
        if (row - cbase >= 32) {
          cbase = row;
          rend_l = (cbase + lane < rb) ? static_cast<int32_t>(rowptr[cbase + 1 + lane]) : kend;
        }
        row_end = __shfl_sync(FULL, rend_l, row - cbase);
      }
    };
    // (evict_last for the plan's hot destinations measured 12.3 -> 13.3 ms on C4)
    auto fetch = [&](int32_t kb, int32_t& c, int32_t& e) {
      if (lane < U) {
        const int32_t k = min(kb + lane, kend - 1);
        c = col[k];
        e = eid[k];
      }
    };
    int4 av[U];
#define GM_MB_LOAD_ARG(cbatch)                                                                         \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {                                                     \
    const uint32_t v = static_cast<uint32_t>(__shfl_sync(FULL, (cbatch), u));                          \
    av[u] = __ldcs(reinterpret_cast<const int4*>(arg + static_cast<uint64_t>(v) * fu + soff));       \
  }
    if (kend > kbeg) {
      int32_t c0 = 0, e0 = -2, c1 = 0, e1 = -2;
      fetch(kbeg, c0, e0);
      if (kbeg + U < kend) fetch(kbeg + U, c1, e1);
      GM_MB_LOAD_ARG(c0)
      for (int32_t k0 = kbeg; k0 < kend; k0 += U) {
        const int nb = min(U, kend - k0);
        uint32_t mask = 0;  // 4 match bits per entry
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t eu = __shfl_sync(FULL, e0, u);
          const uint32_t m = static_cast<uint32_t>(av[u].x == eu) | (static_cast<uint32_t>(av[u].y == eu) << 1) |
                             (static_cast<uint32_t>(av[u].z == eu) << 2) |
                             (static_cast<uint32_t>(av[u].w == eu) << 3);
          mask |= (u < nb ? m : 0u) << (4 * u);
        }
        const int32_t cb = c0;
        c0 = c1;
        e0 = e1;
        if (k0 + 2 * U < kend) fetch(k0 + 2 * U, c1, e1);
        if (k0 + U < kend) {  // next batch's argmax slices, in flight with this batch's gradients
          GM_MB_LOAD_ARG(c0)
        }
        float4 gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t v = static_cast<uint32_t>(__shfl_sync(FULL, cb, u));
          if ((mask >> (4 * u)) & 15u)
            gv[u] = __ldg(reinterpret_cast<const float4*>(g + static_cast<uint64_t>(v) * fu + soff));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u < nb) {
            while (k0 + u >= row_end) flush();
            const uint32_t m = (mask >> (4 * u)) & 15u;
            if (m) {
              if (m & 1u) acc[0] = __fadd_rn(acc[0], gv[u].x);
              if (m & 2u) acc[1] = __fadd_rn(acc[1], gv[u].y);
              if (m & 4u) acc[2] = __fadd_rn(acc[2], gv[u].z);
              if (m & 8u) acc[3] = __fadd_rn(acc[3], gv[u].w);
            }
          }
        }
      }
    }
    while (row < rb) flush();
  }
#undef GM_MB_LOAD_ARG
}

// Staged variant (the default; GM_MAXBWD_STAGED=0 selects the register sweep
// above): the same window sweep, but the argmax
// and gradient slices go through a per-warp shared-memory ring with 16-byte
#ifndef GM_MAXBWD_ZFILL
#define GM_MAXBWD_ZFILL 1  // 0: skip the copy of non-matching slices (A/B: 7.94 vs 7.83 ms, the same 44.5 GB of DRAM)
#endif
// cp.async instead of registers, so kStageD batches of U entries are in
// flight per warp without register pressure. Per iteration: issue the argmax
// slices of batch i+2; when batch i+1's have landed, form its match masks and
// issue its gradient slices (zero-filled where no column of the slice
// matches); when batch i's gradients have landed, add them in entry order.
constexpr int kStageD = 3;
template <int U, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 1) maxbwd_staged_kernel(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, const int32_t* __restrict__ eid,
    const int32_t* __restrict__ windows, int64_t num_windows, const int32_t* __restrict__ arg,
    const float* __restrict__ g, int64_t f, float* __restrict__ dx) {
  static_assert(4 * U <= 32, "4 match bits per entry in one word");
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char mb_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // per warp: kStageD stages of {arg[U][32] int4, grad[U][32] float4}
  int4* sarg = reinterpret_cast<int4*>(mb_smem) + static_cast<size_t>(wib) * kStageD * 2 * U * 32;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * WARPS + wib;
  if (w >= num_windows) return;
  const int ra = windows[2 * w], rb = windows[2 * w + 1];
  const int32_t kbeg = static_cast<int32_t>(rowptr[ra]);
  const int32_t kend = static_cast<int32_t>(rowptr[rb]);
  const uint32_t fu = static_cast<uint32_t>(f);
  const int nsl_all = static_cast<int>(f / 4);
  auto st_arg = [&](int b) { return sarg + static_cast<size_t>(b % kStageD) * 2 * U * 32; };
  auto st_grad = [&](int b) { return reinterpret_cast<float4*>(st_arg(b) + U * 32); };
  for (int sb = 0; sb < nsl_all; sb += 32) {  // column passes of 32 16-byte slots
    const int nsl = min(32, nsl_all - sb);
    const bool valid = lane < nsl;
    const uint32_t soff = static_cast<uint32_t>(sb + min(lane, nsl - 1)) * 4u;
    int cbase = ra;
    int32_t rend_l = (cbase + lane < rb) ? static_cast<int32_t>(rowptr[cbase + 1 + lane]) : kend;
    int row = ra;
    int32_t row_end = __shfl_sync(FULL, rend_l, 0);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    auto flush = [&]() {
      if (valid)
        __stcs(reinterpret_cast<float4*>(dx + static_cast<uint64_t>(static_cast<uint32_t>(row)) * fu + soff),
               make_float4(acc[0], acc[1], acc[2], acc[3]));
      acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
      ++row;
      if (row < rb) {
        if (row - cbase >= 32) {
          cbase = row;
          rend_l = (cbase + lane < rb) ? static_cast<int32_t>(rowptr[cbase + 1 + lane]) : kend;
        }
        row_end = __shfl_sync(FULL, rend_l, row - cbase);
      }
    };
    const int nb = (kend - kbeg + U - 1) / U;  // batches of this window
    // per-lane metadata of a batch: lane u < U holds entry u's (destination, edge id)
    auto meta = [&](int b, int32_t& c, int32_t& e) {
      c = 0;
      e = -2;
      if (lane < U && b < nb) {
        const int32_t k = min(kbeg + b * U + lane, kend - 1);
        c = col[k];
        e = (kbeg + b * U + lane < kend) ? eid[k] : -2;
      }
    };
    // plain 16-byte cp.async (an evict_last hint for the plan's hot
    // destinations measured 7.6 -> 8.1 ms, evict_first for the rest slower still)
    auto cp16 = [&](uint32_t sa, const void* src, uint32_t nbytes) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "r"(nbytes) : "memory");
    };
    auto issue_arg = [&](int b, int32_t c) {
      if (b < nb) {
        int4* dst = st_arg(b);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t v = static_cast<uint32_t>(__shfl_sync(FULL, c, u));
          const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst + u * 32 + lane));
          cp16(sa, arg + static_cast<uint64_t>(v) * fu + soff, 16u);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // match masks of batch b (its argmax slices in smem) and its gradient issue
    auto masks_and_grad = [&](int b, int32_t c, int32_t e) -> uint32_t {
      uint32_t mask = 0;
      if (b < nb) {
        const int4* sa = st_arg(b);
        float4* dst = st_grad(b);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t eu = __shfl_sync(FULL, e, u);
          const uint32_t v = static_cast<uint32_t>(__shfl_sync(FULL, c, u));
          const int4 a4 = sa[u * 32 + lane];
          const uint32_t m = static_cast<uint32_t>(a4.x == eu) | (static_cast<uint32_t>(a4.y == eu) << 1) |
                             (static_cast<uint32_t>(a4.z == eu) << 2) | (static_cast<uint32_t>(a4.w == eu) << 3);
          mask |= m << (4 * u);
          const uint32_t gd = static_cast<uint32_t>(__cvta_generic_to_shared(dst + u * 32 + lane));
#if GM_MAXBWD_ZFILL
          // zero-fill where no column of the slice matches
          cp16(gd, g + static_cast<uint64_t>(v) * fu + soff, m ? 16u : 0u);
#else
          // no copy at all where no column of the slice matches (the consumer
          // reads a slice only under its match mask)
          if (m) cp16(gd, g + static_cast<uint64_t>(v) * fu + soff, 16u);
#endif
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return mask;
    };
    int32_t c0, e0, c1, e1, c2, e2;
    meta(0, c0, e0);
    meta(1, c1, e1);
    issue_arg(0, c0);                 // A0
    issue_arg(1, c1);                 // A1
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // A0 landed
    __syncwarp();
    uint32_t mask_cur = masks_and_grad(0, c0, e0);  // G0
    for (int b = 0; b < nb; ++b) {
      meta(b + 2, c2, e2);
      issue_arg(b + 2, c2);                                 // A(b+2)
      asm volatile("cp.async.wait_group 2;" ::: "memory");  // A(b+1) landed (G(b), A(b+2) may fly)
      __syncwarp();
      const uint32_t mask_next = masks_and_grad(b + 1, c1, e1);  // G(b+1)
      asm volatile("cp.async.wait_group 2;" ::: "memory");  // G(b) landed
      __syncwarp();
      const float4* sg = st_grad(b);
      const int32_t k0 = kbeg + b * U;
      const int n_e = min(U, kend - k0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < n_e) {
          while (k0 + u >= row_end) flush();
          const uint32_t m = (mask_cur >> (4 * u)) & 15u;
          if (m) {
            const float4 gv = sg[u * 32 + lane];
            if (m & 1u) acc[0] = __fadd_rn(acc[0], gv.x);
            if (m & 2u) acc[1] = __fadd_rn(acc[1], gv.y);
            if (m & 4u) acc[2] = __fadd_rn(acc[2], gv.z);
            if (m & 8u) acc[3] = __fadd_rn(acc[3], gv.w);
          }
        }
      }
      __syncwarp();  // stage b is reused by A(b+3)
      mask_cur = mask_next;
      c1 = c2;
      e1 = e2;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    while (row < rb) flush();
  }
}

// Hub rows (out-degree > the plan's threshold, up to ~20K entries on C4): one
// CTA per (hub row, 32-column chunk). Per round its 16 (fp64: 8) warps fetch 16
// consecutive entries each (lane = column): all argmax loads, then the
// matching gradient loads, then each entry's contribution — the gradient or
// an exact +0 — goes to a [256 (128) entries x 32 columns] shared tile. Warp 0 then
// adds the tile's rows in entry order. Adding +0 never changes a sum that
// started at +0 (it cannot become -0), so the tile's zeros are exact and each
// column is one lane's sequential sum in the reference's order, while the
// loads of 256 entries are in flight at once instead of one warp's batch.
template <typename S>
constexpr int hub_warps() { return sizeof(S) == 8 ? 8 : 16; }  // tile <= 48 KB static
constexpr int kHubPer = 16;                                     // entries per warp per round
template <typename S>
__global__ void __launch_bounds__(hub_warps<S>() * 32, 2) maxbwd_hub_tile_kernel(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, const int32_t* __restrict__ eid,
    const int32_t* __restrict__ heavy, int64_t num_heavy, const int32_t* __restrict__ arg, const S* __restrict__ g,
    int64_t f, S* __restrict__ dx) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int kHubRound = hub_warps<S>() * kHubPer;
  __shared__ S tile[kHubRound][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t chunks = (f + 31) / 32;
  const int r = heavy[blockIdx.x / chunks];
  const int64_t cc = (blockIdx.x % chunks) * 32 + lane;
  const bool valid = cc < f;
  const int64_t c = valid ? cc : f - 1;  // lanes past f re-read the last column, never store
  const int64_t kb = rowptr[r], ke = rowptr[r + 1];
  S acc = S(0);
  for (int64_t base = kb; base < ke; base += kHubRound) {
    const int64_t m0 = base + w * kHubPer;
    const bool has = lane < kHubPer && m0 + lane < ke;
    const int32_t mv = has ? col[m0 + lane] : 0;
    const int32_t me = has ? eid[m0 + lane] : -2;
    int32_t a[kHubPer];
#pragma unroll
    for (int u = 0; u < kHubPer; ++u) {
      const int32_t vv = __shfl_sync(FULL, mv, u);
      a[u] = m0 + u < ke ? __ldg(arg + static_cast<int64_t>(vv) * f + c) : -3;
    }
    uint32_t hit = 0;
#pragma unroll
    for (int u = 0; u < kHubPer; ++u) hit |= static_cast<uint32_t>(a[u] == __shfl_sync(FULL, me, u)) << u;
    S gv[kHubPer];
#pragma unroll
    for (int u = 0; u < kHubPer; ++u) {
      const int32_t vv = __shfl_sync(FULL, mv, u);
      gv[u] = ((hit >> u) & 1u) ? __ldg(g + static_cast<int64_t>(vv) * f + c) : S(0);
    }
#pragma unroll
    for (int u = 0; u < kHubPer; ++u) tile[w * kHubPer + u][lane] = gv[u];
    __syncthreads();
    if (w == 0) {
      const int n = static_cast<int>(ke - base < kHubRound ? ke - base : kHubRound);
#pragma unroll 8
      for (int i = 0; i < n; ++i) acc = add_rn(acc, tile[i][lane]);
    }
    __syncthreads();
  }
  if (w == 0 && valid) dx[static_cast<int64_t>(r) * f + c] = acc;
}

__global__ void widen_kernel(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void entry_rows64_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int64_t* __restrict__ out) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) out[k - rowptr[0]] = r;
}

__global__ void gather_ids_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ idx, int64_t n,
                                  int32_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = ids[idx[i]];
}

inline unsigned grid_of(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kNumSMs * 32)));
}

struct SourceViewWs {
  int64_t* keys;
  int64_t* vals;
  int32_t* pos;
  unsigned char* build;
  size_t build_bytes;
  size_t bytes;
};

inline SourceViewWs source_view_layout(void* base, int64_t nnz, int64_t n_src) {
  SourceViewWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + off : nullptr;
    off += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  w.keys = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(nnz)));
  w.vals = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(nnz)));
  w.pos = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(nnz)));
  w.build_bytes = gm_build_compressed_workspace(nnz, n_src);
  w.build = take(w.build_bytes);
  w.bytes = off;
  return w;
}

template <typename S>
gm_status launch_bwd(const gm_csr* v, const gm_spmm_plan* plan, const int32_t* arg, const S* g, int64_t f, S* dx,
                     cudaStream_t st) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dx) |
                       reinterpret_cast<uintptr_t>(arg);
  const unsigned lgrid = static_cast<unsigned>(ceil_div(std::max<int64_t>(plan->num_light_windows, 1) * 32, 256));
  if (plan->num_light_windows > 0) {
    bool done = false;
    if constexpr (sizeof(S) == 4) {
      if (f % 4 == 0 && al % 16 == 0) {
        // staged ring (default) vs the register-pipelined sweep (GM_MAXBWD_STAGED=0)
        static const bool staged = [] { const char* ev = getenv("GM_MAXBWD_STAGED"); return !(ev && ev[0] == '0'); }();
        if (staged) {
          constexpr int kU = GM_MAXBWD_SU, kW = GM_MAXBWD_SW;
          const size_t smem = sizeof(int4) * kStageD * 2 * kU * 32 * kW;
          GM_TRY_CUDA(cudaFuncSetAttribute(maxbwd_staged_kernel<kU, kW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
          maxbwd_staged_kernel<kU, kW><<<static_cast<unsigned>(ceil_div(plan->num_light_windows, kW)), 32 * kW, smem,
                                         st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                               plan->num_light_windows, arg, g, f, dx);
        } else {
          maxbwd_flat_kernel<GM_MAXBWD_U><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                                 plan->num_light_windows, arg, g, f, dx);
        }
        done = true;
      }
    }
    if (done) {
    } else if (f % 2 == 0 && al % (2 * sizeof(S)) == 0 && al % 8 == 0)
      maxbwd_light_kernel<S, 2><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                       plan->num_light_windows, arg, g, f, dx);
    else
      maxbwd_light_kernel<S, 1><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                       plan->num_light_windows, arg, g, f, dx);
    GM_CHECK_LAUNCH("maxbwd_light_kernel");
  }
  if (plan->num_heavy > 0) {
    const int64_t warps = plan->num_heavy * ceil_div(f, 32);
    maxbwd_hub_tile_kernel<S><<<static_cast<unsigned>(warps), hub_warps<S>() * 32, 0, st>>>(
        v->rowptr, v->col, v->perm, plan->heavy_rows, plan->num_heavy, arg, g, f, dx);
    GM_CHECK_LAUNCH("maxbwd_hub_tile_kernel");
  }
  return GM_OK;
}

}  // namespace mb
}  // namespace gm

using namespace gm;

extern "C" {

GM_API size_t gm_source_view_workspace(int64_t nnz, int64_t n_src) {
  if (nnz < 0 || n_src < 0) return 0;
  return mb::source_view_layout(nullptr, nnz, n_src).bytes;
}

GM_API gm_status gm_source_view(const gm_csr* csc, int64_t n_src, int64_t* rowptr, int32_t* col, int32_t* eid,
                                void* workspace, size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(csc && rowptr, GM_ERR_INVALID_ARGUMENT, "gm_source_view: null argument");
  GM_REQUIRE(csc->nnz >= 0 && n_src >= 0 && csc->num_rows >= 0, GM_ERR_INVALID_ARGUMENT,
             "gm_source_view: negative size");
  GM_REQUIRE(csc->nnz == 0 || csc->perm, GM_ERR_INVALID_ARGUMENT, "gm_source_view: csc->perm required");
  const mb::SourceViewWs need = mb::source_view_layout(nullptr, csc->nnz, n_src);
  GM_REQUIRE(workspace && workspace_bytes >= need.bytes, GM_ERR_INVALID_ARGUMENT,
             "gm_source_view: workspace too small");
  cudaStream_t st = as_stream(stream);
  const mb::SourceViewWs w = mb::source_view_layout(workspace, csc->nnz, n_src);
  const int64_t nnz = csc->nnz;
  if (nnz > 0) {
    // keys = the CSC's source ids, values = its destination rows, in CSC order
    int64_t k0 = 0;
    GM_TRY_CUDA(cudaMemcpyAsync(&k0, csc->rowptr, sizeof(k0), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    mb::widen_kernel<<<mb::grid_of(nnz), 256, 0, st>>>(csc->col + k0, nnz, w.keys);
    GM_CHECK_LAUNCH("widen_kernel");
    mb::entry_rows64_kernel<<<mb::grid_of(csc->num_rows), 256, 0, st>>>(csc->rowptr, csc->num_rows, w.vals);
    GM_CHECK_LAUNCH("entry_rows64_kernel");
  }
  // stable counting sort by source: per source, ascending CSC position
  gm_status s = gm_build_compressed(w.keys, w.vals, nnz, n_src, rowptr, col, w.pos, w.build, w.build_bytes, stream);
  if (s != GM_OK) return s;
  if (nnz > 0) {
    int64_t k0 = 0;
    GM_TRY_CUDA(cudaMemcpyAsync(&k0, csc->rowptr, sizeof(k0), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    mb::gather_ids_kernel<<<mb::grid_of(nnz), 256, 0, st>>>(csc->perm + k0, w.pos, nnz, eid);
    GM_CHECK_LAUNCH("gather_ids_kernel");
  }
  return GM_OK;
}

GM_API gm_status gm_spmm_max_backward(const gm_csr* source_view, const gm_spmm_plan* plan, gm_dtype dtype,
                                      const int32_t* arg, const void* g, int64_t f, void* dx, gm_stream_t stream) {
  GM_REQUIRE(source_view && plan, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: null view/plan");
  GM_REQUIRE(f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: negative feature width");
  GM_REQUIRE(dtype == GM_F32 || dtype == GM_F64, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: f32/f64 only");
  if (source_view->num_rows == 0 || f == 0) return GM_OK;
  GM_REQUIRE(arg && g && dx, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: null pointer");
  GM_REQUIRE(source_view->nnz == 0 || source_view->perm, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_max_backward: the source view needs edge ids (perm)");
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F32)
    return mb::launch_bwd<float>(source_view, plan, arg, static_cast<const float*>(g), f, static_cast<float*>(dx), st);
  return mb::launch_bwd<double>(source_view, plan, arg, static_cast<const double*>(g), f, static_cast<double*>(dx), st);
}

}  // extern "C"
