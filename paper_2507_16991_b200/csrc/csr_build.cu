// csr_build.cu — graph-structure kernels (L1): bounds/claims checks, degree
// counts and the bit-exact stable CSR/CSC build.
//
// build_compressed (edge_index.cpp:45-62) is a stable counting sort: within a
// row, entries appear in ascending COO position. On the GPU:
//   1. count   : cnt[key]++ (int32 atomics; exact)
//   2. scan    : rowptr = exclusive prefix sum (int64), block-partial scan
//   3. scatter : perm[rowptr[key+1] - atomicSub(&cnt[key], 1)] = i (unstable)
//   4. restore stability by sorting every row's perm segment ascending (the
//      values are distinct COO positions, so ascending order IS the stable
//      order) — warp bitonic for rows <= 32, CTA bitonic in shared memory for
//      rows <= 4096, chunk-sort + exact rank merge for longer (hub) rows —
//      and emit col[k] = values[perm[k]] in the same pass.
// The result is identical to the reference for every input, independent of
// atomic ordering.
#include <algorithm>
#include <climits>
#include <string>

#include "gm_common.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace gm {

// ---------------------------------------------------------------------------
// checks and degrees
// ---------------------------------------------------------------------------
__global__ void bounds_kernel(const int64_t* __restrict__ ids, int64_t len, int64_t bound,
                              unsigned long long* __restrict__ first_bad) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = ids[i];
    if (v < 0 || v >= bound) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
}

__global__ void unsorted_kernel(const int64_t* __restrict__ keys, int64_t len,
                                unsigned long long* __restrict__ first_bad) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (keys[i] < keys[i - 1]) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
}

__global__ void degree_kernel(const int64_t* __restrict__ ids, int64_t len, int64_t n,
                              int32_t* __restrict__ deg) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = ids[i];
    if (v >= 0 && v < n) atomicAdd(&deg[v], 1);
  }
}

__global__ void gcn_finish_kernel(int32_t* __restrict__ deg, int64_t n, int add, int clamp1) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t d = deg[i] + add;
  if (clamp1 && d < 1) d = 1;
  deg[i] = d;
}

static unsigned grid_for(int64_t n, int threads = 256) {
  const int64_t b = ceil_div(std::max<int64_t>(n, 1), threads);
  return static_cast<unsigned>(std::min<int64_t>(b, kNumSMs * 32));
}

// ---------------------------------------------------------------------------
// exclusive scan of int32 counts into int64 rowptr (3 phases)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* warp_tot, int64_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
    int64_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t n = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += n;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  return inc - v + warp_tot[wid];
}

__global__ void scan_reduce_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                   int64_t* __restrict__ partial) {
  __shared__ int64_t wt[kScanThreads / 32];
  __shared__ int64_t tot;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    if (idx < n) s += cnt[idx];
  }
  block_exclusive_scan(s, wt, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void scan_partials_kernel(int64_t* __restrict__ partial, int64_t nb) {
  __shared__ int64_t wt[kScanThreads / 32];
  __shared__ int64_t tot;
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t idx = base + threadIdx.x;
    const int64_t v = idx < nb ? partial[idx] : 0;
    const int64_t ex = block_exclusive_scan(v, wt, &tot);
    if (idx < nb) partial[idx] = carry + ex;
    __syncthreads();
    carry += tot;
    __syncthreads();
  }
}

__global__ void scan_down_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                 const int64_t* __restrict__ partial, int64_t* __restrict__ rowptr) {
  __shared__ int64_t wt[kScanThreads / 32];
  __shared__ int64_t tot;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    v[i] = idx < n ? cnt[idx] : 0;
    s += v[i];
  }
  int64_t run = block_exclusive_scan(s, wt, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    if (idx < n) rowptr[idx] = run;
    run += v[i];
    if (idx == n - 1) rowptr[n] = run;
  }
}

// ---------------------------------------------------------------------------
// scatter + per-row stabilisation
// ---------------------------------------------------------------------------
__global__ void count_kernel(const int64_t* __restrict__ keys, int64_t e, int32_t* __restrict__ cnt) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[keys[i]], 1);
}

__global__ void scatter_kernel(const int64_t* __restrict__ keys, int64_t e,
                               const int64_t* __restrict__ rowptr, int32_t* __restrict__ cnt,
                               int32_t* __restrict__ perm) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = keys[i];
    const int32_t c = atomicSub(&cnt[k], 1);
    perm[rowptr[k + 1] - c] = static_cast<int32_t>(i);
  }
}

constexpr int kMedMax = 4096;  // rows up to this length are sorted in one CTA's smem
constexpr int kSortThreads = 512;

// Warp per row: rows of length <= 32 are sorted in registers (bitonic via
// shuffles); longer rows are queued for the CTA kernels.
__global__ void sort_small_kernel(const int64_t* __restrict__ rowptr, int64_t num_rows,
                                  const int64_t* __restrict__ values, int32_t* __restrict__ perm,
                                  int32_t* __restrict__ col, int32_t* __restrict__ med_list,
                                  int32_t* __restrict__ big_list, unsigned int* __restrict__ counters) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < num_rows; r += nwarps) {
    const int64_t kb = rowptr[r];
    const int64_t len = rowptr[r + 1] - kb;
    if (len <= 32) {
      if (len == 0) continue;
      int32_t v = lane < len ? perm[kb + lane] : INT_MAX;
      if (len > 1) {
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
          for (int j = k >> 1; j > 0; j >>= 1) {
            const int32_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            v = (lower == up) ? min(v, o) : max(v, o);
          }
        }
      }
      if (lane < len) {
        perm[kb + lane] = v;
        col[kb + lane] = static_cast<int32_t>(values[v]);
      }
    } else if (lane == 0) {
      if (len <= kMedMax) med_list[atomicAdd(&counters[0], 1u)] = static_cast<int32_t>(r);
      else big_list[atomicAdd(&counters[1], 1u)] = static_cast<int32_t>(r);
    }
  }
}

// In-smem bitonic sort of `n` (power of two) int32 keys by kSortThreads threads.
__device__ void smem_bitonic(int32_t* s, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const int32_t a = s[i], b = s[ixj];
          if ((a > b) == up) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSortThreads)
sort_med_kernel(const int64_t* __restrict__ rowptr, const int64_t* __restrict__ values,
                int32_t* __restrict__ perm, int32_t* __restrict__ col,
                const int32_t* __restrict__ list, const unsigned int* __restrict__ counters) {
  __shared__ int32_t s[kMedMax];
  const unsigned int n_rows = counters[0];
  for (unsigned int li = blockIdx.x; li < n_rows; li += gridDim.x) {
    const int64_t r = list[li];
    const int64_t kb = rowptr[r];
    const int len = static_cast<int>(rowptr[r + 1] - kb);
    int p2 = 64;
    while (p2 < len) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) s[i] = i < len ? perm[kb + i] : INT_MAX;
    __syncthreads();
    smem_bitonic(s, p2);
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const int32_t v = s[i];
      perm[kb + i] = v;
      col[kb + i] = static_cast<int32_t>(values[v]);
    }
    __syncthreads();
  }
}

// Hub rows: sort kMedMax-chunks in place, then place every element at its
// exact rank (values are distinct): rank = sum over chunks of lower_bound.
__global__ void __launch_bounds__(kSortThreads)
sort_big_kernel(const int64_t* __restrict__ rowptr, const int64_t* __restrict__ values,
                int32_t* __restrict__ perm, int32_t* __restrict__ col,
                int32_t* __restrict__ scratch, const int32_t* __restrict__ list,
                const unsigned int* __restrict__ counters) {
  __shared__ int32_t s[kMedMax];
  const unsigned int n_rows = counters[1];
  for (unsigned int li = blockIdx.x; li < n_rows; li += gridDim.x) {
    const int64_t r = list[li];
    const int64_t kb = rowptr[r];
    const int64_t len = rowptr[r + 1] - kb;
    const int64_t nch = (len + kMedMax - 1) / kMedMax;
    for (int64_t c = 0; c < nch; ++c) {
      const int64_t cb = kb + c * kMedMax;
      const int clen = static_cast<int>(std::min<int64_t>(kMedMax, len - c * kMedMax));
      int p2 = 64;
      while (p2 < clen) p2 <<= 1;
      for (int i = threadIdx.x; i < p2; i += blockDim.x) s[i] = i < clen ? perm[cb + i] : INT_MAX;
      __syncthreads();
      smem_bitonic(s, p2);
      for (int i = threadIdx.x; i < clen; i += blockDim.x) perm[cb + i] = s[i];
      __syncthreads();
    }
    __threadfence_block();
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
      const int32_t v = perm[kb + i];
      int64_t rank = 0;
      for (int64_t c = 0; c < nch; ++c) {
        const int64_t cb = kb + c * kMedMax;
        int64_t lo = 0, hi = std::min<int64_t>(kMedMax, len - c * kMedMax);
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (perm[cb + mid] < v) lo = mid + 1;
          else hi = mid;
        }
        rank += lo;
      }
      scratch[kb + rank] = v;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
      const int32_t v = scratch[kb + i];
      perm[kb + i] = v;
      col[kb + i] = static_cast<int32_t>(values[v]);
    }
    __syncthreads();
  }
}

__global__ void permute_kernel_4(const uint32_t* __restrict__ in, const int32_t* __restrict__ perm,
                                 int64_t n, uint32_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[perm[i]];
}
__global__ void permute_kernel_8(const uint64_t* __restrict__ in, const int32_t* __restrict__ perm,
                                 int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[perm[i]];
}
__global__ void permute_kernel_2(const uint16_t* __restrict__ in, const int32_t* __restrict__ perm,
                                 int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[perm[i]];
}

struct BuildWs {
  int32_t* cnt;
  int64_t* partial;
  int32_t* med;
  int32_t* big;
  unsigned int* counters;
  int32_t* scratch;
  size_t bytes;
};

static BuildWs build_layout(void* base, int64_t e, int64_t n) {
  BuildWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + off : nullptr;
    off += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, kScanTile));
  w.cnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(n)));
  w.partial = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(nb)));
  w.med = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(n)));
  w.big = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(n)));
  w.counters = reinterpret_cast<unsigned int*>(take(64));
  w.scratch = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(e)));
  w.bytes = off;
  return w;
}

}  // namespace gm
#include "csr_bucket.cuh"
#include "csr_radix.cuh"
namespace gm {

// GM_CSR_ALGO (A/B comparison only): radix (default) | bucket | sort
// (scatter + per-row sort).
static int csr_algo() {
  static const int a = [] {
    const char* v = getenv("GM_CSR_ALGO");
    if (!v) return 0;
    const std::string s(v);
    return s == "bucket" ? 1 : s == "sort" ? 2 : 0;
  }();
  return a;
}
static bool use_bucket_build(int64_t e, int64_t rows) { return csr_algo() == 1 && cb::bucket_path_ok(e, rows); }
static bool use_radix_build(int64_t e, int64_t rows) { return csr_algo() == 0 && e > 0 && rows > 0; }

// ---------------------------------------------------------------------------
// Stable split of a CSR's entries into source blocks (multi-GPU overlap):
// entry k of row r goes to block src_block[col[k]] with column src_col[col[k]];
// inside every (block, row) the entries keep their compressed order.
// ---------------------------------------------------------------------------
constexpr int kSplitWarps = 8;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(kSplitWarps * 32)
split_count_kernel(const int64_t* __restrict__ rowptr, int64_t rows, const int32_t* __restrict__ col,
                   const int32_t* __restrict__ src_block, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kSplitWarps;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const int64_t kb = rowptr[r], ke = rowptr[r + 1];
    for (int64_t k0 = kb; k0 < ke; k0 += 32) {
      const int64_t k = k0 + lane;
      const int b = k < ke ? src_block[col[k]] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      if (b >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(&cnt[static_cast<int64_t>(b) * rows + r], __popc(peers));
    }
  }
}

__global__ void __launch_bounds__(kSplitWarps * 32)
split_scatter_kernel(const int64_t* __restrict__ rowptr, int64_t rows, const int32_t* __restrict__ col,
                     const int32_t* __restrict__ perm, const int32_t* __restrict__ src_block,
                     const int32_t* __restrict__ src_col, int32_t nb, const int64_t* __restrict__ off,
                     int32_t* __restrict__ col_out, int32_t* __restrict__ perm_out) {
  extern __shared__ int32_t cursors[];
  const int lane = threadIdx.x & 31;
  int32_t* cur = cursors + (threadIdx.x >> 5) * nb;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kSplitWarps;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    for (int i = lane; i < nb; i += 32) cur[i] = 0;
    __syncwarp();
    const int64_t kb = rowptr[r], ke = rowptr[r + 1];
    for (int64_t k0 = kb; k0 < ke; k0 += 32) {
      const int64_t k = k0 + lane;
      int32_t c = 0;
      int b = -1;
      if (k < ke) {
        c = col[k];
        b = src_block[c];
      }
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int rank = __popc(peers & lanemask_lt());
      const int base = b >= 0 ? cur[b] : 0;
      __syncwarp();
      if (b >= 0) {
        const int64_t pos = off[static_cast<int64_t>(b) * rows + r] + base + rank;
        col_out[pos] = src_col[c];
        perm_out[pos] = perm[k];
        if (rank == 0) cur[b] = base + __popc(peers);
      }
      __syncwarp();
    }
  }
}

// rowptr_out[b][r] = off[b * rows + r] for r in [0, rows] (the scan's last
// entry closes the last block).
__global__ void split_rowptr_kernel(const int64_t* __restrict__ off, int64_t rows, int64_t nb,
                                    int64_t* __restrict__ rowptr_out) {
  const int64_t n = nb * (rows + 1);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / (rows + 1), r = i - b * (rows + 1);
    rowptr_out[i] = off[b * rows + r];
  }
}

// ---------------------------------------------------------------------------
// Undirected-claim check (edge_index.cpp:98-118): count(u,v) == count(v,u)
// for every COO position; the first position that fails is reported.
// ---------------------------------------------------------------------------
__global__ void pair_keys_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t len,
                                 int64_t n, unsigned long long* __restrict__ keys) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keys[i] = static_cast<unsigned long long>(src[i]) * static_cast<unsigned long long>(n) +
              static_cast<unsigned long long>(dst[i]);
}

__device__ __forceinline__ int64_t key_count(const unsigned long long* __restrict__ sorted, int64_t len,
                                             unsigned long long k) {
  int64_t lo = 0, hi = len;  // lower bound
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  int64_t lo2 = lo, hi2 = len;  // upper bound
  while (lo2 < hi2) {
    const int64_t mid = (lo2 + hi2) >> 1;
    if (sorted[mid] <= k) lo2 = mid + 1;
    else hi2 = mid;
  }
  return lo2 - lo;
}

__global__ void asym_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t len, int64_t n,
                            const unsigned long long* __restrict__ sorted, unsigned long long* __restrict__ first) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long u = static_cast<unsigned long long>(src[i]);
    const unsigned long long v = static_cast<unsigned long long>(dst[i]);
    const unsigned long long nn = static_cast<unsigned long long>(n);
    if (key_count(sorted, len, u * nn + v) != key_count(sorted, len, v * nn + u))
      atomicMin(first, static_cast<unsigned long long>(i));
  }
}

static size_t asym_cub_bytes(int64_t len) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, static_cast<const unsigned long long*>(nullptr),
                                 static_cast<unsigned long long*>(nullptr), static_cast<int>(len));
  return tmp;
}

__global__ void mark_columns_kernel(const int64_t* __restrict__ rowptr, int64_t rows, const int32_t* __restrict__ col,
                                    uint8_t* __restrict__ mark) {
  const int64_t k0 = rowptr[0], k1 = rowptr[rows];
  for (int64_t k = k0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < k1;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mark[col[k]] = 1;
}

template <int B>
__global__ void gather_rows_kernel(const unsigned char* __restrict__ x, int64_t row_bytes, const int32_t* __restrict__ idx,
                                   int64_t n, unsigned char* __restrict__ out) {
  // one warp per output row, B-byte vectors
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const unsigned char* src = x + static_cast<int64_t>(idx[i]) * row_bytes;
    unsigned char* dst = out + i * row_bytes;
    for (int64_t b = static_cast<int64_t>(lane) * B; b < row_bytes; b += 32 * B) {
      if constexpr (B == 16) *reinterpret_cast<uint4*>(dst + b) = __ldg(reinterpret_cast<const uint4*>(src + b));
      else if constexpr (B == 8) *reinterpret_cast<uint2*>(dst + b) = __ldg(reinterpret_cast<const uint2*>(src + b));
      else if constexpr (B == 4) *reinterpret_cast<uint32_t*>(dst + b) = __ldg(reinterpret_cast<const uint32_t*>(src + b));
      else *reinterpret_cast<uint16_t*>(dst + b) = __ldg(reinterpret_cast<const uint16_t*>(src + b));
    }
  }
}

struct SplitWs {
  int32_t* cnt;
  int64_t* partial;
  int64_t* off;
  size_t bytes;
};

static SplitWs split_layout(void* base, int64_t rows, int64_t nb) {
  SplitWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + o : nullptr;
    o += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  const int64_t n = rows * nb;
  w.cnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(n)));
  w.partial = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(std::max<int64_t>(1, ceil_div(n, kScanTile)))));
  w.off = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(n + 1)));
  w.bytes = o;
  return w;
}

}  // namespace gm

using namespace gm;

extern "C" {

GM_API size_t gm_first_asymmetric_workspace(int64_t len) {
  if (len < 0 || len >= INT32_MAX) return 0;
  return 2 * align_up(sizeof(unsigned long long) * static_cast<size_t>(std::max<int64_t>(len, 1)), 256) +
         align_up(asym_cub_bytes(len), 256) + 256;
}

GM_API gm_status gm_first_asymmetric(const int64_t* src, const int64_t* dst, int64_t len, int64_t n,
                                     int64_t* pos_host, void* workspace, size_t workspace_bytes,
                                     gm_stream_t stream) {
  GM_REQUIRE(pos_host, GM_ERR_INVALID_ARGUMENT, "gm_first_asymmetric: null output");
  *pos_host = -1;
  if (len == 0) return GM_OK;
  GM_REQUIRE(len > 0 && len < INT32_MAX, GM_ERR_INVALID_ARGUMENT, "gm_first_asymmetric: length must be in [0, 2^31)");
  GM_REQUIRE(n > 0 && n <= (int64_t(1) << 31), GM_ERR_INVALID_ARGUMENT, "gm_first_asymmetric: n must be in (0, 2^31]");
  GM_REQUIRE(src && dst && workspace && workspace_bytes >= gm_first_asymmetric_workspace(len),
             GM_ERR_INVALID_ARGUMENT, "gm_first_asymmetric: null pointer or workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned char* b = static_cast<unsigned char*>(workspace);
  const size_t kb = align_up(sizeof(unsigned long long) * static_cast<size_t>(len), 256);
  auto* keys = reinterpret_cast<unsigned long long*>(b);
  auto* sorted = reinterpret_cast<unsigned long long*>(b + kb);
  void* tmp = b + 2 * kb;
  size_t tmp_bytes = asym_cub_bytes(len);
  auto* first = reinterpret_cast<unsigned long long*>(b + 2 * kb + align_up(tmp_bytes, 256));
  pair_keys_kernel<<<grid_for(len), 256, 0, st>>>(src, dst, len, n, keys);
  GM_CHECK_LAUNCH("pair_keys_kernel");
  int bits = 1;
  while (bits < 64 && (static_cast<unsigned long long>(n) * static_cast<unsigned long long>(n) >> bits) != 0) ++bits;
  GM_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, static_cast<int>(len), 0, bits, st));
  GM_TRY_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st));
  asym_kernel<<<grid_for(len), 256, 0, st>>>(src, dst, len, n, sorted, first);
  GM_CHECK_LAUNCH("asym_kernel");
  unsigned long long pos = 0;
  GM_TRY_CUDA(cudaMemcpyAsync(&pos, first, sizeof(pos), cudaMemcpyDeviceToHost, st));
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  if (pos != ~0ull) *pos_host = static_cast<int64_t>(pos);
  return GM_OK;
}

GM_API gm_status gm_mark_columns(const gm_csr* csr, uint8_t* mark, gm_stream_t stream) {
  GM_REQUIRE(csr && mark, GM_ERR_INVALID_ARGUMENT, "gm_mark_columns: null argument");
  cudaStream_t st = as_stream(stream);
  GM_TRY_CUDA(cudaMemsetAsync(mark, 0, static_cast<size_t>(csr->num_cols), st));
  if (csr->num_rows == 0 || csr->nnz == 0) return GM_OK;
  mark_columns_kernel<<<grid_for(csr->nnz), 256, 0, st>>>(csr->rowptr, csr->num_rows, csr->col, mark);
  GM_CHECK_LAUNCH("mark_columns_kernel");
  return GM_OK;
}

GM_API gm_status gm_gather_rows(gm_dtype dtype, const void* x, int64_t f, const int32_t* idx, int64_t n, void* out,
                                gm_stream_t stream) {
  GM_REQUIRE(f >= 0 && n >= 0, GM_ERR_INVALID_ARGUMENT, "gm_gather_rows: negative size");
  if (n == 0 || f == 0) return GM_OK;
  GM_REQUIRE(x && idx && out, GM_ERR_INVALID_ARGUMENT, "gm_gather_rows: null pointer");
  const int64_t esz = dtype == GM_F64 ? 8 : dtype == GM_F32 ? 4 : 2;
  const int64_t rb = f * esz;
  const uintptr_t al = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) | static_cast<uintptr_t>(rb);
  cudaStream_t st = as_stream(stream);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 8), kNumSMs * 32));
  const auto* xb = static_cast<const unsigned char*>(x);
  auto* ob = static_cast<unsigned char*>(out);
  if (al % 16 == 0) gather_rows_kernel<16><<<grid, 256, 0, st>>>(xb, rb, idx, n, ob);
  else if (al % 8 == 0) gather_rows_kernel<8><<<grid, 256, 0, st>>>(xb, rb, idx, n, ob);
  else if (al % 4 == 0) gather_rows_kernel<4><<<grid, 256, 0, st>>>(xb, rb, idx, n, ob);
  else gather_rows_kernel<2><<<grid, 256, 0, st>>>(xb, rb, idx, n, ob);
  GM_CHECK_LAUNCH("gather_rows_kernel");
  return GM_OK;
}

GM_API size_t gm_csr_split_blocks_workspace(int64_t num_rows, int32_t num_blocks) {
  if (num_rows < 0 || num_blocks < 1) return 0;
  return split_layout(nullptr, num_rows, num_blocks).bytes;
}

GM_API gm_status gm_csr_split_blocks(const gm_csr* csr, const int32_t* src_block, const int32_t* src_col,
                                     int32_t num_blocks, int64_t* rowptr_out, int32_t* col_out,
                                     int32_t* perm_out, void* workspace, size_t workspace_bytes,
                                     gm_stream_t stream) {
  GM_REQUIRE(csr, GM_ERR_INVALID_ARGUMENT, "gm_csr_split_blocks: null csr");
  GM_REQUIRE(num_blocks >= 1 && num_blocks <= 1024, GM_ERR_INVALID_ARGUMENT,
             "gm_csr_split_blocks: num_blocks must be in [1, 1024]");
  GM_REQUIRE(csr->num_rows >= 0 && csr->nnz >= 0, GM_ERR_INVALID_ARGUMENT, "gm_csr_split_blocks: negative size");
  GM_REQUIRE(csr->nnz == 0 || csr->perm, GM_ERR_INVALID_ARGUMENT, "gm_csr_split_blocks: csr->perm required");
  GM_REQUIRE(rowptr_out, GM_ERR_INVALID_ARGUMENT, "gm_csr_split_blocks: null rowptr_out");
  const int64_t rows = csr->num_rows;
  const SplitWs need = split_layout(nullptr, rows, num_blocks);
  GM_REQUIRE(workspace && workspace_bytes >= need.bytes, GM_ERR_INVALID_ARGUMENT,
             "gm_csr_split_blocks: workspace too small (" + std::to_string(workspace_bytes) + " < " +
                 std::to_string(need.bytes) + ")");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) {
    GM_TRY_CUDA(cudaMemsetAsync(rowptr_out, 0, sizeof(int64_t) * static_cast<size_t>(num_blocks), st));
    return GM_OK;
  }
  const SplitWs w = split_layout(workspace, rows, num_blocks);
  const int64_t n = rows * num_blocks;
  GM_TRY_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * static_cast<size_t>(n), st));
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(rows, kSplitWarps), kNumSMs * 16));
  if (csr->nnz > 0) {
    split_count_kernel<<<grid, kSplitWarps * 32, 0, st>>>(csr->rowptr, rows, csr->col, src_block, w.cnt);
    GM_CHECK_LAUNCH("split_count_kernel");
  }
  const int64_t nbk = ceil_div(n, kScanTile);
  scan_reduce_kernel<<<static_cast<unsigned>(nbk), kScanThreads, 0, st>>>(w.cnt, n, w.partial);
  GM_CHECK_LAUNCH("scan_reduce_kernel");
  scan_partials_kernel<<<1, kScanThreads, 0, st>>>(w.partial, nbk);
  GM_CHECK_LAUNCH("scan_partials_kernel");
  scan_down_kernel<<<static_cast<unsigned>(nbk), kScanThreads, 0, st>>>(w.cnt, n, w.partial, w.off);
  GM_CHECK_LAUNCH("scan_down_kernel");
  if (csr->nnz > 0) {
    const size_t smem = sizeof(int32_t) * kSplitWarps * static_cast<size_t>(num_blocks);
    if (smem > 48 * 1024)
      GM_TRY_CUDA(cudaFuncSetAttribute(split_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    split_scatter_kernel<<<grid, kSplitWarps * 32, smem, st>>>(csr->rowptr, rows, csr->col, csr->perm, src_block,
                                                               src_col, num_blocks, w.off, col_out, perm_out);
    GM_CHECK_LAUNCH("split_scatter_kernel");
  }
  split_rowptr_kernel<<<grid_for(num_blocks * (rows + 1)), 256, 0, st>>>(w.off, rows, num_blocks, rowptr_out);
  GM_CHECK_LAUNCH("split_rowptr_kernel");
  return GM_OK;
}

GM_API gm_status gm_check_index_bounds(const int64_t* ids, int64_t len, int64_t bound,
                                       const char* prefix, void* workspace, gm_stream_t stream) {
  GM_REQUIRE(len >= 0, GM_ERR_INVALID_ARGUMENT, "gm_check_index_bounds: negative length");
  if (len == 0) return GM_OK;
  GM_REQUIRE(ids && workspace, GM_ERR_INVALID_ARGUMENT, "gm_check_index_bounds: null pointer");
  cudaStream_t st = as_stream(stream);
  auto* first = static_cast<unsigned long long*>(workspace);
  GM_TRY_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st));
  bounds_kernel<<<grid_for(len), 256, 0, st>>>(ids, len, bound, first);
  GM_CHECK_LAUNCH("bounds_kernel");
  unsigned long long pos = 0;
  GM_TRY_CUDA(cudaMemcpyAsync(&pos, first, sizeof(pos), cudaMemcpyDeviceToHost, st));
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  if (pos == ~0ull) return GM_OK;
  int64_t bad = 0;
  GM_TRY_CUDA(cudaMemcpy(&bad, ids + pos, sizeof(bad), cudaMemcpyDeviceToHost));
  return fail(GM_ERR_OUT_OF_RANGE, std::string(prefix ? prefix : "") + " index " + std::to_string(bad) +
                                       " at position " + std::to_string(pos) + " outside [0, " +
                                       std::to_string(bound) + ")");
}

GM_API gm_status gm_first_unsorted(const int64_t* keys, int64_t len, int64_t* pos_host,
                                   void* workspace, gm_stream_t stream) {
  GM_REQUIRE(pos_host, GM_ERR_INVALID_ARGUMENT, "gm_first_unsorted: null output");
  *pos_host = -1;
  if (len < 2) return GM_OK;
  GM_REQUIRE(keys && workspace, GM_ERR_INVALID_ARGUMENT, "gm_first_unsorted: null pointer");
  cudaStream_t st = as_stream(stream);
  auto* first = static_cast<unsigned long long*>(workspace);
  GM_TRY_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st));
  unsorted_kernel<<<grid_for(len), 256, 0, st>>>(keys, len, first);
  GM_CHECK_LAUNCH("unsorted_kernel");
  unsigned long long pos = 0;
  GM_TRY_CUDA(cudaMemcpyAsync(&pos, first, sizeof(pos), cudaMemcpyDeviceToHost, st));
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  if (pos != ~0ull) *pos_host = static_cast<int64_t>(pos);
  return GM_OK;
}

GM_API gm_status gm_degree(const int64_t* ids, int64_t len, int64_t n, int32_t* deg,
                           gm_stream_t stream) {
  GM_REQUIRE(len >= 0 && n >= 0, GM_ERR_INVALID_ARGUMENT, "gm_degree: negative size");
  if (n == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  GM_TRY_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * static_cast<size_t>(n), st));
  if (len == 0) return GM_OK;
  degree_kernel<<<grid_for(len), 256, 0, st>>>(ids, len, n, deg);
  GM_CHECK_LAUNCH("degree_kernel");
  return GM_OK;
}

GM_API gm_status gm_gcn_degrees(const int64_t* full_src, const int64_t* full_dst, int64_t len,
                                int64_t n_src, int64_t n_dst, int square, int32_t* deg_src,
                                int32_t* deg_dst, gm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  gm_status s = gm_degree(full_dst, len, n_dst, deg_dst, stream);
  if (s != GM_OK) return s;
  if (square) {
    // message_passing.hpp:447: din += 1 for the self loop every node receives
    if (n_dst > 0) {
      gcn_finish_kernel<<<static_cast<unsigned>(ceil_div(n_dst, 256)), 256, 0, st>>>(deg_dst, n_dst, 1, 0);
      GM_CHECK_LAUNCH("gcn_finish_kernel");
    }
    if (deg_src != deg_dst && n_dst > 0)
      GM_TRY_CUDA(cudaMemcpyAsync(deg_src, deg_dst, sizeof(int32_t) * static_cast<size_t>(n_dst),
                                  cudaMemcpyDeviceToDevice, st));
    return GM_OK;
  }
  // message_passing.hpp:452-460: dout(src), din(dst), each clamped to >= 1
  s = gm_degree(full_src, len, n_src, deg_src, stream);
  if (s != GM_OK) return s;
  if (n_src > 0) {
    gcn_finish_kernel<<<static_cast<unsigned>(ceil_div(n_src, 256)), 256, 0, st>>>(deg_src, n_src, 0, 1);
    GM_CHECK_LAUNCH("gcn_finish_kernel");
  }
  if (n_dst > 0) {
    gcn_finish_kernel<<<static_cast<unsigned>(ceil_div(n_dst, 256)), 256, 0, st>>>(deg_dst, n_dst, 0, 1);
    GM_CHECK_LAUNCH("gcn_finish_kernel");
  }
  return GM_OK;
}

GM_API size_t gm_build_compressed_workspace(int64_t num_edges, int64_t num_rows) {
  if (num_edges < 0 || num_rows < 0) return 0;
  size_t b = build_layout(nullptr, num_edges, num_rows).bytes;
  size_t extra = 0;
  if (cb::bucket_path_ok(num_edges, num_rows)) extra = cb::bucket_layout(nullptr, num_edges, num_rows).bytes;
  if (num_edges > 0) extra = std::max(extra, rx::radix_layout(nullptr, num_edges).bytes);
  return b + extra;
}

GM_API gm_status gm_build_compressed(const int64_t* keys, const int64_t* values,
                                     int64_t num_edges, int64_t num_rows, int64_t* rowptr,
                                     int32_t* col, int32_t* perm, void* workspace,
                                     size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(num_edges >= 0 && num_rows >= 0, GM_ERR_INVALID_ARGUMENT,
             "build_compressed: negative size");
  GM_REQUIRE(num_edges < INT32_MAX && num_rows < INT32_MAX, GM_ERR_INVALID_ARGUMENT,
             "build_compressed: num_edges and num_rows must be < 2^31 (int32 col/perm)");
  GM_REQUIRE(rowptr, GM_ERR_INVALID_ARGUMENT, "build_compressed: null rowptr");
  const size_t need = gm_build_compressed_workspace(num_edges, num_rows);
  GM_REQUIRE(workspace_bytes >= need && workspace, GM_ERR_INVALID_ARGUMENT,
             "build_compressed: workspace too small (" + std::to_string(workspace_bytes) + " < " +
                 std::to_string(need) + ")");
  cudaStream_t st = as_stream(stream);
  if (num_rows == 0) {  // rowptr = {0}
    GM_TRY_CUDA(cudaMemsetAsync(rowptr, 0, sizeof(int64_t), st));
    return GM_OK;
  }
  if (use_radix_build(num_edges, num_rows)) {  // needs no count pass: rowptr comes from the sorted keys
    const rx::RadixWs rw = rx::radix_layout(static_cast<unsigned char*>(workspace) +
                                                build_layout(nullptr, num_edges, num_rows).bytes, num_edges);
    return rx::radix_build(keys, values, num_edges, num_rows, rowptr, col, perm, rw, st);
  }
  const BuildWs w = build_layout(workspace, num_edges, num_rows);
  GM_TRY_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * static_cast<size_t>(num_rows), st));
  GM_TRY_CUDA(cudaMemsetAsync(w.counters, 0, 64, st));
  if (num_edges > 0) {
    count_kernel<<<grid_for(num_edges), 256, 0, st>>>(keys, num_edges, w.cnt);
    GM_CHECK_LAUNCH("count_kernel");
  }
  const int64_t nb = ceil_div(num_rows, kScanTile);
  scan_reduce_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(w.cnt, num_rows, w.partial);
  GM_CHECK_LAUNCH("scan_reduce_kernel");
  scan_partials_kernel<<<1, kScanThreads, 0, st>>>(w.partial, nb);
  GM_CHECK_LAUNCH("scan_partials_kernel");
  scan_down_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(w.cnt, num_rows, w.partial, rowptr);
  GM_CHECK_LAUNCH("scan_down_kernel");
  if (num_edges == 0) return GM_OK;
  if (use_bucket_build(num_edges, num_rows)) {
    const cb::BucketWs bw = cb::bucket_layout(static_cast<unsigned char*>(workspace) + w.bytes, num_edges, num_rows);
    return cb::bucket_build(keys, values, num_edges, num_rows, rowptr, col, perm, bw, st);
  }
  scatter_kernel<<<grid_for(num_edges), 256, 0, st>>>(keys, num_edges, rowptr, w.cnt, perm);
  GM_CHECK_LAUNCH("scatter_kernel");
  sort_small_kernel<<<grid_for(num_rows * 32), 256, 0, st>>>(rowptr, num_rows, values, perm, col,
                                                             w.med, w.big, w.counters);
  GM_CHECK_LAUNCH("sort_small_kernel");
  sort_med_kernel<<<kNumSMs * 4, kSortThreads, 0, st>>>(rowptr, values, perm, col, w.med, w.counters);
  GM_CHECK_LAUNCH("sort_med_kernel");
  sort_big_kernel<<<kNumSMs, kSortThreads, 0, st>>>(rowptr, values, perm, col, w.scratch, w.big,
                                                    w.counters);
  GM_CHECK_LAUNCH("sort_big_kernel");
  return GM_OK;
}

GM_API gm_status gm_permute_edge_values(gm_dtype dtype, const void* in, const int32_t* perm,
                                        int64_t nnz, void* out, gm_stream_t stream) {
  GM_REQUIRE(nnz >= 0, GM_ERR_INVALID_ARGUMENT, "gm_permute_edge_values: negative nnz");
  if (nnz == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F32)
    permute_kernel_4<<<grid_for(nnz), 256, 0, st>>>(static_cast<const uint32_t*>(in), perm, nnz,
                                                    static_cast<uint32_t*>(out));
  else if (dtype == GM_F64)
    permute_kernel_8<<<grid_for(nnz), 256, 0, st>>>(static_cast<const uint64_t*>(in), perm, nnz,
                                                    static_cast<uint64_t*>(out));
  else
    permute_kernel_2<<<grid_for(nnz), 256, 0, st>>>(static_cast<const uint16_t*>(in), perm, nnz,
                                                    static_cast<uint16_t*>(out));
  GM_CHECK_LAUNCH("permute_kernel");
  return GM_OK;
}

}  // extern "C"
