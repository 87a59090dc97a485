// csr_bucket.cuh — build_compressed (edge_index.cpp:45-62) as a two-level
// STABLE bucket sort (included by csr_build.cu; uses its count/scan kernels).
//
// The reference is a stable counting sort: rowptr from the key counts, then a
// cursor scatter in ascending COO position, so within a row entries keep
// their COO order. Here, with rowptr known from the counts:
//   1. buckets: consecutive row ranges of <= kBucketRows rows and about
//      kBucketEdges entries; a row with more than kBucketEdges entries is a
//      bucket of its own. A bucket's entries occupy [rowptr[r0], rowptr[r1])
//      of the output, exactly like its rows do.
//   2. tile histograms of the bucket id (8192 consecutive COO positions per
//      tile) -> table[bucket][tile], exclusive scan (bucket-major) = the first
//      output slot of every (bucket, tile) run.
//   3. stable scatter: inside a tile every warp walks its 512 positions in
//      order (__match_any_sync ranks equal buckets inside a 32-position round,
//      per-warp shared counters carry across rounds, a per-bucket prefix over
//      warps orders the warps), so a bucket's entries land in COO order;
//      staged as (local row u16, COO position, value).
//   4. per bucket, one CTA ranks its entries by row the same way (per-warp
//      row counters over contiguous sub-ranges, prefix over warps) and writes
//      perm / col at their final slots; single-row buckets are plain copies.
// Every rank is computed in position order, so the result is the reference's
// bit for bit, independent of scheduling (no atomics decide an order).
// Traffic: ~56 B per entry (keys read 3x, values once, 10 B staged out and
// back, 8 B of col/perm) against 7.8 ms of per-row sorting before.
#pragma once

namespace gm {
namespace cb {

constexpr int kBucketRows = 1024;         // K4 shared row counters per warp (10-bit local row)
constexpr int64_t kBucketEdges = 131072;  // target entries per bucket
constexpr int kMaxBuckets = 4096;         // K1/K3 shared histograms
constexpr int kTileWarps = 16;
constexpr int kTileThreads = 32 * kTileWarps;
constexpr int kRounds = 16;               // 32-position rounds per warp
constexpr int kTileItems = kTileThreads * kRounds;  // 8192 positions per tile
constexpr int kFinWarps = 16;  // one 64 KB CTA per SM keeps the open output regions L2-resident

// Upper bound of the bucket count (boundaries: every kBucketRows rows, every
// kBucketEdges entries, and both sides of every hub row).
inline int64_t max_buckets(int64_t rows, int64_t edges) {
  return ceil_div(rows, kBucketRows) + ceil_div(edges, kBucketEdges) + 2 * (edges / kBucketEdges) + 1;
}

__device__ __forceinline__ bool bucket_starts_at(const int64_t* __restrict__ rowptr, int64_t r) {
  if (r == 0 || r % kBucketRows == 0) return true;
  const int64_t a = rowptr[r - 1], b = rowptr[r], c = rowptr[r + 1];
  if (a / kBucketEdges != b / kBucketEdges) return true;               // an entry-count cut
  return (c - b) > kBucketEdges || (b - a) > kBucketEdges;             // a hub row starts / ends here
}

__global__ void bucket_flags_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int32_t* __restrict__ flag) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[r] = bucket_starts_at(rowptr, r) ? 1 : 0;
}

// excl = exclusive scan of the flags: bucket_of[r] = excl[r] + flag[r] - 1,
// first_row[b] = the row that opens bucket b, first_row[D] = rows, *num = D.
__global__ void bucket_finish_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int32_t* __restrict__ bucket_of,
                                     int32_t* __restrict__ first_row, int32_t* __restrict__ num) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool f = bucket_starts_at(rowptr, r);
    const int32_t b = bucket_of[r] + (f ? 1 : 0) - 1;
    bucket_of[r] = b;
    if (f) first_row[b] = static_cast<int32_t>(r);
    if (r == rows - 1) {
      first_row[b + 1] = static_cast<int32_t>(rows);
      *num = b + 1;
    }
  }
}

// 2. table[d * tiles + t] = entries of tile t whose row lies in bucket d;
// code[i] = bucket << 16 | local row (read back by the scatter instead of the
// int64 key and the bucket_of gather).
__global__ void __launch_bounds__(kTileThreads) tile_hist_kernel(const int64_t* __restrict__ keys, int64_t e,
                                                                 const int32_t* __restrict__ bucket_of,
                                                                 const int32_t* __restrict__ first_row, int32_t nb_max,
                                                                 int64_t tiles, int32_t* __restrict__ table,
                                                                 uint32_t* __restrict__ code) {
  __shared__ int32_t hist[kMaxBuckets];
  const int64_t t = blockIdx.x;
  for (int d = threadIdx.x; d < nb_max; d += kTileThreads) hist[d] = 0;
  __syncthreads();
  const int64_t base = t * kTileItems;
  const int64_t end = min(e, base + kTileItems);
  for (int64_t i = base + threadIdx.x; i < end; i += kTileThreads) {
    const int64_t k = keys[i];
    const int32_t d = bucket_of[k];
    atomicAdd(&hist[d], 1);
    code[i] = (static_cast<uint32_t>(d) << 16) | static_cast<uint32_t>(k - first_row[d]);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nb_max; d += kTileThreads) table[static_cast<int64_t>(d) * tiles + t] = hist[d];
}

// Lanes of the warp holding the same BITS-bit key as this lane: one ballot
// per key bit (warp multisplit; cheaper than __match_any_sync). Invalid lanes
// pass valid = false and are never anyone's peer.
template <int BITS>
__device__ __forceinline__ unsigned peers_of(uint32_t key, bool valid) {
  unsigned m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bb = __ballot_sync(0xffffffffu, (key >> b) & 1u);
    m &= ((key >> b) & 1u) ? bb : ~bb;
  }
  return m;
}

// 3. stable scatter of each tile's entries into their buckets' runs.
// Persistent CTAs (one per SM: the per-warp histograms fill shared memory)
// walk tiles blockIdx.x, +gridDim.x, ...; the next tile's codes, values and
// table offsets are loaded into registers while the current tile is ranked
// and scattered, so the SM's memory pipe never idles between phases. Staged as
// (local row u16) and (COO position, value) int2.
__global__ void __launch_bounds__(kTileThreads, 1) tile_scatter_kernel(
    const uint32_t* __restrict__ code, const int64_t* __restrict__ values, int64_t e, int32_t nb_max, int64_t tiles,
    const int32_t* __restrict__ table_off, uint16_t* __restrict__ st_row, int2* __restrict__ st_pv) {
  extern __shared__ int32_t tile_off[];  // [nb_max] this tile's first slot per bucket, then whist
  uint16_t* whist = reinterpret_cast<uint16_t*>(tile_off + nb_max);  // [kTileWarps][nb_max]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint16_t* my = whist + w * nb_max;
  const unsigned lt = (1u << lane) - 1u;
  constexpr int kOffPer = kMaxBuckets / kTileThreads;
  uint32_t c[kRounds], cn[kRounds];  // bucket << 16 | local row (ranked: rank << 22 | bucket << 10 | row)
  int32_t val[kRounds], valn[kRounds];
  int32_t toff[kOffPer], toffn[kOffPer];
  auto load = [&](int64_t t, uint32_t* cc, int32_t* vv, int32_t* oo) {
    const int64_t wbase = t * kTileItems + static_cast<int64_t>(w) * (32 * kRounds);
#pragma unroll
    for (int j = 0; j < kRounds; ++j) {
      const int64_t i = wbase + j * 32 + lane;
      const bool ok = t < tiles && i < e;
      cc[j] = ok ? __ldcs(code + i) : 0xffffffffu;
      vv[j] = ok ? static_cast<int32_t>(__ldcs(values + i)) : 0;
    }
#pragma unroll
    for (int q = 0; q < kOffPer; ++q) {
      const int d = threadIdx.x + q * kTileThreads;
      oo[q] = (t < tiles && d < nb_max) ? table_off[static_cast<int64_t>(d) * tiles + t] : 0;
    }
  };
  int64_t t = blockIdx.x;
  load(t, c, val, toff);
  for (int i = threadIdx.x; i < (kTileWarps * nb_max + 1) / 2; i += kTileThreads) reinterpret_cast<uint32_t*>(whist)[i] = 0u;
  for (; t < tiles; t += gridDim.x) {
    __syncthreads();  // counters zeroed, previous tile's scatter done
    load(t + gridDim.x, cn, valn, toffn);  // next tile, in flight during this one
#pragma unroll
    for (int j = 0; j < kRounds; ++j) {
      const bool valid = c[j] != 0xffffffffu;
      const uint32_t d = valid ? (c[j] >> 16) : 0u;
      const unsigned peers = peers_of<12>(d, valid);
      uint16_t old = 0;
      if (valid) old = my[d];
      __syncwarp();
      if (valid && (peers & lt) == 0) my[d] = static_cast<uint16_t>(old + __popc(peers));
      __syncwarp();
      // rank inside the warp's 512 positions (< 512) in bits 22..31, bucket in
      // bits 10..21, local row (kBucketRows = 1024) in bits 0..9
      if (valid) c[j] = (static_cast<uint32_t>(old + __popc(peers & lt)) << 22) | (d << 10) | (c[j] & 0x3ffu);
    }
    __syncthreads();
    // per bucket: exclusive prefix over the warps (tile totals <= 8192 fit
    // u16) and this tile's first output slot
#pragma unroll
    for (int q = 0; q < kOffPer; ++q) {
      const int d = threadIdx.x + q * kTileThreads;
      if (d < nb_max) {
        uint16_t run = 0;
#pragma unroll
        for (int ww = 0; ww < kTileWarps; ++ww) {
          const uint16_t cnt = whist[ww * nb_max + d];
          whist[ww * nb_max + d] = run;
          run = static_cast<uint16_t>(run + cnt);
        }
        tile_off[d] = toff[q];
      }
    }
    __syncthreads();
    const int64_t wbase = t * kTileItems + static_cast<int64_t>(w) * (32 * kRounds);
#pragma unroll
    for (int j = 0; j < kRounds; ++j) {
      const int64_t i = wbase + j * 32 + lane;
      if (i < e) {
        const int32_t d = static_cast<int32_t>((c[j] >> 10) & 0xfffu);
        const int64_t out = static_cast<int64_t>(tile_off[d]) + my[d] + (c[j] >> 22);
        st_row[out] = static_cast<uint16_t>(c[j] & 0x3ffu);
        st_pv[out] = make_int2(static_cast<int32_t>(i), val[j]);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (kTileWarps * nb_max + 1) / 2; i += kTileThreads)
      reinterpret_cast<uint32_t*>(whist)[i] = 0u;
#pragma unroll
    for (int j = 0; j < kRounds; ++j) {
      c[j] = cn[j];
      val[j] = valn[j];
    }
#pragma unroll
    for (int q = 0; q < kOffPer; ++q) toff[q] = toffn[q];
  }
}

// 4. per bucket: rank by row (stable), write perm / col at the final slots.
__global__ void __launch_bounds__(32 * kFinWarps) bucket_finalize_kernel(
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ first_row, const int32_t* __restrict__ num,
    const uint16_t* __restrict__ st_row, const int2* __restrict__ st_pv, int32_t* __restrict__ perm,
    int32_t* __restrict__ col) {
  extern __shared__ int32_t fin_smem[];  // [kFinWarps][kBucketRows] row counters
  int32_t(*cnt)[kBucketRows] = reinterpret_cast<int32_t(*)[kBucketRows]>(fin_smem);
  const int b = blockIdx.x;
  if (b >= *num) return;
  const int32_t r0 = first_row[b], r1 = first_row[b + 1];
  const int64_t s = rowptr[r0], e = rowptr[r1];
  if (e == s) return;
  if (r1 - r0 == 1) {  // one row (a hub): already in COO order
    for (int64_t k = s + threadIdx.x; k < e; k += blockDim.x) {
      const int2 pv = st_pv[k];
      perm[k] = pv.x;
      col[k] = pv.y;
    }
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nr = r1 - r0;
  for (int i = threadIdx.x; i < kFinWarps * kBucketRows; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t len = e - s;
  const int64_t ws = s + len * w / kFinWarps, we = s + len * (w + 1) / kFinWarps;
  constexpr int kFinU = 4;  // 32-entry batches in flight per warp
  for (int64_t k0 = ws; k0 < we; k0 += 32 * kFinU) {
    uint16_t rr[kFinU];
#pragma unroll
    for (int u = 0; u < kFinU; ++u) {
      const int64_t k = k0 + u * 32 + lane;
      rr[u] = k < we ? st_row[k] : 0xffff;
    }
#pragma unroll
    for (int u = 0; u < kFinU; ++u)
      if (rr[u] != 0xffff) atomicAdd(&cnt[w][rr[u]], 1);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    int32_t run = static_cast<int32_t>(rowptr[r0 + r] - s);
#pragma unroll
    for (int ww = 0; ww < kFinWarps; ++ww) {
      const int32_t c = cnt[ww][r];
      cnt[ww][r] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t k1 = ws; k1 < we; k1 += 32 * kFinU) {
    uint32_t rr[kFinU];
    int2 pv[kFinU];
#pragma unroll
    for (int u = 0; u < kFinU; ++u) {
      const int64_t k = k1 + u * 32 + lane;
      const bool valid = k < we;
      rr[u] = valid ? static_cast<uint32_t>(st_row[k]) : 0xffffffffu;
      pv[u] = valid ? st_pv[k] : make_int2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kFinU; ++u) {
      const bool valid = rr[u] != 0xffffffffu;
      const uint32_t r = valid ? rr[u] : 0u;
      const unsigned peers = peers_of<10>(r, valid);
      int32_t old = 0;
      if (valid) old = cnt[w][r];
      __syncwarp();
      if (valid && (peers & lt) == 0) cnt[w][r] = old + __popc(peers);
      __syncwarp();
      if (valid) {
        const int64_t dst = s + old + __popc(peers & lt);
        perm[dst] = pv[u].x;
        col[dst] = pv[u].y;
      }
    }
  }
}

// int32 exclusive scan in place (values and total < 2^31): per-block sums,
// one block scans the sums, then the down-sweep.
constexpr int kScan32Threads = 512;
constexpr int kScan32Items = 16;
constexpr int kScan32Tile = kScan32Threads * kScan32Items;

__device__ __forceinline__ int32_t block_excl_scan32(int32_t v, int32_t* warp_tot, int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int32_t t = lane < kScan32Threads / 32 ? warp_tot[lane] : 0;
    int32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t n = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += n;
    }
    if (lane < kScan32Threads / 32) warp_tot[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  return inc - v + warp_tot[wid];
}

__global__ void __launch_bounds__(kScan32Threads) scan32_reduce_kernel(const int32_t* __restrict__ a, int64_t n,
                                                                       int32_t* __restrict__ partial) {
  __shared__ int32_t wt[kScan32Threads / 32];
  __shared__ int32_t tot;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScan32Tile;
  int32_t s = 0;
  for (int i = 0; i < kScan32Items; ++i) {
    const int64_t idx = base + static_cast<int64_t>(i) * kScan32Threads + threadIdx.x;
    if (idx < n) s += a[idx];
  }
  block_excl_scan32(s, wt, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScan32Threads) scan32_partials_kernel(int32_t* __restrict__ partial, int64_t nb) {
  __shared__ int32_t wt[kScan32Threads / 32];
  __shared__ int32_t tot;
  int32_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScan32Threads) {
    const int64_t idx = base + threadIdx.x;
    const int32_t v = idx < nb ? partial[idx] : 0;
    const int32_t ex = block_excl_scan32(v, wt, &tot);
    if (idx < nb) partial[idx] = carry + ex;
    __syncthreads();
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScan32Threads) scan32_down_kernel(int32_t* __restrict__ a, int64_t n,
                                                                     const int32_t* __restrict__ partial) {
  __shared__ int32_t wt[kScan32Threads / 32];
  __shared__ int32_t tot;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScan32Tile + static_cast<int64_t>(threadIdx.x) * kScan32Items;
  int32_t v[kScan32Items];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScan32Items; ++i) {
    v[i] = base + i < n ? a[base + i] : 0;
    s += v[i];
  }
  int32_t run = block_excl_scan32(s, wt, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScan32Items; ++i) {
    if (base + i < n) a[base + i] = run;
    run += v[i];
  }
}

inline int64_t scan32_blocks(int64_t n) { return std::max<int64_t>(1, ceil_div(n, kScan32Tile)); }

inline gm_status scan32_exclusive(int32_t* a, int64_t n, int32_t* partial, cudaStream_t st) {
  if (n == 0) return GM_OK;
  const int64_t nb = scan32_blocks(n);
  scan32_reduce_kernel<<<static_cast<unsigned>(nb), kScan32Threads, 0, st>>>(a, n, partial);
  GM_CHECK_LAUNCH("scan32_reduce_kernel");
  scan32_partials_kernel<<<1, kScan32Threads, 0, st>>>(partial, nb);
  GM_CHECK_LAUNCH("scan32_partials_kernel");
  scan32_down_kernel<<<static_cast<unsigned>(nb), kScan32Threads, 0, st>>>(a, n, partial);
  GM_CHECK_LAUNCH("scan32_down_kernel");
  return GM_OK;
}

struct BucketWs {
  int32_t* bucket_of;  // [rows]
  int32_t* first_row;  // [nb_max + 1]
  int32_t* num;        // [1]
  int32_t* table;      // [nb_max * tiles]
  int32_t* partial;    // scan32 block sums
  uint32_t* code;      // [e] bucket << 16 | local row
  uint16_t* st_row;    // [e]
  int2* st_pv;         // [e] (COO position, value)
  size_t bytes;
};

inline BucketWs bucket_layout(void* base, int64_t e, int64_t rows) {
  BucketWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + off : nullptr;
    off += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  const int64_t nb = max_buckets(rows, e);
  const int64_t tiles = ceil_div(e, kTileItems);
  w.bucket_of = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(rows)));
  w.first_row = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(nb + 1)));
  w.num = reinterpret_cast<int32_t*>(take(sizeof(int32_t)));
  w.table = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(nb * tiles)));
  w.partial = reinterpret_cast<int32_t*>(
      take(sizeof(int32_t) * static_cast<size_t>(scan32_blocks(std::max(nb * tiles, rows)))));
  w.code = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * static_cast<size_t>(e)));
  w.st_row = reinterpret_cast<uint16_t*>(take(sizeof(uint16_t) * static_cast<size_t>(e)));
  w.st_pv = reinterpret_cast<int2*>(take(sizeof(int2) * static_cast<size_t>(e)));
  w.bytes = off;
  return w;
}

// The bucketed path applies when every histogram fits shared memory.
inline bool bucket_path_ok(int64_t e, int64_t rows) {
  return e > 0 && rows > 0 && max_buckets(rows, e) <= kMaxBuckets;
}

// Steps 1-4 (rowptr already computed). values may be any int64 ids < 2^31.
inline gm_status bucket_build(const int64_t* keys, const int64_t* values, int64_t e, int64_t rows,
                              const int64_t* rowptr, int32_t* col, int32_t* perm, const BucketWs& w,
                              cudaStream_t st) {
  const int64_t nb = max_buckets(rows, e);
  const int64_t tiles = ceil_div(e, kTileItems);
  const unsigned g_rows = static_cast<unsigned>(std::min<int64_t>(ceil_div(rows, 256), kNumSMs * 32));
  bucket_flags_kernel<<<g_rows, 256, 0, st>>>(rowptr, rows, w.bucket_of);
  GM_CHECK_LAUNCH("bucket_flags_kernel");
  gm_status s = scan32_exclusive(w.bucket_of, rows, w.partial, st);
  if (s != GM_OK) return s;
  bucket_finish_kernel<<<g_rows, 256, 0, st>>>(rowptr, rows, w.bucket_of, w.first_row, w.num);
  GM_CHECK_LAUNCH("bucket_finish_kernel");
  tile_hist_kernel<<<static_cast<unsigned>(tiles), kTileThreads, 0, st>>>(keys, e, w.bucket_of, w.first_row,
                                                                           static_cast<int32_t>(nb), tiles, w.table,
                                                                           w.code);
  GM_CHECK_LAUNCH("tile_hist_kernel");
  s = scan32_exclusive(w.table, nb * tiles, w.partial, st);
  if (s != GM_OK) return s;
  const size_t smem = (sizeof(int32_t) + sizeof(uint16_t) * kTileWarps) * static_cast<size_t>(nb) + 4;
  if (smem > 48 * 1024)
    GM_TRY_CUDA(cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  tile_scatter_kernel<<<static_cast<unsigned>(std::min<int64_t>(tiles, kNumSMs)), kTileThreads, smem, st>>>(
      w.code, values, e, static_cast<int32_t>(nb), tiles, w.table, w.st_row, w.st_pv);
  GM_CHECK_LAUNCH("tile_scatter_kernel");
  // GM_CSR_FIN_SMEM (bytes, tuning only) can reserve more shared memory to
  // cap the finalize CTAs per SM (fewer open output regions in L2)
  static const size_t fin_env = [] { const char* v = getenv("GM_CSR_FIN_SMEM"); return v ? static_cast<size_t>(atoll(v)) : 0; }();
  const size_t fin_smem = std::max(sizeof(int32_t) * kFinWarps * kBucketRows, std::min<size_t>(fin_env, 227 * 1024));
  GM_TRY_CUDA(cudaFuncSetAttribute(bucket_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(fin_smem)));
  bucket_finalize_kernel<<<static_cast<unsigned>(nb), 32 * kFinWarps, fin_smem, st>>>(rowptr, w.first_row, w.num, w.st_row,
                                                                             w.st_pv, perm, col);
  GM_CHECK_LAUNCH("bucket_finalize_kernel");
  return GM_OK;
}

}  // namespace cb
}  // namespace gm
