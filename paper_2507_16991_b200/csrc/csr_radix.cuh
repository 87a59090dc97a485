// csr_radix.cuh — build_compressed (edge_index.cpp:45-62) as a least-
// significant-digit radix sort of (key, COO position, value) triples (included
// by csr_build.cu).
//
// The reference is a stable counting sort by key: within a row, entries keep
// ascending COO position. An LSD radix sort whose every pass is stable yields
// exactly that order, so col / perm come out bit-identical to the reference
// for any input. Digits are 8 bits wide (11 as an A/B knob). Per pass
// (2048-entry tiles of 8 warps):
//   1. radix_hist: per-tile digit counts -> table[tile][digit] (one contiguous
//      row per tile);
//   2. radix_colscan: exclusive scan of every digit's column over the tiles
//      (in place) plus the digit totals; a one-CTA scan of the totals gives
//      each digit's first output slot;
//   3. radix_scatter: every warp ranks its 256 entries round by round
//      (ballot multisplit: one ballot per digit bit, per-warp u16 counters), a
//      per-digit prefix over warps and over digits gives each entry's slot in a
//      digit-sorted copy of the tile in shared memory, and the tile leaves as
//      contiguous digit runs.
// rowptr comes from the sorted keys of the last pass (row boundaries), so no
// atomics anywhere: the result does not depend on scheduling.
#pragma once

namespace gm {
namespace rx {

constexpr int kMaxBits = 11;
#ifndef GM_RADIX_WARPS  // warps per tile (A/B: 4 warps x 8 / 16 rounds 2.48 / 2.05 ms, 2 x 16 2.58; 8 x 8 1.95)
#define GM_RADIX_WARPS 8
#endif
constexpr int kWarps = GM_RADIX_WARPS;
constexpr int kThreads = 32 * kWarps;
// Entries per lane per tile and the scatter's CTAs per SM (same-box A/B on
// C4, whole build: 16 rounds / 2 CTAs 2.06 ms, 12 / 2 2.09, 8 / 3 2.02,
// 8 / 4 (64 registers) 1.94)
#ifndef GM_RADIX_ROUNDS
#define GM_RADIX_ROUNDS 8
#endif
constexpr int kRounds = GM_RADIX_ROUNDS;
constexpr int kTile = kThreads * kRounds;  // entries per tile

// lanes holding the same BITS-bit digit (invalid lanes excluded)
template <int BITS>
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool valid) {
  unsigned m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return m;
}

// Pass input: the first pass reads the caller's int64 keys / values (and the
// position is the index); later passes read the previous pass's u32 triples.
struct In {
  const int64_t* keys64;
  const int64_t* vals64;
  const uint32_t* key;
  const uint32_t* pos;
  const uint32_t* val;
};

__device__ __forceinline__ uint32_t key_at(const In& in, int64_t i) {
  return in.keys64 ? static_cast<uint32_t>(in.keys64[i]) : in.key[i];
}

template <int BITS>
__global__ void __launch_bounds__(kThreads) radix_hist_kernel(In in, int64_t e, int shift,
                                                              int32_t* __restrict__ table) {
  constexpr int kBins = 1 << BITS;
  __shared__ int32_t hist[kBins];
  const int64_t t = blockIdx.x;
  for (int d = threadIdx.x; d < kBins; d += kThreads) hist[d] = 0;
  __syncthreads();
  const int64_t base = t * kTile;
  const int64_t end = min(e, base + kTile);
  for (int64_t i = base + threadIdx.x; i < end; i += kThreads)
    atomicAdd(&hist[(key_at(in, i) >> shift) & (kBins - 1)], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < kBins; d += kThreads) table[t * kBins + d] = hist[d];
}

// Digit counts of every pass in one read of the original keys (counts do not
// depend on the order a pass sees): total[p * 256 + d], 8-bit digits.
__global__ void __launch_bounds__(256) radix_global_hist_kernel(const int64_t* __restrict__ keys, int64_t e, int passes,
                                                                int dbits, int32_t* __restrict__ total) {
  __shared__ int32_t h[4 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < e;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = static_cast<uint32_t>(__ldcs(keys + i));
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * 256 + ((k >> (p * dbits)) & 255u)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
    if (h[i]) atomicAdd(total + i, h[i]);
}

// Exclusive scan of the tile-major table over tiles, per digit, in place, in
// three steps so every step has thousands of warps in flight:
//   colsum:  warp (digit group of 32, chunk of kChunk tiles) -> part[chunk][d];
//   colscan: the partial table scanned over chunks (one CTA per digit group,
//            its warps owning contiguous chunk ranges) + the digit totals;
//   coldown: each (group, chunk) warp rewrites its tiles as running prefixes.
constexpr int kChunk = 16;  // tiles per warp in colsum / coldown
constexpr int kColWarps = 32;
__global__ void radix_colsum_kernel(const int32_t* __restrict__ table, int64_t tiles, int bins,
                                    int32_t* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int groups = bins / 32;
  const int64_t c = gw / groups;
  const int d = static_cast<int>(gw % groups) * 32 + lane;
  const int64_t t0 = c * kChunk;
  if (t0 >= tiles) return;
  const int64_t t1 = min(tiles, t0 + kChunk);
  int32_t s = 0;
#pragma unroll 4
  for (int64_t t = t0; t < t1; ++t) s += table[t * bins + d];
  part[c * bins + d] = s;
}
__global__ void radix_coldown_kernel(int32_t* __restrict__ table, int64_t tiles, int bins,
                                     const int32_t* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int groups = bins / 32;
  const int64_t c = gw / groups;
  const int d = static_cast<int>(gw % groups) * 32 + lane;
  const int64_t t0 = c * kChunk;
  if (t0 >= tiles) return;
  const int64_t t1 = min(tiles, t0 + kChunk);
  int32_t v[kChunk];
#pragma unroll
  for (int i = 0; i < kChunk; ++i) v[i] = t0 + i < t1 ? table[(t0 + i) * bins + d] : 0;
  int32_t run = part[c * bins + d];
#pragma unroll
  for (int i = 0; i < kChunk; ++i) {
    if (t0 + i < t1) table[(t0 + i) * bins + d] = run;
    run += v[i];
  }
}
// in-place exclusive scan of a [rows][bins] table over rows, per column, plus
// the column totals; one CTA per 32 columns (lane = column)
__global__ void __launch_bounds__(32 * kColWarps) radix_colscan_kernel(int32_t* __restrict__ table, int64_t rows,
                                                                       int bins, int32_t* __restrict__ total) {
  __shared__ int32_t psum[kColWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d = blockIdx.x * 32 + lane;
  const int64_t per = (rows + kColWarps - 1) / kColWarps;
  const int64_t t0 = min(rows, static_cast<int64_t>(w) * per), t1 = min(rows, t0 + per);
  int32_t s = 0;
#pragma unroll 8
  for (int64_t t = t0; t < t1; ++t) s += table[t * bins + d];
  psum[w][lane] = s;
  __syncthreads();
  int32_t before = 0, all = 0;
#pragma unroll 8
  for (int ww = 0; ww < kColWarps; ++ww) {
    const int32_t c = psum[ww][lane];
    before += ww < w ? c : 0;
    all += c;
  }
  int32_t run = before;
  // the rows' counts in flight 8 at a time (the column walk was latency-bound)
  int64_t t = t0;
  for (; t + 8 <= t1; t += 8) {
    int32_t c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = table[(t + i) * bins + d];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      table[(t + i) * bins + d] = run;
      run += c[i];
    }
  }
  for (; t < t1; ++t) {
    const int32_t c = table[t * bins + d];
    table[t * bins + d] = run;
    run += c;
  }
  if (w == 0) total[d] = all;
}

// Exclusive scan of the digit totals (bins <= 2048, one CTA of 1024 threads).
__global__ void __launch_bounds__(1024) radix_digit_scan_kernel(const int32_t* __restrict__ total, int bins,
                                                                int32_t* __restrict__ start) {
  __shared__ int32_t wsum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (bins + 1023) / 1024;
  int32_t v[2] = {0, 0};
  int32_t s = 0;
  for (int j = 0; j < per; ++j) {
    const int d = threadIdx.x * per + j;
    v[j] = d < bins ? total[d] : 0;
    s += v[j];
  }
  int32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int32_t t = wsum[lane];
    int32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t n = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += n;
    }
    wsum[lane] = ti - t;
  }
  __syncthreads();
  int32_t run = wsum[w] + inc - s;
  for (int j = 0; j < per; ++j) {
    const int d = threadIdx.x * per + j;
    if (d < bins) start[d] = run;
    run += v[j];
  }
}

template <int BITS>
constexpr size_t scatter_smem_bytes() {
  return 3 * kTile * sizeof(uint32_t) + kWarps * (1 << BITS) * sizeof(uint16_t) + 2 * ((1 << BITS) + 1) * sizeof(int32_t);
}

// LAST: write perm / col (int32) and the sorted keys (for rowptr) instead of
// the next pass's triples.
#ifndef GM_RADIX_STCS  // intermediate passes: streaming (evict-first) stores of the next pass's triples
#define GM_RADIX_STCS 1
#endif
#ifndef GM_RADIX_MINB
#define GM_RADIX_MINB 4
#endif
// OS (one sweep): no per-pass histogram / column scans; tiles take their index
// from a counter in launch order, publish their digit counts, and find their
// global offsets by decoupled look-back over the predecessors' published
// counts / inclusive prefixes (64-bit status words: epoch-tagged flag << 32 |
// count). The digit starts come from one global histogram of all passes.
template <int BITS, bool LAST, bool OS = false>
__global__ void __launch_bounds__(kThreads, GM_RADIX_MINB) radix_scatter_kernel(In in, int64_t e, int shift,
                                                                 const int32_t* __restrict__ table_off,
                                                                 const int32_t* __restrict__ digit_start,
                                                                 uint32_t* __restrict__ okey, uint32_t* __restrict__ opos,
                                                                 uint32_t* __restrict__ oval,
                                                                 unsigned long long* __restrict__ status = nullptr,
                                                                 int* __restrict__ tile_ctr = nullptr,
                                                                 uint32_t epoch = 0) {
  constexpr int kBins = 1 << BITS;
  constexpr int kPer = kBins >= kThreads ? kBins / kThreads : 1;  // digits per thread
  __shared__ int32_t wsum[kWarps];
  __shared__ int64_t tile_sh;
  extern __shared__ __align__(16) uint32_t stage[];  // digit-sorted tile: key, position, value
  uint32_t* skey = stage;
  uint32_t* spos = stage + kTile;
  uint32_t* sval = stage + 2 * kTile;
  uint16_t* whist = reinterpret_cast<uint16_t*>(stage + 3 * kTile);  // [kWarps][kBins]
  int32_t* dstart = reinterpret_cast<int32_t*>(whist + kWarps * kBins);  // [kBins + 1]
  int32_t* gout = dstart + kBins + 1;                                      // [kBins]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t t = blockIdx.x;
  if constexpr (OS) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(tile_ctr, 1);
    __syncthreads();
    t = tile_sh;
  }
  for (int i = threadIdx.x; i < kWarps * kBins / 2; i += kThreads) reinterpret_cast<uint32_t*>(whist)[i] = 0;
  if constexpr (!OS)
    for (int d = threadIdx.x; d < kBins; d += kThreads)
      gout[d] = digit_start[d] + table_off[t * kBins + d];
  const int64_t wbase = t * kTile + static_cast<int64_t>(w) * (32 * kRounds);
  uint32_t k[kRounds], p[kRounds], v[kRounds];
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    const int64_t i = wbase + j * 32 + lane;
    const bool ok = i < e;
    if (in.keys64) {
      k[j] = ok ? static_cast<uint32_t>(__ldcs(in.keys64 + i)) : 0u;
      v[j] = ok ? static_cast<uint32_t>(__ldcs(in.vals64 + i)) : 0u;
      p[j] = static_cast<uint32_t>(i);
    } else {
      k[j] = ok ? __ldcs(in.key + i) : 0u;
      v[j] = ok ? __ldcs(in.val + i) : 0u;
      p[j] = ok ? __ldcs(in.pos + i) : 0u;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  uint16_t rank[kRounds];
  uint16_t* wh = whist + w * kBins;
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    const bool valid = wbase + j * 32 + lane < e;
    const uint32_t d = (k[j] >> shift) & (kBins - 1);
    // (one __match_any_sync instead of the ballots measured 10% slower per build)
    const unsigned peers = digit_peers<BITS>(d, valid);
    uint16_t old = 0;
    if (valid) old = wh[d];
    __syncwarp();
    if (valid && (peers & lt) == 0) wh[d] = static_cast<uint16_t>(old + __popc(peers));
    __syncwarp();
    rank[j] = static_cast<uint16_t>(old + __popc(peers & lt));
  }
  __syncthreads();
  // per digit: prefix over warps (in place), then an exclusive scan over digits
  // (thread owns kPer consecutive digits)
  {
    int32_t run_d[kPer];
    int32_t s = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int d = threadIdx.x * kPer + q;
      int32_t run = 0;
      if (d < kBins) {
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
          const int32_t c = whist[ww * kBins + d];
          whist[ww * kBins + d] = static_cast<uint16_t>(run);
          run += c;
        }
      }
      run_d[q] = run;
      s += run;
    }
    int32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int32_t before = 0;
    for (int ww = 0; ww < w; ++ww) before += wsum[ww];
    int32_t r = before + inc - s;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int d = threadIdx.x * kPer + q;
      if (d < kBins) dstart[d] = r;
      r += run_d[q];
    }
    if (threadIdx.x == kThreads - 1) dstart[kBins] = r;
  }
  __syncthreads();
  if constexpr (OS) {
    // publish this tile's digit counts, look back for the exclusive prefix
    const unsigned long long f_agg = static_cast<unsigned long long>(2u * epoch + 1u) << 32;
    const unsigned long long f_pre = static_cast<unsigned long long>(2u * epoch + 2u) << 32;
    for (int d = threadIdx.x; d < kBins; d += kThreads) {
      const uint32_t cnt = static_cast<uint32_t>(dstart[d + 1] - dstart[d]);
      unsigned long long* my = status + t * kBins + d;
      if (t == 0) {
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(my), "l"(f_pre | cnt) : "memory");
        gout[d] = digit_start[d];
        continue;
      }
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(my), "l"(f_agg | cnt) : "memory");
      uint32_t excl = 0;
      for (int64_t tp = t - 1; tp >= 0;) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(status + tp * kBins + d) : "memory");
        const unsigned long long fl = v & 0xffffffff00000000ull;
        if (fl == f_pre) {
          excl += static_cast<uint32_t>(v);
          break;
        }
        if (fl == f_agg) {
          excl += static_cast<uint32_t>(v);
          --tp;
        }
      }
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(my), "l"(f_pre | (excl + cnt)) : "memory");
      gout[d] = digit_start[d] + static_cast<int32_t>(excl);
    }
    __syncthreads();
  }
  // digit-sorted copy of the tile in shared memory
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    if (wbase + j * 32 + lane < e) {
      const uint32_t d = (k[j] >> shift) & (kBins - 1);
      const int s = dstart[d] + wh[d] + rank[j];
      skey[s] = k[j];
      spos[s] = p[j];
      sval[s] = v[j];
    }
  }
  __syncthreads();
  // contiguous digit runs out
  const int n = dstart[kBins];
  for (int s = threadIdx.x; s < n; s += kThreads) {
    const uint32_t key = skey[s];
    const uint32_t d = (key >> shift) & (kBins - 1);
    const int64_t o = static_cast<int64_t>(gout[d]) + (s - dstart[d]);
    if constexpr (LAST) {
      okey[o] = key;
      opos[o] = spos[s];  // perm
      oval[o] = sval[s];  // col
    } else {
#if GM_RADIX_STCS
      __stcs(okey + o, key);
      __stcs(opos + o, spos[s]);
      __stcs(oval + o, sval[s]);
#else
      okey[o] = key;
      opos[o] = spos[s];
      oval[o] = sval[s];
#endif
    }
  }
}

// rowptr from the sorted keys: rowptr[r] = first slot with key >= r. Thread q
// owns slots [16q, 16q+16): four 16-byte loads (all in flight) plus the
// previous key; the row starts inside the range (usually none or one) are
// written directly.
constexpr int kRowptrPer = 16;
__global__ void rowptr_from_sorted_kernel(const uint32_t* __restrict__ key, int64_t e, int64_t rows,
                                          int64_t* __restrict__ rowptr) {
  const int64_t groups = (e + kRowptrPer) / kRowptrPer;  // slots 0..e (slot e closes the last rows)
  const bool aligned = (reinterpret_cast<uintptr_t>(key) & 15) == 0;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < groups;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k0 = q * kRowptrPer;
    uint32_t kk[kRowptrPer];
    const int64_t prev = k0 == 0 ? -1 : static_cast<int64_t>(__ldg(key + k0 - 1));
    if (k0 + kRowptrPer <= e && aligned) {
#pragma unroll
      for (int j = 0; j < kRowptrPer / 4; ++j) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(key + k0) + j);
        kk[4 * j] = v.x;
        kk[4 * j + 1] = v.y;
        kk[4 * j + 2] = v.z;
        kk[4 * j + 3] = v.w;
      }
      if (static_cast<int64_t>(kk[kRowptrPer - 1]) == prev) continue;  // no row starts in this range
    } else {
#pragma unroll
      for (int j = 0; j < kRowptrPer; ++j)
        kk[j] = k0 + j < e ? __ldg(key + k0 + j) : static_cast<uint32_t>(rows);
    }
    int64_t before = prev;
#pragma unroll
    for (int j = 0; j < kRowptrPer; ++j) {
      const int64_t k = k0 + j;
      if (k > e) break;
      const int64_t cur = static_cast<int64_t>(kk[j]);
      for (int64_t r = before + 1; r <= cur; ++r) rowptr[r] = k;  // rows (prev, key[k]] start at k
      before = cur;
    }
  }
}

struct RadixWs {
  int32_t* table;    // [bins * tiles]
  int32_t* part;     // [chunks * bins] (scan partials)
  int32_t* total;    // [bins]
  int32_t* start;    // [bins]
  uint32_t* buf[2][3];  // ping-pong (key, pos, val)
  size_t bytes;
};

inline RadixWs radix_layout(void* base, int64_t e) {
  RadixWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + off : nullptr;
    off += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  const int64_t tiles = std::max<int64_t>(1, ceil_div(e, kTile));
  constexpr int64_t bins = int64_t{1} << kMaxBits;
  w.table = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(bins * tiles)));  // [tile][digit]
  w.part = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(bins * ceil_div(tiles, kChunk))));
  w.total = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(bins)));
  w.start = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(bins)));
  for (int b = 0; b < 2; ++b)
    for (int a = 0; a < 3; ++a) w.buf[b][a] = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * static_cast<size_t>(e)));
  w.bytes = off;
  return w;
}

inline int key_bits(int64_t rows) {
  int b = 1;
  while (b < 31 && (int64_t{1} << b) < rows) ++b;
  return b;
}

template <int BITS>
inline gm_status radix_pass(const In& in, int64_t e, int shift, bool last, const RadixWs& w, uint32_t* ok,
                            uint32_t* op, uint32_t* ov, cudaStream_t st) {
  const int64_t tiles = ceil_div(e, kTile);
  constexpr int bins = 1 << BITS;
  radix_hist_kernel<BITS><<<static_cast<unsigned>(tiles), kThreads, 0, st>>>(in, e, shift, w.table);
  GM_CHECK_LAUNCH("radix_hist_kernel");
  const int64_t chunks = ceil_div(tiles, kChunk);
  const unsigned col_grid = static_cast<unsigned>(ceil_div(chunks * (bins / 32) * 32, 256));
  radix_colsum_kernel<<<col_grid, 256, 0, st>>>(w.table, tiles, bins, w.part);
  GM_CHECK_LAUNCH("radix_colsum_kernel");
  radix_colscan_kernel<<<static_cast<unsigned>(bins / 32), 32 * kColWarps, 0, st>>>(w.part, chunks, bins, w.total);
  GM_CHECK_LAUNCH("radix_colscan_kernel");
  radix_coldown_kernel<<<col_grid, 256, 0, st>>>(w.table, tiles, bins, w.part);
  GM_CHECK_LAUNCH("radix_coldown_kernel");
  radix_digit_scan_kernel<<<1, 1024, 0, st>>>(w.total, bins, w.start);
  GM_CHECK_LAUNCH("radix_digit_scan_kernel");
  constexpr size_t smem = scatter_smem_bytes<BITS>();
  if (last) {
    GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<BITS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<BITS, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
    radix_scatter_kernel<BITS, true><<<static_cast<unsigned>(tiles), kThreads, smem, st>>>(in, e, shift, w.table,
                                                                                          w.start, ok, op, ov);
  } else {
    GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<BITS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<BITS, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
    radix_scatter_kernel<BITS, false><<<static_cast<unsigned>(tiles), kThreads, smem, st>>>(in, e, shift, w.table,
                                                                                           w.start, ok, op, ov);
  }
  GM_CHECK_LAUNCH("radix_scatter_kernel");
  return GM_OK;
}

template <bool LAST>
inline gm_status onesweep_pass(const In& in, int64_t e, int shift, const int32_t* start, unsigned long long* status,
                               int* ctr, uint32_t epoch, uint32_t* ok, uint32_t* op, uint32_t* ov, cudaStream_t st) {
  const int64_t tiles = ceil_div(e, kTile);
  constexpr size_t smem = scatter_smem_bytes<8>();
  auto kern = radix_scatter_kernel<8, LAST, true>;
  GM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  GM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  kern<<<static_cast<unsigned>(tiles), kThreads, smem, st>>>(in, e, shift, nullptr, start, ok, op, ov, status, ctr, epoch);
  GM_CHECK_LAUNCH("radix_scatter_kernel(onesweep)");
  return GM_OK;
}

// Full build: rowptr, col, perm. keys in [0, rows), values < 2^31.
inline gm_status radix_build(const int64_t* keys, const int64_t* values, int64_t e, int64_t rows, int64_t* rowptr,
                             int32_t* col, int32_t* perm, const RadixWs& w, cudaStream_t st) {
  const int bits = key_bits(rows);
  // widest digit (A/B knob GM_RADIX_BITS, 8 or 11)
  // (C4: 3 passes of 8 bits 1.5 ms of scatter vs 2 passes of 11 bits 2.06 ms:
  // the 2048-digit tiles leave ~2-entry runs and 8x the ranking work)
  static const int max_bits = [] {
    const char* ev = getenv("GM_RADIX_BITS");
    return ev && atoi(ev) == 11 ? kMaxBits : 8;
  }();
  const int passes = (bits + max_bits - 1) / max_bits;
  const int dbits = (bits + passes - 1) / passes;  // <= 11
  In in{keys, values, nullptr, nullptr, nullptr};
  int cur = 0;
  uint32_t* last_keys = nullptr;
  // one-sweep passes, an A/B variant (GM_CSR_ONESWEEP=1): bit-identical, but C4
  // builds in 2.57 ms vs 1.95 — each scatter pass 0.77-0.81 ms instead of 0.41-0.55
  // (the look-back over ~30k 2048-entry tiles serialises the tiles' offset
  // resolution), and the 3-digit global histogram takes 132 us of shared-memory
  // atomics against ~60 us per per-pass histogram
  static const bool onesweep = [] { const char* ev = getenv("GM_CSR_ONESWEEP"); return ev && ev[0] == '1'; }();
  if (onesweep && dbits <= 8 && passes <= 4) {
    const int64_t tiles = ceil_div(e, kTile);
    auto* status = reinterpret_cast<unsigned long long*>(w.table);  // [tiles][256] (the table holds 2048 x 4 B per tile)
    int* ctr = w.part;                                                 // [passes] tile counters
    GM_TRY_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * 256 * static_cast<size_t>(tiles), st));
    GM_TRY_CUDA(cudaMemsetAsync(w.total, 0, sizeof(int32_t) * 256 * passes, st));
    GM_TRY_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int) * passes, st));
    const unsigned hgrid = static_cast<unsigned>(std::min<int64_t>(ceil_div(e, 256 * 16), kNumSMs * 8));
    radix_global_hist_kernel<<<std::max(hgrid, 1u), 256, 0, st>>>(keys, e, passes, dbits, w.total);
    GM_CHECK_LAUNCH("radix_global_hist_kernel");
    for (int ps = 0; ps < passes; ++ps) {
      radix_digit_scan_kernel<<<1, 1024, 0, st>>>(w.total + ps * 256, 256, w.start + ps * 256);
      GM_CHECK_LAUNCH("radix_digit_scan_kernel");
    }
    for (int ps = 0; ps < passes; ++ps) {
      const bool last = ps == passes - 1;
      uint32_t* ok = w.buf[cur][0];
      uint32_t* op = last ? reinterpret_cast<uint32_t*>(perm) : w.buf[cur][1];
      uint32_t* ov = last ? reinterpret_cast<uint32_t*>(col) : w.buf[cur][2];
      const gm_status s = last ? onesweep_pass<true>(in, e, ps * dbits, w.start + ps * 256, status, ctr + ps, ps, ok, op, ov, st)
                               : onesweep_pass<false>(in, e, ps * dbits, w.start + ps * 256, status, ctr + ps, ps, ok, op, ov, st);
      if (s != GM_OK) return s;
      in = In{nullptr, nullptr, ok, op, ov};
      last_keys = ok;
      cur ^= 1;
    }
    rowptr_from_sorted_kernel<<<static_cast<unsigned>(ceil_div((e + kRowptrPer) / kRowptrPer, 256)), 256, 0, st>>>(
        last_keys, e, rows, rowptr);
    GM_CHECK_LAUNCH("rowptr_from_sorted_kernel");
    return GM_OK;
  }
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * dbits;
    const bool last = ps == passes - 1;
    uint32_t* ok = w.buf[cur][0];
    uint32_t* op = last ? reinterpret_cast<uint32_t*>(perm) : w.buf[cur][1];
    uint32_t* ov = last ? reinterpret_cast<uint32_t*>(col) : w.buf[cur][2];
    const gm_status s = dbits <= 8 ? radix_pass<8>(in, e, shift, last, w, ok, op, ov, st)
                                   : radix_pass<11>(in, e, shift, last, w, ok, op, ov, st);
    if (s != GM_OK) return s;
    in = In{nullptr, nullptr, ok, op, ov};
    last_keys = ok;
    cur ^= 1;
  }
  rowptr_from_sorted_kernel<<<static_cast<unsigned>(ceil_div((e + kRowptrPer) / kRowptrPer, 256)), 256, 0, st>>>(
      last_keys, e, rows, rowptr);
  GM_CHECK_LAUNCH("rowptr_from_sorted_kernel");
  return GM_OK;
}

}  // namespace rx
}  // namespace gm
