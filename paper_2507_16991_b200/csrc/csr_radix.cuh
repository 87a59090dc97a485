// csr_radix.cuh — build_compressed (edge_index.cpp:45-62) as a least-
// significant-digit radix sort of (key, COO position, value) triples (included
// by csr_build.cu).
//
// The reference is a stable counting sort by key: within a row, entries keep
// ascending COO position. An LSD radix sort whose every pass is stable yields
// exactly that order, so col / perm come out bit-identical to the reference
// for any input. Per pass (8-bit digit, 4096-entry tiles of 8 warps):
//   1. radix_hist: per-tile digit counts -> table[digit][tile];
//   2. exclusive scan of the table (digit-major) = each (digit, tile) run's
//      first output slot;
//   3. radix_scatter: every warp ranks its 512 entries round by round
//      (ballot multisplit: one ballot per digit bit, per-warp u16 counters), a
//      per-digit prefix over warps and over digits gives each entry's slot in a
//      digit-sorted copy of the tile in shared memory, and the tile leaves as
//      contiguous digit runs (coalesced stores, ~16 entries per run).
// rowptr comes from the sorted keys of the last pass (row boundaries), so no
// atomics anywhere: the result does not depend on scheduling.
#pragma once

namespace gm {
namespace rx {

constexpr int kBits = 8;
constexpr int kBins = 1 << kBits;
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // 4096 entries

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
  return in.keys64 ? static_cast<uint32_t>(in.keys64[i]) : __ldcs(in.key + i);
}

__global__ void __launch_bounds__(kThreads) radix_hist_kernel(In in, int64_t e, int shift, int64_t tiles,
                                                              int32_t* __restrict__ table) {
  __shared__ int32_t hist[kBins];
  const int64_t t = blockIdx.x;
  hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = t * kTile;
  const int64_t end = min(e, base + kTile);
  for (int64_t i = base + threadIdx.x; i < end; i += kThreads)
    atomicAdd(&hist[(key_at(in, i) >> shift) & (kBins - 1)], 1);
  __syncthreads();
  table[static_cast<int64_t>(threadIdx.x) * tiles + t] = hist[threadIdx.x];
}

// LAST: write perm / col (int32) and the sorted keys (for rowptr) instead of
// the next pass's triples.
template <bool LAST>
__global__ void __launch_bounds__(kThreads) radix_scatter_kernel(In in, int64_t e, int shift, int64_t tiles,
                                                                 const int32_t* __restrict__ table_off,
                                                                 uint32_t* __restrict__ okey, uint32_t* __restrict__ opos,
                                                                 uint32_t* __restrict__ oval) {
  __shared__ uint16_t whist[kWarps][kBins];
  __shared__ int32_t dstart[kBins + 1];
  __shared__ int32_t gout[kBins];
  __shared__ int32_t wsum[kWarps];
  extern __shared__ uint32_t stage[];  // digit-sorted tile: key, position, value
  uint32_t* skey = stage;
  uint32_t* spos = stage + kTile;
  uint32_t* sval = stage + 2 * kTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = blockIdx.x;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&whist[0][0])[i] = 0;
  gout[threadIdx.x] = table_off[static_cast<int64_t>(threadIdx.x) * tiles + t];
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
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    const bool valid = wbase + j * 32 + lane < e;
    const uint32_t d = (k[j] >> shift) & (kBins - 1);
    const unsigned peers = digit_peers<kBits>(d, valid);
    uint16_t old = 0;
    if (valid) old = whist[w][d];
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[w][d] = static_cast<uint16_t>(old + __popc(peers));
    __syncwarp();
    rank[j] = static_cast<uint16_t>(old + __popc(peers & lt));
  }
  __syncthreads();
  // per digit (one per thread): prefix over warps, then exclusive scan over digits
  {
    const int d = threadIdx.x;
    int32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      const int32_t c = whist[ww][d];
      whist[ww][d] = static_cast<uint16_t>(run);
      run += c;
    }
    // block exclusive scan of the per-digit tile counts
    int32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int32_t before = 0;
    for (int ww = 0; ww < w; ++ww) before += wsum[ww];
    dstart[d] = before + inc - run;
    if (d == kBins - 1) dstart[kBins] = before + inc;
  }
  __syncthreads();
  // digit-sorted copy of the tile in shared memory
#pragma unroll
  for (int j = 0; j < kRounds; ++j) {
    if (wbase + j * 32 + lane < e) {
      const uint32_t d = (k[j] >> shift) & (kBins - 1);
      const int s = dstart[d] + whist[w][d] + rank[j];
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
      __stcs(okey + o, key);
      __stcs(opos + o, spos[s]);
      __stcs(oval + o, sval[s]);
    }
  }
}

// rowptr from the sorted keys: rowptr[r] = first slot with key >= r. Each
// thread owns 4 consecutive slots (one 16-byte load + the previous key).
__global__ void rowptr_from_sorted_kernel(const uint32_t* __restrict__ key, int64_t e, int64_t rows,
                                          int64_t* __restrict__ rowptr) {
  const int64_t quads = (e + 4) / 4;  // slots 0..e (slot e closes the last rows)
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < quads;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k0 = q * 4;
    int64_t kk[5];
    kk[0] = k0 == 0 ? -1 : static_cast<int64_t>(key[k0 - 1]);
    if (k0 + 4 <= e && (reinterpret_cast<uintptr_t>(key + k0) & 15) == 0) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(key + k0));
      kk[1] = v.x;
      kk[2] = v.y;
      kk[3] = v.z;
      kk[4] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) kk[j + 1] = k0 + j < e ? static_cast<int64_t>(key[k0 + j]) : rows;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = k0 + j;
      if (k > e) break;
      for (int64_t r = kk[j] + 1; r <= kk[j + 1]; ++r) rowptr[r] = k;  // rows (prev, key[k]] start at k
    }
  }
}

struct RadixWs {
  int32_t* table;    // [kBins * tiles]
  int32_t* partial;  // scan block sums
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
  w.table = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(kBins * tiles)));
  w.partial = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(cb::scan32_blocks(kBins * tiles))));
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

// Full build: rowptr, col, perm. keys in [0, rows), values < 2^31.
inline gm_status radix_build(const int64_t* keys, const int64_t* values, int64_t e, int64_t rows, int64_t* rowptr,
                             int32_t* col, int32_t* perm, const RadixWs& w, cudaStream_t st) {
  const int64_t tiles = ceil_div(e, kTile);
  const int passes = (key_bits(rows) + kBits - 1) / kBits;
  In in{keys, values, nullptr, nullptr, nullptr};
  int cur = 0;
  uint32_t* last_keys = nullptr;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * kBits;
    radix_hist_kernel<<<static_cast<unsigned>(tiles), kThreads, 0, st>>>(in, e, shift, tiles, w.table);
    GM_CHECK_LAUNCH("radix_hist_kernel");
    gm_status s = cb::scan32_exclusive(w.table, kBins * tiles, w.partial, st);
    if (s != GM_OK) return s;
    const bool last = ps == passes - 1;
    uint32_t* ok = w.buf[cur][0];
    uint32_t* op = last ? reinterpret_cast<uint32_t*>(perm) : w.buf[cur][1];
    uint32_t* ov = last ? reinterpret_cast<uint32_t*>(col) : w.buf[cur][2];
    constexpr size_t stage_bytes = 3 * kTile * sizeof(uint32_t);
    if (last) {
      GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(stage_bytes)));
      radix_scatter_kernel<true><<<static_cast<unsigned>(tiles), kThreads, stage_bytes, st>>>(in, e, shift, tiles,
                                                                                             w.table, ok, op, ov);
    } else {
      GM_TRY_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(stage_bytes)));
      radix_scatter_kernel<false><<<static_cast<unsigned>(tiles), kThreads, stage_bytes, st>>>(in, e, shift, tiles,
                                                                                              w.table, ok, op, ov);
    }
    GM_CHECK_LAUNCH("radix_scatter_kernel");
    in = In{nullptr, nullptr, ok, op, ov};
    last_keys = ok;
    cur ^= 1;
  }
  rowptr_from_sorted_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div((e + 4) / 4, 256), kNumSMs * 64)), 256,
                              0, st>>>(last_keys, e, rows, rowptr);
  GM_CHECK_LAUNCH("rowptr_from_sorted_kernel");
  return GM_OK;
}

}  // namespace rx
}  // namespace gm
