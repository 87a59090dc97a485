// segment_matmul.cu — grouped GEMM over node-type segments on 5th-gen tensor
// cores (tcgen05 / TMEM / TMA), sm_100a.
//
// Replaces grouped_matmul (hetero.hpp:134-157): for each group g,
//   out[ptr[g]:ptr[g+1], :] = x[ptr[g]:ptr[g+1], :] @ W[g]        (W: [G, K, N])
// bf16 operands, fp32 accumulation in TMEM, bf16 or fp32 output.
//
// Structure (persistent, one CTA per SM, 6 warps):
//   warp 0  TMA producer: A k-blocks (128 rows x 64 k, SWIZZLE_128B) into an
//           S-stage ring; W^T[g] either resident (loaded once per group run)
//           or streamed per k-block when it does not fit.
//   warp 1  TMEM allocator + single-thread MMA issuer: tcgen05.mma
//           kind::f16, M=128, N=BN, K=16 steps; tcgen05.commit releases smem
//           stages and signals the epilogue. Two TMEM accumulators so the
//           epilogue of tile i overlaps the MMAs of tile i+1.
//   warps 2-5 epilogue: tcgen05.ld 32x32b (each warp its TMEM lane quarter =
//           32 output rows), convert, 16-byte stores of whole row segments;
//           rows past the group end are masked (tiles never straddle groups).
// Tiles: (group, 128-row m-tile, BN-column n-tile), group-major, assigned
// round-robin to CTAs, so each CTA sees groups in non-decreasing order.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "gm_common.cuh"

namespace gm {
namespace gmm {

constexpr int kMaxGroups = 128;
constexpr int BM = 128;          // UMMA M (cta_group::1)
constexpr int BK = 64;           // k elements per stage (128 B rows, SWIZZLE_128B)
constexpr int kEpiWarps = 8;     // two per TMEM lane quarter, each half the tile's columns
constexpr int kThreads = 64 + 32 * kEpiWarps;  // producer + MMA warps + epilogue
constexpr uint32_t kAStageBytes = BM * BK * 2;  // 16 KB
constexpr uint32_t kCBoxBytes = 32 * 128;       // 32 rows x 128 B
constexpr uint32_t kCStageBytes = kEpiWarps * kCBoxBytes;  // one 4 KB staging box per epilogue warp = 32 KB
#ifndef GM_CVT_WARPS
#define GM_CVT_WARPS 8
#endif
constexpr int kCvtWarps = GM_CVT_WARPS;     // fp32 split path: warps converting x tiles into bf16 pieces in smem

// Pointer-array mode (grouped_matmul over separate tensors, hetero.hpp:134-157):
// one TMA map per group for x and for out, rows addressed group-locally.
constexpr int kMaxPtrGroups = 8;
struct GroupMaps {
  CUtensorMap a[kMaxPtrGroups];
  CUtensorMap c[kMaxPtrGroups];
  void* out[kMaxPtrGroups];
};

struct Params {
  int64_t ptr[kMaxGroups + 1];        // group row offsets
  int32_t tile_start[kMaxGroups + 1]; // first m-tile id of each group (n-tiles folded in)
  int32_t groups;
  int32_t num_tiles;
  int32_t n_tiles;                    // BN-wide column tiles
  int32_t k_blocks;                   // K / 64
  int32_t n;                          // total output columns
  int32_t bn;                         // columns per tile (<= 256)
  int32_t out_f32;
  int32_t stages;
  int32_t b_resident;
  int32_t tma_store;                  // full tiles leave through TMA bulk stores
  uint32_t tmem_cols;
  // A operand as segments of a narrower matrix (fp32 split path): K' k-block
  // coordinate kc reads column (seg_map[kc / a_seg_k]) * a_seg_k + kc % a_seg_k
  // of x; 2 bits per segment. a_seg_k == 0: identity.
  int32_t a_seg_k;
  uint32_t a_seg_map;
  // fused fp32 split (SPLIT kernels): x [rows, a_ld] fp32 read by the
  // converter warps; a_seg_k = padded K (piece stride of the W pieces)
  const float* a_f32;
  int32_t a_ld;
  int32_t x_stages;                   // SPLIT: fp32 x staging ring depth
  // fp32-accurate split (CVT = 3): acc_sets > 0 keeps the hi*hi product and
  // the five correction products in separate TMEM accumulators and spreads
  // the k-blocks round-robin over acc_sets such pairs, summed in the
  // epilogue: each fp32 accumulator sees ~1/(6 acc_sets) of the MMA steps, so
  // the tensor pipe's per-step accumulation error grows that much slower.
  int32_t acc_sets;
  int32_t acc_cols;                   // TMEM columns per double-buffer slot
  int32_t ptr_groups;                 // 1: x / out per group (GroupMaps), rows group-local
  void* out;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major, SWIZZLE_128B smem matrix descriptor: 8-row x 128-byte atoms,
// atoms 1024 B apart (SBO), LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// K-major, SWIZZLE_64B: 8-row x 64-byte atoms, 512 B apart (SBO), layout 4.
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}
template <int KBLK>
__device__ __forceinline__ uint64_t sdesc_k(uint32_t saddr) {
  if constexpr (KBLK == 64) return sdesc_sw128(saddr);
  else return sdesc_sw64(saddr);
}
// Instruction descriptor: bf16 x bf16 -> f32, both K-major, M=128, N=bn.
__device__ __forceinline__ uint32_t idesc_bf16(int bn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(bn >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void decode_tile(const Params& P, int t, int& g, int& mt, int& nt) {
  g = 0;
  while (g + 1 < P.groups && P.tile_start[g + 1] <= t) ++g;
  const int local = t - P.tile_start[g];
  mt = local / P.n_tiles;
  nt = local - mt * P.n_tiles;
}

template <int CHUNK>
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v);
template <>
__device__ __forceinline__ void tmem_ld32<32>(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld32<16>(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void st_na_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo_f32, uint32_t hi_f32) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo_f32), __uint_as_float(hi_f32));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// KBLK: k elements per pipeline stage — 64 (128-byte rows, SWIZZLE_128B) or 32
// (64-byte rows, SWIZZLE_64B: twice the stages for the same bytes in flight,
// each released after half the MMAs).
// fp32 -> three bf16 pieces (see kSplit below) for two values at once:
// hi = bf16(v), mid = bf16(v - hi), lo = bf16(v - hi - mid), the subtractions
// exact; one bf16x2 cvt per piece pair, halves widened back by shift / mask.
__device__ __forceinline__ void split3x2(float a, float b, uint32_t& hw, uint32_t& mw, uint32_t& lw) {
  hw = pack_bf16(__float_as_uint(a), __float_as_uint(b));
  const float ra = __fsub_rn(a, __uint_as_float(hw << 16)), rb = __fsub_rn(b, __uint_as_float(hw & 0xffff0000u));
  mw = pack_bf16(__float_as_uint(ra), __float_as_uint(rb));
  lw = pack_bf16(__float_as_uint(__fsub_rn(ra, __uint_as_float(mw << 16))),
                 __float_as_uint(__fsub_rn(rb, __uint_as_float(mw & 0xffff0000u))));
}

// SPLIT: fp32 operands at fp32 accuracy with the split fused into the kernel.
// The producer TMA-loads each fp32 x tile ONCE into a staging ring; kCvtWarps
// converter warps turn it into hi/mid/lo bf16 pieces in three swizzled smem
// buffers of the MMA stage, and the MMA issuer forms the six products hi*hi + hi*mid + mid*hi +
// hi*lo + lo*hi + mid*mid against the matching W pieces (K-major [G*N, 3*Kp]).
// CVT = 1: the same converter path with a single piece (fp32 x rounded to bf16
// in the kernel, bf16 W): x is read once as fp32 instead of a separate cast pass.
// SPLITACC: the split-accumulator variant (P.acc_sets > 0) is its own
// instantiation, so the single-accumulator epilogue carries none of its
// registers (the shared form spilled 120 B per thread).
template <int KBLK, int CVT, bool SPLITACC = false>
__global__ void __launch_bounds__(CVT > 0 ? kThreads + 32 * kCvtWarps : kThreads, 1)
segment_matmul_kernel(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_c,
                      const __grid_constant__ GroupMaps G) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B alignment for the SWIZZLE_128B atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = P.stages;
  constexpr bool SPLIT = CVT > 0;           // x arrives as fp32 through the converter warps
  constexpr int kPieces = CVT == 3 ? 3 : 1;  // bf16 pieces per operand
  const uint32_t b_kblock_bytes = static_cast<uint32_t>(P.bn) * KBLK * 2;
  constexpr uint32_t kAStage = BM * KBLK * 2;  // one piece
  constexpr uint32_t kXStage = BM * KBLK * 4;  // SPLIT: one fp32 x tile
  const int SX = SPLIT ? P.x_stages : 0;
  unsigned char* a_ring = smem;
  unsigned char* x_ring = smem + static_cast<size_t>(S) * kPieces * kAStage;
  unsigned char* b_buf = x_ring + static_cast<size_t>(SX) * kXStage;
  const size_t b_bytes = P.b_resident ? static_cast<size_t>(kPieces) * P.k_blocks * b_kblock_bytes
                                      : static_cast<size_t>(S) * kPieces * b_kblock_bytes;
  // output staging: per epilogue warp two 32-row x 128-byte SWIZZLE_128B boxes
  unsigned char* c_stage = b_buf + b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(c_stage + kCStageBytes);
  uint64_t* full = bars;              // [S]
  uint64_t* empty = bars + S;         // [S]
  uint64_t* tfull = bars + 2 * S;     // [2]
  uint64_t* tempty = bars + 2 * S + 2;// [2]
  uint64_t* bfull = bars + 2 * S + 4;
  uint64_t* bempty = bars + 2 * S + 5;
  uint64_t* xfull = bars + 2 * S + 6;       // [SX]
  uint64_t* xempty = bars + 2 * S + 6 + SX; // [SX]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6 + 2 * SX);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // SPLIT: each converter warp (+ the producer's W bytes when W streams)
      mbar_init(&full[s], SPLIT ? kCvtWarps + (P.b_resident ? 0 : 1) : 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < SX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], kCvtWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int cur_g = -1;
      uint32_t nbload = 0;
      int sx = 0;
      uint32_t xph = 0;
      for (int t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
        int g, mt, nt;
        decode_tile(P, t, g, mt, nt);
        // A rows: global (one matrix) or group-local (pointer-array mode)
        const int row0 = P.ptr_groups ? mt * BM : static_cast<int>(P.ptr[g]) + mt * BM;
        const CUtensorMap* ma = P.ptr_groups ? &G.a[g] : &map_a;
        const int brow0 = g * P.n + nt * P.bn;
        if (P.b_resident && g != cur_g) {
          if (nbload > 0) mbar_wait(bempty, (nbload - 1) & 1);
          mbar_expect_tx(bfull, static_cast<uint32_t>(kPieces * P.k_blocks) * b_kblock_bytes);
          for (int pc = 0; pc < kPieces; ++pc)
            for (int kb = 0; kb < P.k_blocks; ++kb)
              tma_load_2d(b_buf + static_cast<size_t>(pc * P.k_blocks + kb) * b_kblock_bytes, &map_b, bfull,
                          pc * P.a_seg_k + kb * KBLK, brow0);
          cur_g = g;
          ++nbload;
        }
        for (int kb = 0; kb < P.k_blocks; ++kb) {
          if constexpr (SPLIT) {
            // fp32 x tile -> staging ring (rows / columns past the end read as zero)
            mbar_wait(&xempty[sx], xph ^ 1);
            mbar_expect_tx(&xfull[sx], kXStage);
            tma_load_2d(x_ring + static_cast<size_t>(sx) * kXStage, ma, &xfull[sx], kb * KBLK, row0);
            if (++sx == SX) {
              sx = 0;
              xph ^= 1;
            }
            if (P.b_resident) continue;
            // streamed W pieces for this k-block
            mbar_wait(&empty[s], ph ^ 1);
            {
              mbar_expect_tx(&full[s], kPieces * b_kblock_bytes);
              for (int pc = 0; pc < kPieces; ++pc)
                tma_load_2d(b_buf + static_cast<size_t>(s * kPieces + pc) * b_kblock_bytes, &map_b, &full[s],
                            pc * P.a_seg_k + kb * KBLK, brow0);
            }
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          mbar_wait(&empty[s], ph ^ 1);
          if (P.b_resident) {
            mbar_expect_tx(&full[s], kAStage);
          } else {
            mbar_expect_tx(&full[s], kAStage + b_kblock_bytes);
            tma_load_2d(b_buf + static_cast<size_t>(s) * b_kblock_bytes, &map_b, &full[s], kb * KBLK, brow0);
          }
          int ac = kb * KBLK;
          if (P.a_seg_k > 0) {
            const int seg = ac / P.a_seg_k;
            ac += (static_cast<int>((P.a_seg_map >> (2 * seg)) & 3u) - seg) * P.a_seg_k;
          }
          tma_load_2d(a_ring + static_cast<size_t>(s) * kAStage, ma, &full[s], ac, row0);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16(P.bn);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph = 0;
    int cur_g = -1;
    uint32_t nbwait = 0;
    for (int t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
      int g, mt, nt;
      decode_tile(P, t, g, mt, nt);
      if (P.b_resident && g != cur_g) {
        mbar_wait(bfull, nbwait & 1);
        ++nbwait;
        cur_g = g;
      }
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * P.acc_cols);
      for (int kb = 0; kb < P.k_blocks; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (SPLIT && lane == 0) {
          const uint32_t a_addr = smem_u32(a_ring + static_cast<size_t>(s) * kPieces * kAStage);
          uint32_t b_addr[3] = {0u, 0u, 0u};
#pragma unroll
          for (int pc = 0; pc < kPieces; ++pc)
            b_addr[pc] = P.b_resident
                             ? smem_u32(b_buf + static_cast<size_t>(pc * P.k_blocks + kb) * b_kblock_bytes)
                             : smem_u32(b_buf + static_cast<size_t>(s * kPieces + pc) * b_kblock_bytes);
          // (x piece, W piece): hi*hi, hi*mid, mid*hi, hi*lo, lo*hi, mid*mid
          constexpr int kPa[6] = {0, 0, 1, 0, 2, 1};
          constexpr int kPb[6] = {0, 1, 0, 2, 0, 1};
          constexpr int kPairs = CVT == 3 ? 6 : 1;
          if (SPLITACC && CVT == 3 && P.acc_sets > 0) {
            // set kb % R: columns [2 set, 2 set + 1) * bn hold (hi*hi, corrections)
            const int set = kb % P.acc_sets;
            const bool first_use = kb < P.acc_sets;
            const uint32_t d_main = tmem_d + static_cast<uint32_t>(2 * set * P.bn);
            const uint32_t d_corr = d_main + static_cast<uint32_t>(P.bn);
#pragma unroll
            for (int pr = 0; pr < kPairs; ++pr)
#pragma unroll
              for (int k = 0; k < KBLK / 16; ++k)
                tc_mma(pr == 0 ? d_main : d_corr, sdesc_k<KBLK>(a_addr + kPa[pr] * kAStage + k * 32),
                       sdesc_k<KBLK>(b_addr[kPb[pr]] + k * 32), idesc,
                       (!first_use || k > 0 || pr > 1) ? 1u : 0u);
          } else {
#pragma unroll
            for (int pr = 0; pr < kPairs; ++pr)
#pragma unroll
              for (int k = 0; k < KBLK / 16; ++k)
                tc_mma(tmem_d, sdesc_k<KBLK>(a_addr + kPa[pr] * kAStage + k * 32),
                       sdesc_k<KBLK>(b_addr[kPb[pr]] + k * 32), idesc, (kb > 0 || pr > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        } else if (!SPLIT && lane == 0) {
          const uint32_t a_addr = smem_u32(a_ring + static_cast<size_t>(s) * kAStage);
          const uint32_t b_addr = P.b_resident ? smem_u32(b_buf + static_cast<size_t>(kb) * b_kblock_bytes)
                                               : smem_u32(b_buf + static_cast<size_t>(s) * b_kblock_bytes);
          uint32_t d = tmem_d;
          bool fresh = kb == 0;
          if (SPLITACC && CVT == 0 && P.acc_sets > 0) {
            // staged fp32 split: k-blocks of segment 0 (hi*hi) -> main sets,
            // segments 1..5 (corrections) -> correction sets
            const int segb = P.a_seg_k / KBLK;
            const int part = kb >= segb ? 1 : 0;
            const int kk = part ? kb - segb : kb;
            d = tmem_d + static_cast<uint32_t>((2 * (kk % P.acc_sets) + part) * P.bn);
            fresh = kk < P.acc_sets;
          }
#pragma unroll
          for (int k = 0; k < KBLK / 16; ++k) {
            // advancing 16 bf16 = 32 B inside the swizzle atom
            tc_mma(d, sdesc_k<KBLK>(a_addr + k * 32), sdesc_k<KBLK>(b_addr + k * 32), idesc,
                   (!fresh || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);  // smem stage free once these MMAs retire
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (lane == 0) {
        tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (P.b_resident) {
          const int tn = t + static_cast<int>(gridDim.x);
          int g2 = -1, m2, n2;
          if (tn < P.num_tiles) decode_tile(P, tn, g2, m2, n2);
          if (g2 != g) tc_commit(bempty);  // W^T[g] no longer read by this CTA
        }
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const bool out_f32 = SPLIT || P.out_f32 != 0;  // SPLIT writes fp32
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int esz = out_f32 ? 4 : 2;
    const int chunk_cols = 128 / esz;  // columns per 128-byte TMA box
    unsigned char* my_stage = c_stage + static_cast<size_t>(warp - 2) * kCBoxBytes;
    // the two warps of a quarter split the columns; a tile too narrow to split
    // (half not a multiple of the TMA box / 16-column loads) stays on half 0
    const int half = (warp - 2) >> 2;
    const bool split = (P.bn / 2) % chunk_cols == 0 && (P.bn / 2) % 16 == 0;
    const int c_lo = split ? half * (P.bn / 2) : 0;
    const int c_hi = split ? c_lo + P.bn / 2 : (half == 0 ? P.bn : 0);
    int acc = 0;
    uint32_t aph = 0;
    int nstore = 0;
    for (int t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
      int g, mt, nt;
      decode_tile(P, t, g, mt, nt);
      const int64_t grow_end = P.ptr[g + 1];
      const int64_t row0 = P.ptr[g] + static_cast<int64_t>(mt) * BM;
      const int64_t row = row0 + q * 32 + lane;
      const bool full_tile = P.tma_store && row0 + BM <= grow_end;  // else: masked direct stores
      // output rows: global, or group-local in pointer-array mode
      const CUtensorMap* mc = P.ptr_groups ? &G.c[g] : &map_c;
      const int64_t orow0 = P.ptr_groups ? static_cast<int64_t>(mt) * BM : row0;
      void* const obase = P.ptr_groups ? G.out[g] : P.out;
      const int64_t orow = orow0 + q * 32 + lane;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * P.acc_cols);
      // split accumulators: (sum of the hi*hi sets) + (sum of the correction sets), fp32 RN
      auto load_cols = [&](uint32_t col, uint32_t* v, auto width_c) {
        constexpr int W = decltype(width_c)::value;
        if (!SPLITACC || CVT == 1 || P.acc_sets == 0) {
          tmem_ld32<W>(tbase + col, v);
          tmem_wait_ld();
          return;
        }
        // 16 columns at a time keeps the partial sums in registers
#pragma unroll
        for (int h = 0; h < W; h += 16) {
          uint32_t* vh = v + h;
          uint32_t t[16];
          float corr[16];
          tmem_ld32<16>(tbase + col + h, vh);
          tmem_ld32<16>(tbase + static_cast<uint32_t>(P.bn) + col + h, t);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) corr[i] = __uint_as_float(t[i]);
          for (int set = 1; set < P.acc_sets; ++set) {
            tmem_ld32<16>(tbase + static_cast<uint32_t>(2 * set * P.bn) + col + h, t);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) vh[i] = __float_as_uint(__fadd_rn(__uint_as_float(vh[i]), __uint_as_float(t[i])));
            tmem_ld32<16>(tbase + static_cast<uint32_t>((2 * set + 1) * P.bn) + col + h, t);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) corr[i] = __fadd_rn(corr[i], __uint_as_float(t[i]));
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) vh[i] = __float_as_uint(__fadd_rn(__uint_as_float(vh[i]), corr[i]));
        }
      };
      if (full_tile) {
        for (int c = c_lo; c < c_hi; c += chunk_cols) {
          if (SPLITACC && (CVT == 3 || (CVT == 0 && out_f32)) && P.acc_sets > 0) {
            // split accumulators: summed and staged 16 columns at a time
            if (lane == 0 && nstore >= 1) bulk_wait_read<0>();  // the previous store has read the box
            __syncwarp();
            const uint32_t sb = smem_u32(my_stage) + lane * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t part[16];
              load_cols(static_cast<uint32_t>(c + 16 * h), part, std::integral_constant<int, 16>{});
#pragma unroll
              for (int ch = 0; ch < 4; ++ch)
                st_shared_v4(sb + (((4 * h + ch) ^ (lane & 7)) << 4), part[4 * ch], part[4 * ch + 1],
                             part[4 * ch + 2], part[4 * ch + 3]);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(mc, my_stage, nt * P.bn + c, static_cast<int32_t>(orow0 + q * 32));
              bulk_commit();
            }
            ++nstore;
            continue;
          }
          // 128 bytes of this lane's row: 32 fp32 or 64 bf16 values
          uint32_t packed[32];
          if (out_f32) {
            load_cols(static_cast<uint32_t>(c), packed, std::integral_constant<int, 32>{});
          } else {
            uint32_t v[32];
            tmem_ld32<32>(tbase + c, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) packed[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
            tmem_ld32<32>(tbase + c + 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) packed[16 + i] = pack_bf16(v[2 * i], v[2 * i + 1]);
          }
          const int b = 0;
          if (lane == 0 && nstore >= 1) bulk_wait_read<0>();  // the previous store has read the box
          __syncwarp();
          const uint32_t sbase = smem_u32(my_stage + b * kCBoxBytes) + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)  // SWIZZLE_128B: 16-B chunk ch lands at ch ^ (row % 8)
            st_shared_v4(sbase + ((ch ^ (lane & 7)) << 4), packed[4 * ch], packed[4 * ch + 1], packed[4 * ch + 2],
                         packed[4 * ch + 3]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(mc, my_stage + b * kCBoxBytes, nt * P.bn + c, static_cast<int32_t>(orow0 + q * 32));
            bulk_commit();
          }
          ++nstore;
        }
      } else {
        const bool live = row < grow_end;
        for (int c = c_lo; c < c_hi; c += 16) {  // bn is a multiple of 16
          uint32_t v[16];
          load_cols(static_cast<uint32_t>(c), v, std::integral_constant<int, 16>{});
          if (live) {
            const int64_t col0 = static_cast<int64_t>(nt) * P.bn + c;
            if (out_f32) {
              float* o = static_cast<float*>(obase) + orow * P.n + col0;
#pragma unroll
              for (int i = 0; i < 16; i += 4) st_na_v4(o + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
              __nv_bfloat16* o = static_cast<__nv_bfloat16*>(obase) + orow * P.n + col0;
#pragma unroll
              for (int i = 0; i < 16; i += 8)
                st_na_v4(o + i, pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]),
                         pack_bf16(v[i + 4], v[i + 5]), pack_bf16(v[i + 6], v[i + 7]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();  // stores complete before the CTA exits
    __syncwarp();
  } else if constexpr (SPLIT) {
    // ------------------------------------------------------------ converters
    // unit u of a stage = 4 consecutive k of one row: 16 B of fp32 read from the
    // staging tile, 8 B of bf16 written per piece at its swizzled position;
    // consecutive lanes take consecutive units, so both sides are conflict-free
    constexpr int kUnits = KBLK / 4;  // per row
    constexpr int kPer = BM * kUnits / (32 * kCvtWarps);
    const int ct = (warp - 2 - kEpiWarps) * 32 + lane;
    int s = 0, sx = 0;
    uint32_t ph = 0, xph = 0;
    for (int t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
      for (int kb = 0; kb < P.k_blocks; ++kb) {
        mbar_wait(&xfull[sx], xph);
        const uint32_t xbase = smem_u32(x_ring + static_cast<size_t>(sx) * kXStage);
        float4 v[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const uint32_t a = xbase + static_cast<uint32_t>(ct + i * 32 * kCvtWarps) * 16;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[i].x), "=f"(v[i].y), "=f"(v[i].z), "=f"(v[i].w) : "r"(a));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[sx]);  // staging tile consumed
        if (++sx == SX) {
          sx = 0;
          xph ^= 1;
        }
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t base = smem_u32(a_ring + static_cast<size_t>(s) * kPieces * kAStage);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int u = ct + i * 32 * kCvtWarps;
          const int r = u / kUnits, q = u % kUnits;
          const int sw = KBLK == 64 ? (r & 7) : ((r >> 1) & 3);  // SWIZZLE_128B / SWIZZLE_64B
          const uint32_t off = static_cast<uint32_t>(r * KBLK * 2 + (((q >> 1) ^ sw) << 4) + (q & 1) * 8);
          if constexpr (CVT == 3) {
            uint32_t h0, m0, l0, h1, m1, l1;
            split3x2(v[i].x, v[i].y, h0, m0, l0);
            split3x2(v[i].z, v[i].w, h1, m1, l1);
            asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(base + off), "r"(h0), "r"(h1) : "memory");
            asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(base + kAStage + off), "r"(m0), "r"(m1) : "memory");
            asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(base + 2 * kAStage + off), "r"(l0), "r"(l1)
                         : "memory");
          } else {
            const uint32_t h0 = pack_bf16(__float_as_uint(v[i].x), __float_as_uint(v[i].y));
            const uint32_t h1 = pack_bf16(__float_as_uint(v[i].z), __float_as_uint(v[i].w));
            asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(base + off), "r"(h0), "r"(h1) : "memory");
          }
        }
        fence_async_smem();  // generic-proxy smem writes visible to tcgen05.mma
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(P.tmem_cols)
                 : "memory");
  }
}

// W[g] [K, N] row-major -> W^T [G*Np, Kp] (K-major B operand), zero-padded
__global__ void transpose_w_kernel(const __nv_bfloat16* __restrict__ w, int groups, int k, int n, int kp, int np,
                                   __nv_bfloat16* __restrict__ wt) {
  const int64_t total = static_cast<int64_t>(groups) * kp * np;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / (static_cast<int64_t>(np) * kp);
    const int64_t rem = i - g * np * kp;
    const int64_t nn = rem / kp;
    const int64_t kk = rem - nn * kp;
    wt[i] = (nn < n && kk < k) ? w[(g * k + kk) * n + nn] : __float2bfloat16_rn(0.f);
  }
}

// zero-padded copy of a row-major [rows, c] bf16 matrix into [rows, cp]
__global__ void pad_cols_kernel(const __nv_bfloat16* __restrict__ a, int64_t rows, int c, int cp,
                                __nv_bfloat16* __restrict__ b) {
  const int64_t total = rows * cp;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cp;
    const int64_t j = i - r * cp;
    b[i] = j < c ? a[r * c + j] : __float2bfloat16_rn(0.f);
  }
}
// [rows, np] -> [rows, n] (element size esz)
__global__ void unpad_cols_kernel(const unsigned char* __restrict__ a, int64_t rows, int n, int np, int esz,
                                  unsigned char* __restrict__ b) {
  const int64_t total = rows * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / n;
    const int64_t j = i - r * n;
    for (int e = 0; e < esz; ++e) b[i * esz + e] = a[(r * np + j) * esz + e];
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static gm_status make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                          uint32_t box_outer, CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          uint64_t esz = 2, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  GM_REQUIRE(fn, GM_ERR_CUDA, "segment_matmul: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * esz};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  GM_REQUIRE(r == CUDA_SUCCESS, GM_ERR_CUDA, "segment_matmul: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return GM_OK;
}

}  // namespace gmm
}  // namespace gm

using namespace gm;

static int64_t pad_to(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

namespace gm {
namespace gmm {

// fp32 operands as three bf16 pieces: hi = bf16(v), mid = bf16(v - hi),
// lo = bf16(v - hi - mid), |v - hi - mid - lo| <= 2^-27 |v|. Along K the
// operands are arranged so that ONE bf16 tcgen05 GEMM over K' = 6K with fp32
// TMEM accumulation forms the six products down to 2^-18 scale:
//   x' = [hi | hi | mid | hi | lo | mid],  W' = [hi; mid; hi; lo; hi; mid]
//   sum = hi*hi + hi*mid + mid*hi + hi*lo + lo*hi + mid*mid = x W + O(2^-26)|x||W|.
// x' is never materialised: x is split once into [hi | mid | lo] (3K wide,
// each piece zero-padded to a whole number of 64-deep k-blocks) and the
// producer's TMA coordinates walk the six segments over it (Params::a_seg_*),
// so the repeated pieces are re-read from L2 within a tile, not from HBM.
constexpr int kSplit = 6;
constexpr uint32_t kSplitSegMap = 0u | (0u << 2) | (1u << 4) | (0u << 6) | (2u << 8) | (1u << 10);
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  const float r1 = __fsub_rn(v, __bfloat162float(hi));  // exact (Sterbenz-range subtraction)
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(mid)));
}

// x [rows, k] fp32 -> pieces [rows, 3*kp] bf16, four columns per thread
// (8-byte stores per piece); columns k..kp-1 of every piece are zero.
__global__ void split_x_kernel(const float* __restrict__ x, int64_t rows, int k, int kp,
                               __nv_bfloat16* __restrict__ xs) {
  const int q = kp / 4;
  const int64_t total = rows * q;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / q;
    const int c = static_cast<int>(i - r * q) * 4;
    __align__(8) __nv_bfloat16 hi[4], mid[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float v = c + j < k ? __ldcs(x + r * k + c + j) : 0.f;
      split_bf16(v, hi[j], mid[j], lo[j]);
    }
    __nv_bfloat16* o = xs + r * 3 * kp + c;
    *reinterpret_cast<uint2*>(o) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(o + kp) = *reinterpret_cast<const uint2*>(mid);
    *reinterpret_cast<uint2*>(o + 2 * kp) = *reinterpret_cast<const uint2*>(lo);
  }
}

// w [G, k, n] fp32 -> W' [G, 6*kp, n] bf16 (rows k..kp-1 of each segment zero).
__global__ void split_w_kernel(const float* __restrict__ w, int groups, int k, int kp, int n,
                               __nv_bfloat16* __restrict__ ws) {
  const int64_t total = static_cast<int64_t>(groups) * kp * n;
  const int64_t kpn = static_cast<int64_t>(kp) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / kpn;
    const int64_t rem = i - g * kpn;  // kk * n + nn
    const int kk = static_cast<int>(rem / n);
    __nv_bfloat16 hi, mid, lo;
    split_bf16(kk < k ? w[g * k * n + rem] : 0.f, hi, mid, lo);
    __nv_bfloat16* o = ws + g * kSplit * kpn + rem;
    o[0] = hi;
    o[kpn] = mid;
    o[2 * kpn] = hi;
    o[3 * kpn] = lo;
    o[4 * kpn] = hi;
    o[5 * kpn] = mid;
  }
}

// w [G, k, n] fp32 -> K-major pieces [G*np, 3*kp] bf16 (hi | mid | lo along K),
// zero-padded: the B operand of the fused-split kernel.
__global__ void split_wt_kernel(const float* __restrict__ w, int groups, int k, int n, int kp, int np,
                                __nv_bfloat16* __restrict__ wt) {
  const int64_t total = static_cast<int64_t>(groups) * np * kp;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = i / (static_cast<int64_t>(np) * kp);
    const int64_t rem = i - g * np * kp;
    const int64_t nn = rem / kp;
    const int64_t kk = rem - nn * kp;
    __nv_bfloat16 hi, mid, lo;
    split_bf16((nn < n && kk < k) ? w[(g * k + kk) * n + nn] : 0.f, hi, mid, lo);
    __nv_bfloat16* o = wt + (g * np + nn) * 3 * kp + kk;
    o[0] = hi;
    o[kp] = mid;
    o[2 * kp] = lo;
  }
}

}  // namespace gmm
}  // namespace gm
using namespace gm::gmm;

extern "C" {

GM_API size_t gm_segment_matmul_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n) {
  if (rows < 0 || groups < 0 || k < 0 || n < 0) return 0;
  const int64_t kp = pad_to(std::max<int64_t>(k, 1), 64), np = pad_to(std::max<int64_t>(n, 1), 16);
  size_t b = align_up(static_cast<size_t>(groups * kp * np) * 2, 256);  // K-major W^T
  if (kp != k) b += align_up(static_cast<size_t>(rows * kp) * 2, 256);   // padded x
  if (np != n) b += align_up(static_cast<size_t>(rows * np) * 4, 256);   // padded out
  return b;
}

static gm_status segment_matmul_impl(const void* x, const int64_t* ptr_host, int64_t groups, int64_t k_in,
                                     int64_t n_in, const void* w, const void* w_packed, gm_dtype out_dtype, void* out,
                                     void* workspace, size_t workspace_bytes, gm_stream_t stream,
                                     int64_t a_seg_k = 0, uint32_t a_seg_map = 0, int64_t a_cols = 0,
                                     const float* a_f32 = nullptr, int64_t a_ld = 0, int a_pieces = 3,
                                     const void* const* gx = nullptr, void* const* gout = nullptr) {
  using namespace gm::gmm;
  GM_REQUIRE(ptr_host && groups >= 1 && groups <= kMaxGroups, GM_ERR_INVALID_ARGUMENT,
             "segment_matmul: groups must be in [1, " + std::to_string(kMaxGroups) + "]");
  GM_REQUIRE(k_in > 0 && n_in > 0, GM_ERR_INVALID_ARGUMENT, "segment_matmul: K and N must be positive");
  // odd shapes run zero-padded (K to 64, N to 16) through the workspace
  const int64_t k = pad_to(k_in, BK), n = pad_to(n_in, 16);
  GM_REQUIRE(out_dtype == GM_BF16 || out_dtype == GM_F32, GM_ERR_INVALID_ARGUMENT,
             "segment_matmul: out dtype must be bf16 or f32");
  GM_REQUIRE(ptr_host[0] == 0, GM_ERR_INVALID_ARGUMENT, "segment_matmul: ptr[0] must be 0");
  for (int64_t g = 0; g < groups; ++g)
    GM_REQUIRE(ptr_host[g + 1] >= ptr_host[g], GM_ERR_INVALID_ARGUMENT, "segment_matmul: ptr must be non-decreasing");
  const int64_t rows = ptr_host[groups];
  GM_REQUIRE(rows < INT32_MAX, GM_ERR_INVALID_ARGUMENT, "segment_matmul: too many rows");
  if (rows == 0) return GM_OK;
  GM_REQUIRE(x && (w || w_packed) && out, GM_ERR_INVALID_ARGUMENT, "segment_matmul: null pointer");
  const size_t wt_bytes = w_packed ? 0 : align_up(static_cast<size_t>(groups * k * n) * 2, 256);
  const size_t need = gm_segment_matmul_workspace(rows, groups, k_in, n_in) -
                      align_up(static_cast<size_t>(groups * k * n) * 2, 256) + wt_bytes;
  GM_REQUIRE(need == 0 || (workspace && workspace_bytes >= need), GM_ERR_INVALID_ARGUMENT,
             "segment_matmul: workspace too small");
  cudaStream_t st = as_stream(stream);
  unsigned char* wsp = static_cast<unsigned char*>(workspace);
  __nv_bfloat16* wt = w_packed ? static_cast<__nv_bfloat16*>(const_cast<void*>(w_packed))
                               : reinterpret_cast<__nv_bfloat16*>(wsp);
  wsp += wt_bytes;
  const void* xk = x;
  if (k != k_in) {
    __nv_bfloat16* xp = reinterpret_cast<__nv_bfloat16*>(wsp);
    wsp += align_up(static_cast<size_t>(rows * k) * 2, 256);
    pad_cols_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(rows * k, 256), 8192)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), rows, static_cast<int>(k_in), static_cast<int>(k), xp);
    GM_CHECK_LAUNCH("pad_cols_kernel");
    xk = xp;
  }
  const size_t esz = out_dtype == GM_F32 ? 4 : 2;
  void* outk = out;
  if (n != n_in) {
    outk = wsp;
    wsp += align_up(static_cast<size_t>(rows * n) * 4, 256);
  }
  GM_REQUIRE((reinterpret_cast<uintptr_t>(xk) | reinterpret_cast<uintptr_t>(outk)) % 16 == 0,
             GM_ERR_INVALID_ARGUMENT, "segment_matmul: x and out must be 16-byte aligned");
  const bool ptr_mode = gx != nullptr;
  GM_REQUIRE(!ptr_mode || (gout && groups <= kMaxPtrGroups && k == k_in && n == n_in && a_seg_k == 0),
             GM_ERR_INVALID_ARGUMENT, "segment_matmul: pointer-array groups need <= 8 groups and unpadded shapes");

  Params P{};
  P.groups = static_cast<int32_t>(groups);
  P.bn = static_cast<int32_t>(std::min<int64_t>(n, 256));
  while (n % P.bn != 0) P.bn -= 16;
  P.n_tiles = static_cast<int32_t>(n / P.bn);
  // 64-deep k-blocks (SWIZZLE_128B). 32-deep blocks (SWIZZLE_64B, twice the
  // stages) measured slower at F=2048 (1.41 vs 1.11 PFLOP/s); GM_GEMM_KBLK=32
  // selects them for experiments.
  static const int kblk_env = [] { const char* e = getenv("GM_GEMM_KBLK"); return e ? atoi(e) : 0; }();
  // the fused fp32 split path runs 32-deep blocks: three bf16 pieces + an fp32
  // staging tile per stage leave room for 3-4 stages only at that depth
  const int kblk = (kblk_env == 32 || (a_f32 && kblk_env != 64)) ? 32 : 64;
  P.k_blocks = static_cast<int32_t>(k / kblk);
  P.n = static_cast<int32_t>(n);
  P.out_f32 = out_dtype == GM_F32;
  P.out = outk;
  P.ptr_groups = ptr_mode ? 1 : 0;
  P.tma_store = (P.bn % (128 / static_cast<int>(out_dtype == GM_F32 ? 4 : 2))) == 0 ? 1 : 0;
  P.a_seg_k = static_cast<int32_t>(a_f32 ? k : a_seg_k);
  P.a_seg_map = a_seg_map;
  P.a_f32 = a_f32;
  P.a_ld = static_cast<int32_t>(a_ld);
  const int pieces = a_f32 ? a_pieces : 1;
  int32_t tiles = 0;
  for (int64_t g = 0; g < groups; ++g) {
    P.ptr[g] = ptr_host[g];
    P.tile_start[g] = tiles;
    tiles += static_cast<int32_t>(ceil_div(ptr_host[g + 1] - ptr_host[g], BM)) * P.n_tiles;
  }
  P.ptr[groups] = ptr_host[groups];
  P.tile_start[groups] = tiles;
  P.num_tiles = tiles;
  // fp32-accurate split: separate hi*hi / correction accumulators, spread over
  // as many k-block sets as TMEM's 512 columns hold (two buffered tiles)
  P.acc_sets = 0;
  // only where K is long enough for the mixed accumulator to cost accuracy
  // (K=1433: norm error 1.6e-5 with one accumulator, 2.7e-7 split; K=128 stays
  // inside the 1e-5 bar with one, and the split epilogue costs C3 0.35 -> 0.46 ms)
  static const int64_t acc_min_k = [] { const char* e = getenv("GM_GEMM_ACC_MIN_K"); return e ? atoll(e) : 512; }();
  const int64_t logical_k = a_f32 ? k_in : a_seg_k;
  if (((a_f32 && a_pieces == 3) || (a_seg_k > 0 && out_dtype == GM_F32)) && logical_k >= acc_min_k) {
    static const int sets_env = [] { const char* e = getenv("GM_GEMM_ACC_SETS"); return e ? atoi(e) : 4; }();
    int sets = std::max(0, std::min(sets_env, 512 / (4 * P.bn)));
    sets = std::min(sets, a_f32 ? P.k_blocks : static_cast<int>(a_seg_k / kblk));
    P.acc_sets = sets;
  }
  P.acc_cols = P.acc_sets > 0 ? 2 * P.acc_sets * P.bn : P.bn;
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * P.acc_cols)) cols <<= 1;
  P.tmem_cols = cols;

  const size_t b_full_bytes = static_cast<size_t>(pieces) * P.k_blocks * P.bn * kblk * 2;
  const size_t b_stage_bytes = static_cast<size_t>(pieces) * P.bn * kblk * 2;
  const size_t a_stage_bytes = static_cast<size_t>(pieces) * BM * kblk * 2;
  const size_t budget = 227 * 1024 - 1024 - 512 - kCStageBytes;  // alignment slack, barriers, out staging
  // SPLIT: an fp32 staging tile rides along with every MMA stage
  const size_t x_stage_bytes = a_f32 ? static_cast<size_t>(BM) * kblk * 4 : 0;
  int stages;
  int xstages = 0;
  if (a_f32) {
    static const int res_min = [] { const char* e = getenv("GM_GEMM_SPLIT_RES"); return e ? atoi(e) : 2; }();
    const int res = P.n_tiles == 1 && b_full_bytes < budget
                        ? static_cast<int>((budget - b_full_bytes) / (a_stage_bytes + x_stage_bytes)) : 0;
    P.b_resident = res >= res_min ? 1 : 0;
    stages = P.b_resident ? res : static_cast<int>(budget / (a_stage_bytes + b_stage_bytes + x_stage_bytes));
    stages = std::max(2, std::min(stages, 8));
    xstages = stages;
    if (P.b_resident)  // spare bytes deepen the fp32 staging ring
      xstages = std::min<int>(8, static_cast<int>((budget - b_full_bytes - stages * a_stage_bytes) / x_stage_bytes));
  } else {
    P.b_resident = (P.n_tiles == 1 && b_full_bytes <= 64 * 1024) ? 1 : 0;
    if (P.b_resident) stages = static_cast<int>((budget - b_full_bytes) / a_stage_bytes);
    else stages = static_cast<int>(budget / (a_stage_bytes + b_stage_bytes));
    stages = std::max(2, std::min(stages, kblk == 32 ? 16 : 8));
  }
  P.stages = stages;
  P.x_stages = xstages;
  const size_t smem = 1024 + static_cast<size_t>(stages) * a_stage_bytes + static_cast<size_t>(xstages) * x_stage_bytes +
                      (P.b_resident ? b_full_bytes : static_cast<size_t>(stages) * b_stage_bytes) + kCStageBytes + 512;
  GM_REQUIRE(smem <= 227 * 1024, GM_ERR_INVALID_ARGUMENT, "segment_matmul: tile does not fit shared memory");

  // K-major copy of the weights: W^T as a zero-padded [G*N, K] bf16 matrix
  // (skipped when the caller pre-packed it with gm_segment_matmul_pack_w)
  if (!w_packed) {
    transpose_w_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(groups * k * n, 256), 4096)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(w), static_cast<int>(groups), static_cast<int>(k_in), static_cast<int>(n_in),
        static_cast<int>(k), static_cast<int>(n), wt);
    GM_CHECK_LAUNCH("transpose_w_kernel");
  }

  CUtensorMap map_a, map_b;
  const CUtensorMapSwizzle swz = kblk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  gm_status s = make_map(&map_b, wt, static_cast<uint64_t>(pieces * k), static_cast<uint64_t>(groups * n), kblk,
                         static_cast<uint32_t>(P.bn), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, swz);
  if (s != GM_OK) return s;
  if (a_f32) {
    // fp32 x tiles for the staging ring: KBLK columns x BM rows, zero-filled past the edges
    s = make_map(&map_a, a_f32, static_cast<uint64_t>(a_ld), static_cast<uint64_t>(rows), kblk, BM,
                 CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (s != GM_OK) return s;
  } else {
    s = make_map(&map_a, xk, static_cast<uint64_t>(a_seg_k > 0 ? a_cols : k), static_cast<uint64_t>(rows), kblk, BM,
                 CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, swz);
    if (s != GM_OK) return s;
  }
  // output map: [rows, n] of the output dtype, 128-byte x 32-row SWIZZLE_128B boxes
  CUtensorMap map_c;
  s = make_map(&map_c, outk, static_cast<uint64_t>(n), static_cast<uint64_t>(rows), 128 / static_cast<uint32_t>(esz),
               32, out_dtype == GM_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
               static_cast<uint64_t>(esz));
  if (s != GM_OK) return s;

  GroupMaps G{};
  if (ptr_mode) {
    for (int64_t g = 0; g < groups; ++g) {
      const int64_t rg = ptr_host[g + 1] - ptr_host[g];
      G.a[g] = map_a;  // empty groups own no tiles; any valid map
      G.c[g] = map_c;
      G.out[g] = gout[g];
      if (rg == 0) continue;
      GM_REQUIRE((reinterpret_cast<uintptr_t>(gx[g]) | reinterpret_cast<uintptr_t>(gout[g])) % 16 == 0,
                 GM_ERR_INVALID_ARGUMENT, "grouped_matmul: every x / out must be 16-byte aligned");
      if (a_f32)
        s = make_map(&G.a[g], gx[g], static_cast<uint64_t>(a_ld), static_cast<uint64_t>(rg), kblk, BM,
                     CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, CU_TENSOR_MAP_SWIZZLE_NONE);
      else
        s = make_map(&G.a[g], gx[g], static_cast<uint64_t>(k), static_cast<uint64_t>(rg), kblk, BM,
                     CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, swz);
      if (s != GM_OK) return s;
      s = make_map(&G.c[g], gout[g], static_cast<uint64_t>(n), static_cast<uint64_t>(rg),
                   128 / static_cast<uint32_t>(esz), 32,
                   out_dtype == GM_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   static_cast<uint64_t>(esz));
      if (s != GM_OK) return s;
    }
  }

  // per call: the attribute is per device, and a process may drive several
  const bool split = P.acc_sets > 0;
  auto kern = a_f32 ? (a_pieces == 3 ? (split ? (kblk == 64 ? segment_matmul_kernel<64, 3, true>
                                                            : segment_matmul_kernel<32, 3, true>)
                                              : (kblk == 64 ? segment_matmul_kernel<64, 3> : segment_matmul_kernel<32, 3>))
                                      : (kblk == 64 ? segment_matmul_kernel<64, 1> : segment_matmul_kernel<32, 1>))
                    : (split ? (kblk == 64 ? segment_matmul_kernel<64, 0, true> : segment_matmul_kernel<32, 0, true>)
                             : (kblk == 64 ? segment_matmul_kernel<64, 0> : segment_matmul_kernel<32, 0>));
  GM_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  const unsigned grid = static_cast<unsigned>(std::min<int32_t>(tiles, kNumSMs));
  kern<<<grid, a_f32 ? kThreads + 32 * kCvtWarps : kThreads, smem, st>>>(P, map_a, map_b, map_c, G);
  GM_CHECK_LAUNCH("segment_matmul_kernel");
  if (n != n_in) {
    unpad_cols_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(rows * n_in, 256), 8192)), 256, 0, st>>>(
        static_cast<const unsigned char*>(outk), rows, static_cast<int>(n_in), static_cast<int>(n),
        static_cast<int>(esz), static_cast<unsigned char*>(out));
    GM_CHECK_LAUNCH("unpad_cols_kernel");
  }
  return GM_OK;
}

GM_API gm_status gm_segment_matmul(const void* x, const int64_t* ptr_host, int64_t groups, int64_t k_in,
                                   int64_t n_in, const void* w, gm_dtype out_dtype, void* out, void* workspace,
                                   size_t workspace_bytes, gm_stream_t stream) {
  return segment_matmul_impl(x, ptr_host, groups, k_in, n_in, w, nullptr, out_dtype, out, workspace, workspace_bytes,
                             stream);
}

GM_API size_t gm_segment_matmul_packed_w_bytes(int64_t groups, int64_t k, int64_t n) {
  if (groups < 0 || k < 0 || n < 0) return 0;
  return static_cast<size_t>(groups * pad_to(std::max<int64_t>(k, 1), 64) * pad_to(std::max<int64_t>(n, 1), 16)) * 2;
}

GM_API gm_status gm_segment_matmul_pack_w(const void* w, int64_t groups, int64_t k, int64_t n, void* packed,
                                          gm_stream_t stream) {
  GM_REQUIRE(w && packed && groups >= 1 && k > 0 && n > 0, GM_ERR_INVALID_ARGUMENT, "segment_matmul_pack_w: bad args");
  const int64_t kp = pad_to(k, 64), np = pad_to(n, 16);
  cudaStream_t st = as_stream(stream);
  gm::gmm::transpose_w_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(groups * kp * np, 256), 4096)), 256, 0,
                                st>>>(static_cast<const __nv_bfloat16*>(w), static_cast<int>(groups), static_cast<int>(k),
                                      static_cast<int>(n), static_cast<int>(kp), static_cast<int>(np),
                                      static_cast<__nv_bfloat16*>(packed));
  GM_CHECK_LAUNCH("transpose_w_kernel");
  return GM_OK;
}

GM_API size_t gm_segment_matmul_packed_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n) {
  return gm_segment_matmul_workspace(rows, groups, k, n) -
         align_up(gm_segment_matmul_packed_w_bytes(groups, k, n), 256);
}

GM_API gm_status gm_segment_matmul_packed(const void* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                          int64_t n, const void* packed_w, gm_dtype out_dtype, void* out,
                                          void* workspace, size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(packed_w, GM_ERR_INVALID_ARGUMENT, "segment_matmul: null packed weights");
  return segment_matmul_impl(x, ptr_host, groups, k, n, nullptr, packed_w, out_dtype, out, workspace, workspace_bytes,
                             stream);
}

GM_API gm_status gm_segment_matmul_packed_xf32(const float* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                               int64_t n, const void* packed_w, float* out, void* workspace,
                                               size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(packed_w, GM_ERR_INVALID_ARGUMENT, "segment_matmul: null packed weights");
  GM_REQUIRE(k % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, GM_ERR_INVALID_ARGUMENT,
             "segment_matmul: fp32 x needs k % 4 == 0 and 16-byte alignment");
  const int64_t kp = pad_to(std::max<int64_t>(k, 1), 64);
  return segment_matmul_impl(x, ptr_host, groups, kp, n, nullptr, packed_w, GM_F32, out, workspace, workspace_bytes,
                             stream, 0, 0, 0, x, k, 1);
}

GM_API size_t gm_segment_matmul_f32_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n) {
  if (rows < 0 || groups < 0 || k < 0 || n < 0) return 0;
  const int64_t kp = pad_to(std::max<int64_t>(k, 1), 64);
  return align_up(static_cast<size_t>(rows * 3 * kp) * 2, 256) +
         align_up(static_cast<size_t>(groups * kSplit * kp * n) * 2, 256) +
         gm_segment_matmul_workspace(rows, groups, kSplit * kp, n);
}

static gm_status segment_matmul_f32_impl(const float* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                         int64_t n, const float* w, float* out, void* workspace,
                                         size_t workspace_bytes, gm_stream_t stream, const void* const* gx,
                                         void* const* gout) {
  GM_REQUIRE(ptr_host && groups >= 1, GM_ERR_INVALID_ARGUMENT, "segment_matmul: bad groups");
  GM_REQUIRE(k > 0 && n > 0, GM_ERR_INVALID_ARGUMENT, "segment_matmul: K and N must be positive");
  const int64_t rows = ptr_host[groups];
  if (rows == 0) return GM_OK;
  GM_REQUIRE(x && w && out, GM_ERR_INVALID_ARGUMENT, "segment_matmul: null pointer");
  const size_t need = gm_segment_matmul_f32_workspace(rows, groups, k, n);
  GM_REQUIRE(workspace && workspace_bytes >= need, GM_ERR_INVALID_ARGUMENT, "segment_matmul: workspace too small");
  const int64_t kp = pad_to(k, 64);
  GM_REQUIRE(rows * 3 * kp < (int64_t{1} << 40) && 3 * kp < (int64_t{1} << 31), GM_ERR_INVALID_ARGUMENT,
             "segment_matmul: operand too large");
  cudaStream_t st = as_stream(stream);
  // fused split (x read once by TMA, pieces formed in shared memory) when x
  // rows meet TMA's 16-byte stride rule; GM_GEMM_FUSED_SPLIT=0 selects the staged path below
  static const bool fused_env = [] { const char* e = getenv("GM_GEMM_FUSED_SPLIT"); return !(e && e[0] == '0'); }();
  if (fused_env && k % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 && (!gx || n % 16 == 0)) {
    const int64_t np = pad_to(n, 16);
    auto* wt = static_cast<__nv_bfloat16*>(workspace);
    const size_t wt_bytes = align_up(static_cast<size_t>(groups * np * 3 * kp) * 2, 256);
    split_wt_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(groups * np * kp, 256), kNumSMs * 32)), 256, 0,
                      st>>>(w, static_cast<int>(groups), static_cast<int>(k), static_cast<int>(n), static_cast<int>(kp),
                            static_cast<int>(np), wt);
    GM_CHECK_LAUNCH("split_wt_kernel");
    return segment_matmul_impl(x, ptr_host, groups, kp, n, nullptr, wt, GM_F32, out,
                               static_cast<unsigned char*>(workspace) + wt_bytes, workspace_bytes - wt_bytes, stream,
                               0, 0, 0, x, k, 3, gx, gout);
  }
  GM_REQUIRE(!gx, GM_ERR_INVALID_ARGUMENT, "grouped_matmul: pointer-array route needs k % 4 == 0, n % 16 == 0");
  unsigned char* b = static_cast<unsigned char*>(workspace);
  auto* xs = reinterpret_cast<__nv_bfloat16*>(b);
  b += align_up(static_cast<size_t>(rows * 3 * kp) * 2, 256);
  auto* ws = reinterpret_cast<__nv_bfloat16*>(b);
  b += align_up(static_cast<size_t>(groups * kSplit * kp * n) * 2, 256);
  split_x_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(rows * kp / 4, 256), kNumSMs * 32)), 256, 0, st>>>(
      x, rows, static_cast<int>(k), static_cast<int>(kp), xs);
  GM_CHECK_LAUNCH("split_x_kernel");
  split_w_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(groups * kp * n, 256), kNumSMs * 32)), 256, 0,
                   st>>>(w, static_cast<int>(groups), static_cast<int>(k), static_cast<int>(kp), static_cast<int>(n), ws);
  GM_CHECK_LAUNCH("split_w_kernel");
  return segment_matmul_impl(xs, ptr_host, groups, kSplit * kp, n, ws, nullptr, GM_F32, out, b,
                             workspace_bytes - static_cast<size_t>(b - static_cast<unsigned char*>(workspace)), stream,
                             kp, kSplitSegMap, 3 * kp);
}

GM_API gm_status gm_segment_matmul_f32(const float* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                       int64_t n, const float* w, float* out, void* workspace, size_t workspace_bytes,
                                       gm_stream_t stream) {
  return segment_matmul_f32_impl(x, ptr_host, groups, k, n, w, out, workspace, workspace_bytes, stream, nullptr,
                                 nullptr);
}

// grouped_matmul over separate per-group tensors (hetero.hpp:134-157): one
// TMA map per group for x and out, so nothing is concatenated when the shapes
// run unpadded (<= 8 groups, n % 16 == 0, 16-byte aligned; x f32: k % 4 == 0,
// x bf16: k % 64 == 0); otherwise the groups are gathered into the workspace
// (stream-ordered copies) and the results copied back.
// Operand routes: (f32 x, f32 w) fp32-accurate split; (f32 x, bf16 w) x
// rounded to bf16 inside the kernel; (bf16, bf16).
static bool grouped_direct(int64_t groups, int64_t k, int64_t n, gm_dtype x_dtype) {
  if (groups > gm::gmm::kMaxPtrGroups || n % 16 != 0) return false;
  return x_dtype == GM_F32 ? k % 4 == 0 : k % 64 == 0;
}

static size_t grouped_inner_ws(int64_t rows, int64_t groups, int64_t k, int64_t n, gm_dtype x_dtype,
                               gm_dtype w_dtype) {
  if (x_dtype == GM_F32 && w_dtype == GM_F32) return gm_segment_matmul_f32_workspace(rows, groups, k, n);
  if (x_dtype == GM_F32)  // packed bf16 W + the packed route's workspace
    return align_up(gm_segment_matmul_packed_w_bytes(groups, k, n), 256) +
           gm_segment_matmul_packed_workspace(rows, groups, k, n);
  return gm_segment_matmul_workspace(rows, groups, k, n);
}

GM_API size_t gm_grouped_matmul_workspace(const int64_t* rows_host, int64_t groups, int64_t k, int64_t n,
                                          gm_dtype x_dtype, gm_dtype w_dtype, gm_dtype out_dtype) {
  if (!rows_host || groups < 1 || k < 1 || n < 1) return 0;
  int64_t rows = 0;
  for (int64_t g = 0; g < groups; ++g) rows += rows_host[g];
  const size_t inner = grouped_inner_ws(rows, groups, k, n, x_dtype, w_dtype);
  if (grouped_direct(groups, k, n, x_dtype)) return inner;
  const size_t xe = x_dtype == GM_F32 ? 4 : 2, oe = out_dtype == GM_F32 ? 4 : 2;
  return inner + align_up(static_cast<size_t>(rows * k) * xe, 256) + align_up(static_cast<size_t>(rows * n) * oe, 256);
}

// one launch over the groups described by (x, out) — contiguous, or per-group
// pointers when gx / gout are given
static gm_status grouped_run(const void* x, const int64_t* ptr, int64_t groups, int64_t k, int64_t n, const void* w,
                             gm_dtype x_dtype, gm_dtype w_dtype, void* out, gm_dtype out_dtype, void* ws,
                             size_t ws_bytes, gm_stream_t stream, const void* const* gx, void* const* gout) {
  if (x_dtype == GM_F32 && w_dtype == GM_F32)
    return segment_matmul_f32_impl(static_cast<const float*>(x), ptr, groups, k, n, static_cast<const float*>(w),
                                   static_cast<float*>(out), ws, ws_bytes, stream, gx, gout);
  if (x_dtype == GM_F32) {
    unsigned char* packed = static_cast<unsigned char*>(ws);
    const size_t pb = align_up(gm_segment_matmul_packed_w_bytes(groups, k, n), 256);
    gm_status s = gm_segment_matmul_pack_w(w, groups, k, n, packed, stream);
    if (s != GM_OK) return s;
    GM_REQUIRE(k % 4 == 0 && out_dtype == GM_F32, GM_ERR_INVALID_ARGUMENT,
               "grouped_matmul: f32 x with bf16 weights needs k % 4 == 0 and f32 out");
    const int64_t kp = pad_to(k, 64);
    return segment_matmul_impl(x, ptr, groups, kp, n, nullptr, packed, GM_F32, out, packed + pb, ws_bytes - pb,
                               stream, 0, 0, 0, static_cast<const float*>(x), k, 1, gx, gout);
  }
  return segment_matmul_impl(x, ptr, groups, k, n, w, nullptr, out_dtype, out, ws, ws_bytes, stream, 0, 0, 0,
                             nullptr, 0, 3, gx, gout);
}

GM_API gm_status gm_grouped_matmul(const void* const* x_host, const int64_t* rows_host, int64_t groups, int64_t k,
                                   int64_t n, const void* w, gm_dtype x_dtype, gm_dtype w_dtype, void* const* out_host,
                                   gm_dtype out_dtype, void* workspace, size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(x_host && rows_host && out_host && groups >= 1, GM_ERR_INVALID_ARGUMENT,
             "grouped_matmul: null group arrays");
  GM_REQUIRE((x_dtype == GM_F32 || x_dtype == GM_BF16) && (w_dtype == GM_F32 || w_dtype == GM_BF16) &&
                 !(x_dtype == GM_BF16 && w_dtype == GM_F32),
             GM_ERR_INVALID_ARGUMENT, "grouped_matmul: operands (f32, f32), (f32, bf16) or (bf16, bf16)");
  GM_REQUIRE(x_dtype == GM_BF16 || out_dtype == GM_F32, GM_ERR_INVALID_ARGUMENT,
             "grouped_matmul: f32 activations produce f32");
  GM_REQUIRE(workspace_bytes >= gm_grouped_matmul_workspace(rows_host, groups, k, n, x_dtype, w_dtype, out_dtype),
             GM_ERR_INVALID_ARGUMENT, "grouped_matmul: workspace too small");
  std::vector<int64_t> ptr(static_cast<size_t>(groups) + 1, 0);
  for (int64_t g = 0; g < groups; ++g) {
    GM_REQUIRE(rows_host[g] >= 0, GM_ERR_INVALID_ARGUMENT, "grouped_matmul: negative group rows");
    ptr[static_cast<size_t>(g) + 1] = ptr[static_cast<size_t>(g)] + rows_host[g];
  }
  const int64_t rows = ptr.back();
  if (rows == 0) return GM_OK;
  int64_t first = 0;
  while (rows_host[first] == 0) ++first;
  if (grouped_direct(groups, k, n, x_dtype))
    return grouped_run(x_host[first], ptr.data(), groups, k, n, w, x_dtype, w_dtype, out_host[first], out_dtype,
                       workspace, workspace_bytes, stream, x_host, out_host);
  // gathered route
  cudaStream_t st = as_stream(stream);
  const size_t xe = x_dtype == GM_F32 ? 4 : 2, oe = out_dtype == GM_F32 ? 4 : 2;
  unsigned char* xb = static_cast<unsigned char*>(workspace);
  unsigned char* ob = xb + align_up(static_cast<size_t>(rows * k) * xe, 256);
  unsigned char* inner = ob + align_up(static_cast<size_t>(rows * n) * oe, 256);
  const size_t inner_bytes = workspace_bytes - static_cast<size_t>(inner - xb);
  for (int64_t g = 0; g < groups; ++g)
    if (rows_host[g] > 0)
      GM_TRY_CUDA(cudaMemcpyAsync(xb + ptr[static_cast<size_t>(g)] * k * xe, x_host[g],
                                  static_cast<size_t>(rows_host[g] * k) * xe, cudaMemcpyDeviceToDevice, st));
  gm_status s = x_dtype == GM_F32 && w_dtype == GM_BF16 && k % 4 != 0
                    ? fail(GM_ERR_INVALID_ARGUMENT, "grouped_matmul: f32 x with bf16 weights needs k % 4 == 0")
                    : grouped_run(xb, ptr.data(), groups, k, n, w, x_dtype, w_dtype, ob, out_dtype, inner,
                                  inner_bytes, stream, nullptr, nullptr);
  if (s != GM_OK) return s;
  for (int64_t g = 0; g < groups; ++g)
    if (rows_host[g] > 0)
      GM_TRY_CUDA(cudaMemcpyAsync(out_host[g], ob + ptr[static_cast<size_t>(g)] * n * oe,
                                  static_cast<size_t>(rows_host[g] * n) * oe, cudaMemcpyDeviceToDevice, st));
  return GM_OK;
}

}  // extern "C"
