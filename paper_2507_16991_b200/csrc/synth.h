// synth.h — counter-based synthetic graph/feature generators, compiled both
// for the host (g++, -ffp-contract=off) and the device (nvcc), so CPU oracle
// inputs and GPU inputs are bit-identical.
//
// The RNG is the reference's (random.hpp:9-65): splitmix64 `mix`, `derive`,
// `Stream::{next_u64,next_below,next_real}`. Every edge / row draws from its
// own derived stream, so generation is order- and thread-count-invariant.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GM_HD __host__ __device__ __forceinline__
#else
#define GM_HD inline
#endif

namespace gm_synth {

// Correctly rounded fp64 ops with no FMA contraction on either side.
GM_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
GM_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
GM_HD double dsqrt(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  return __builtin_sqrt(a);
#endif
}

// random.hpp:9-14
GM_HD uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// random.hpp:19-32
GM_HD uint64_t derive(uint64_t seed, uint64_t a) { return mix(seed ^ mix(a)); }
GM_HD uint64_t derive(uint64_t seed, uint64_t a, uint64_t b) { return derive(derive(seed, a), b); }
GM_HD uint64_t derive(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return derive(derive(seed, a, b), c);
}

// random.hpp:37-65
struct Stream {
  uint64_t state;
  GM_HD explicit Stream(uint64_t key) : state(mix(key)) {}
  GM_HD uint64_t next_u64() {
    state += 0x9e3779b97f4a7c15ull;
    uint64_t x = state;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  GM_HD uint64_t next_below(uint64_t n) {
    const uint64_t limit = n * (~uint64_t{0} / n);
    uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % n;
  }
  GM_HD double next_real() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
  GM_HD double next_real(double lo, double hi) { return dadd(lo, dmul(hi - lo, next_real())); }
};

// Stream purposes (mixed into derive()).
enum : uint64_t {
  kTagSrc = 0x737263ull,      // "src"
  kTagDst = 0x647374ull,      // "dst"
  kTagFeat = 0x66656174ull,   // "feat"
  kTagWgt = 0x776774ull,      // "wgt"
  kTagPerm = 0x7065726dull,   // "perm"
  kTagQuant = 0x7175616eull,  // "quan"
};

// Bijective permutation of [0, n) (Feistel network on the smallest even-bit
// power-of-two domain >= n, cycle-walking), keyed by `key`. Integer-only.
GM_HD uint64_t permute(uint64_t x, uint64_t n, uint64_t key) {
  if (n <= 1) return 0;
  int bits = 0;
  while ((uint64_t{1} << bits) < n) ++bits;
  if (bits & 1) ++bits;
  if (bits < 2) bits = 2;
  const int half = bits / 2;
  const uint64_t mask = (uint64_t{1} << half) - 1;
  do {
    uint64_t l = x >> half, r = x & mask;
    for (int round = 0; round < 4; ++round) {
      const uint64_t nl = r;
      r = l ^ (mix(key ^ (r * 0x100000001b3ull) ^ (uint64_t)round) & mask);
      l = nl;
    }
    x = (l << half) | r;
  } while (x >= n);
  return x;
}

// Chung-Lu endpoint with weight (p+1)^-1/2 over positions p in [0, n), by
// inverse CDF of the continuous density: x = (1 + u(sqrt(n+1) - 1))^2 - 1,
// then a keyed permutation maps positions to node ids. Only correctly rounded
// fp64 ops (sqrt, mul, add), so host and device agree bit-for-bit.
GM_HD uint64_t powerlaw_node(double u, uint64_t n, uint64_t perm_key) {
  const double s = dadd(dsqrt((double)(n + 1)), -1.0);
  const double t = dadd(1.0, dmul(u, s));
  double xpos = dadd(dmul(t, t), -1.0);
  uint64_t p = xpos <= 0.0 ? 0 : (uint64_t)xpos;
  if (p >= n) p = n - 1;
  return permute(p, n, perm_key);
}

// Edge i of a synthetic COO list. kind 0 = uniform (next_below, as the
// reference tests' random_graph, test_message_passing.cpp:17-25, but with a
// per-edge stream), kind 1 = power-law Chung-Lu alpha=0.5 on both endpoints
// with independent permutations.
GM_HD void edge(int kind, uint64_t seed, uint64_t i, uint64_t n_src, uint64_t n_dst,
                int64_t* s_out, int64_t* d_out) {
  Stream ss(derive(seed, kTagSrc, i));
  Stream ds(derive(seed, kTagDst, i));
  if (kind == 0) {
    *s_out = (int64_t)ss.next_below(n_src);
    *d_out = (int64_t)ds.next_below(n_dst);
  } else {
    *s_out = (int64_t)powerlaw_node(ss.next_real(), n_src, derive(seed, kTagPerm, 1));
    *d_out = (int64_t)powerlaw_node(ds.next_real(), n_dst, derive(seed, kTagPerm, 2));
  }
}

// Feature x[row][j] ~ U[-1, 1) from the row's stream (Tensor::rand_uniform,
// tensor.hpp:147-152, per row). quantize != 0: rows selected by a hash (1 in
// 4) are snapped down to multiples of 1/8 so max ties exist at scale, and a
// snapped zero becomes -0.0 for half of those rows (±0 tie semantics).
struct FeatureRow {
  Stream s;
  bool snap;
  bool negzero;
  GM_HD FeatureRow(uint64_t seed, uint64_t row, int quantize) : s(derive(seed, kTagFeat, row)) {
    const uint64_t h = mix(derive(seed, kTagQuant, row));
    snap = quantize && (h & 3) == 0;
    negzero = (h >> 2) & 1;
  }
  GM_HD double next() {
    double v = s.next_real(-1.0, 1.0);
    if (snap) {
      double q = (double)(int64_t)dmul(v, 8.0);
      if (q > dmul(v, 8.0)) q = dadd(q, -1.0);  // floor
      v = dmul(q, 0.125);
      if (v == 0.0 && negzero) v = -0.0;
    }
    return v;
  }
};

// Edge weight ~ U[0.5, 1.5).
GM_HD double weight(uint64_t seed, uint64_t i) {
  Stream s(derive(seed, kTagWgt, i));
  return s.next_real(0.5, 1.5);
}

}  // namespace gm_synth
