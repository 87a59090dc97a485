// vec.cuh — vector load/convert/store helpers for f32 / f64 / bf16 feature
// rows. A lane moves VB bytes (16/8/4/2) per access; values are widened to the
// accumulation type (fp32 for f32/bf16, fp64 for f64) exactly.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "gm_common.cuh"

namespace gm {

template <int VB>
struct RawT;
template <>
struct RawT<16> {
  using type = uint4;
};
template <>
struct RawT<8> {
  using type = uint2;
};
template <>
struct RawT<4> {
  using type = uint32_t;
};
template <>
struct RawT<2> {
  using type = unsigned short;
};

template <typename T>
struct AccOf {
  using type = float;
};
template <>
struct AccOf<double> {
  using type = double;
};

// Exact widening of one stored element.
__device__ __forceinline__ float widen(float v) { return v; }
__device__ __forceinline__ double widen(double v) { return v; }
__device__ __forceinline__ float widen(__nv_bfloat16 v) { return __bfloat162float(v); }

// Narrowing for the store (RNE for bf16).
template <typename T, typename A>
__device__ __forceinline__ T narrow(A v);
template <>
__device__ __forceinline__ float narrow<float, float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ double narrow<double, double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 narrow<__nv_bfloat16, float>(float v) {
  return __float2bfloat16_rn(v);
}

// IEEE round-to-nearest arithmetic with no contraction (parity path).
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

// Streaming (evict-first) stores of raw vectors: output rows are written once.
__device__ __forceinline__ void st_cs(uint4* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_cs(uint2* p, const uint2& v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_cs(uint32_t* p, const uint32_t& v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs(unsigned short* p, const unsigned short& v) {
  asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

template <typename T, int VB>
struct Vec {
  static constexpr int V = VB / (int)sizeof(T);
  static_assert(V >= 1, "vector narrower than one element");
  using A = typename AccOf<T>::type;
  using R = typename RawT<VB>::type;
  A v[V];

  __device__ __forceinline__ void from_raw(const R& r) {
    T tmp[V];
    memcpy(tmp, &r, VB);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = widen(tmp[i]);
  }
  // Global gather (read-only, L1 no-allocate).
  __device__ __forceinline__ void load_global(const T* p) {
    from_raw(ldg_na<R>(reinterpret_cast<const R*>(p)));
  }
  __device__ __forceinline__ void load_shared(const T* p) {
    from_raw(*reinterpret_cast<const R*>(p));
  }
  // Raw (still packed) gather, widened later at consume time: keeps bf16
  // batches at half the registers.
  __device__ static __forceinline__ R load_raw(const T* p) {
    return ldg_na<R>(reinterpret_cast<const R*>(p));
  }
  __device__ static __forceinline__ void unpack(const R& r, A* out) {
    if constexpr (sizeof(T) == 2 && VB >= 4) {
      // bf16 -> fp32 is exact: the low half shifts up 16 bits, the high half
      // keeps its upper 16 bits (2 integer ops per packed word)
      uint32_t words[VB / 4];
      memcpy(words, &r, VB);
#pragma unroll
      for (int i = 0; i < VB / 4; ++i) {
        out[2 * i] = __uint_as_float(words[i] << 16);
        out[2 * i + 1] = __uint_as_float(words[i] & 0xffff0000u);
      }
    } else {
      T tmp[V];
      memcpy(tmp, &r, VB);
#pragma unroll
      for (int i = 0; i < V; ++i) out[i] = widen(tmp[i]);
    }
  }
  __device__ static __forceinline__ R pack(const A* vals) {
    T tmp[V];
#pragma unroll
    for (int i = 0; i < V; ++i) tmp[i] = narrow<T, A>(vals[i]);
    R r;
    memcpy(&r, tmp, VB);
    return r;
  }
  __device__ static __forceinline__ void store_global(T* p, const A* vals) {
    T tmp[V];
#pragma unroll
    for (int i = 0; i < V; ++i) tmp[i] = narrow<T, A>(vals[i]);
    R r;
    memcpy(&r, tmp, VB);
    st_cs(reinterpret_cast<R*>(p), r);
  }
};

}  // namespace gm
