// gm_common.cuh — shared plumbing for the sm_100a kernels: status/error TLS,
// launch checks, dtype traits and cache-hinted memory ops.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "graphmill_b200.h"

namespace gm {

// Thread-local error text (set on failure, returned by gm_last_error()).
void set_error(const std::string& msg);

inline gm_status fail(gm_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

inline gm_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return GM_OK;
  return fail(GM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define GM_TRY_CUDA(expr)                                            \
  do {                                                               \
    cudaError_t gm_e_ = (expr);                                      \
    if (gm_e_ != cudaSuccess) return ::gm::cuda_status(gm_e_, #expr); \
  } while (0)

#define GM_CHECK_LAUNCH(name)                                       \
  do {                                                              \
    cudaError_t gm_e_ = cudaGetLastError();                         \
    if (gm_e_ != cudaSuccess) return ::gm::cuda_status(gm_e_, name); \
  } while (0)

#define GM_REQUIRE(cond, st, msg) \
  do {                            \
    if (!(cond)) return ::gm::fail((st), (msg)); \
  } while (0)

inline cudaStream_t as_stream(gm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// Cache-hinted loads/stores (guide §G13/G14)
// ---------------------------------------------------------------------------

// Gathered feature rows: read-only, no L1 allocation (little intra-SM reuse),
// default L2 policy so power-law hub rows stay L2-resident across SMs.
template <typename V>
__device__ __forceinline__ V ldg_na(const V* p);

template <>
__device__ __forceinline__ float4 ldg_na<float4>(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ float2 ldg_na<float2>(const float2* p) {
  float2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ float ldg_na<float>(const float* p) {
  float r;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ double2 ldg_na<double2>(const double2* p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ double ldg_na<double>(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint4 ldg_na<uint4>(const uint4* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint2 ldg_na<uint2>(const uint2* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint32_t ldg_na<uint32_t>(const uint32_t* p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ldg_na<unsigned short>(const unsigned short* p) {
  unsigned short r;
  asm("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

// Output rows are written once and not re-read by this kernel: evict-first.
template <typename V>
__device__ __forceinline__ void stg_cs(V* p, const V& v) {
  __stcs(p, v);
}

}  // namespace gm
