// synth.cu — device and host generators over synth.h (identical arithmetic),
// plus the C-ABI odds and ends: error TLS, version, device probe, partitioner.
#include <cuda_bf16.h>

#include <algorithm>
#include <string>

#include "gm_common.cuh"
#include "synth.h"

namespace gm {

static thread_local std::string t_error;
void set_error(const std::string& msg) { t_error = msg; }

__global__ void synth_edges_kernel(int kind, uint64_t seed, int64_t first, int64_t count,
                                   int64_t n_src, int64_t n_dst, int64_t* __restrict__ src,
                                   int64_t* __restrict__ dst) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t s, d;
    gm_synth::edge(kind, seed, static_cast<uint64_t>(first + i), static_cast<uint64_t>(n_src),
                   static_cast<uint64_t>(n_dst), &s, &d);
    src[i] = s;
    dst[i] = d;
  }
}

template <typename T>
__device__ __forceinline__ T cvt_out(double v);
template <>
__device__ __forceinline__ float cvt_out<float>(double v) {
  return static_cast<float>(v);
}
template <>
__device__ __forceinline__ double cvt_out<double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn(static_cast<float>(v));
}

template <typename T>
__global__ void synth_features_kernel(uint64_t seed, int64_t first_row, int64_t rows, int64_t f,
                                      int quantize, T* __restrict__ x) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    gm_synth::FeatureRow fr(seed, static_cast<uint64_t>(first_row + i), quantize);
    T* row = x + i * f;
    for (int64_t j = 0; j < f; ++j) row[j] = cvt_out<T>(fr.next());
  }
}

template <typename T>
__global__ void synth_weights_kernel(uint64_t seed, int64_t first, int64_t count, T* __restrict__ w) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] = cvt_out<T>(gm_synth::weight(seed, static_cast<uint64_t>(first + i)));
}

static unsigned synth_grid(int64_t n) {
  return static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), kNumSMs * 16));
}

// Host-side bf16 RNE (matches __float2bfloat16_rn for finite values).
static uint16_t host_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40);
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return static_cast<uint16_t>(u >> 16);
}

}  // namespace gm

using namespace gm;

extern "C" {

GM_API const char* gm_last_error(void) { return t_error.c_str(); }
GM_API const char* gm_version(void) { return "graphmill-b200 0.1 (sm_100a)"; }

GM_API int gm_device_supported(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0;
}

GM_API gm_status gm_synth_edges(int kind, uint64_t seed, int64_t first, int64_t count,
                                int64_t n_src, int64_t n_dst, int64_t* src, int64_t* dst,
                                gm_stream_t stream) {
  GM_REQUIRE(count >= 0 && n_src > 0 && n_dst > 0, GM_ERR_INVALID_ARGUMENT,
             "gm_synth_edges: bad sizes");
  if (count == 0) return GM_OK;
  synth_edges_kernel<<<synth_grid(count), 256, 0, as_stream(stream)>>>(kind, seed, first, count,
                                                                      n_src, n_dst, src, dst);
  GM_CHECK_LAUNCH("synth_edges_kernel");
  return GM_OK;
}

GM_API void gm_synth_edges_host(int kind, uint64_t seed, int64_t first, int64_t count,
                                int64_t n_src, int64_t n_dst, int64_t* src, int64_t* dst) {
  for (int64_t i = 0; i < count; ++i)
    gm_synth::edge(kind, seed, static_cast<uint64_t>(first + i), static_cast<uint64_t>(n_src),
                   static_cast<uint64_t>(n_dst), src + i, dst + i);
}

GM_API gm_status gm_synth_features(uint64_t seed, int64_t first_row, int64_t rows, int64_t f,
                                   int quantize, gm_dtype dtype, void* x, gm_stream_t stream) {
  GM_REQUIRE(rows >= 0 && f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_synth_features: bad sizes");
  if (rows == 0 || f == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F32)
    synth_features_kernel<float><<<synth_grid(rows), 256, 0, st>>>(seed, first_row, rows, f, quantize,
                                                                   static_cast<float*>(x));
  else if (dtype == GM_F64)
    synth_features_kernel<double><<<synth_grid(rows), 256, 0, st>>>(seed, first_row, rows, f, quantize,
                                                                    static_cast<double*>(x));
  else
    synth_features_kernel<__nv_bfloat16><<<synth_grid(rows), 256, 0, st>>>(
        seed, first_row, rows, f, quantize, static_cast<__nv_bfloat16*>(x));
  GM_CHECK_LAUNCH("synth_features_kernel");
  return GM_OK;
}

GM_API void gm_synth_features_host(uint64_t seed, int64_t first_row, int64_t rows, int64_t f,
                                   int quantize, gm_dtype dtype, void* x) {
  for (int64_t i = 0; i < rows; ++i) {
    gm_synth::FeatureRow fr(seed, static_cast<uint64_t>(first_row + i), quantize);
    for (int64_t j = 0; j < f; ++j) {
      const double v = fr.next();
      if (dtype == GM_F32) static_cast<float*>(x)[i * f + j] = static_cast<float>(v);
      else if (dtype == GM_F64) static_cast<double*>(x)[i * f + j] = v;
      else static_cast<uint16_t*>(x)[i * f + j] = host_bf16(static_cast<float>(v));
    }
  }
}

GM_API gm_status gm_synth_weights(uint64_t seed, int64_t first, int64_t count, gm_dtype dtype,
                                  void* w, gm_stream_t stream) {
  GM_REQUIRE(count >= 0, GM_ERR_INVALID_ARGUMENT, "gm_synth_weights: bad size");
  if (count == 0) return GM_OK;
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F64)
    synth_weights_kernel<double><<<synth_grid(count), 256, 0, st>>>(seed, first, count, static_cast<double*>(w));
  else if (dtype == GM_F32)
    synth_weights_kernel<float><<<synth_grid(count), 256, 0, st>>>(seed, first, count, static_cast<float*>(w));
  else
    synth_weights_kernel<__nv_bfloat16><<<synth_grid(count), 256, 0, st>>>(
        seed, first, count, static_cast<__nv_bfloat16*>(w));
  GM_CHECK_LAUNCH("synth_weights_kernel");
  return GM_OK;
}

GM_API void gm_synth_weights_host(uint64_t seed, int64_t first, int64_t count, gm_dtype dtype, void* w) {
  for (int64_t i = 0; i < count; ++i) {
    const double v = gm_synth::weight(seed, static_cast<uint64_t>(first + i));
    if (dtype == GM_F64) static_cast<double*>(w)[i] = v;
    else if (dtype == GM_F32) static_cast<float*>(w)[i] = static_cast<float>(v);
    else static_cast<uint16_t*>(w)[i] = host_bf16(static_cast<float>(v));
  }
}

// North-star partitioner: contiguous destination-row ranges with ~nnz/parts
// edges each (SURVEY.md §8e "Compute ranges").
GM_API gm_status gm_partition_rows_by_nnz(const int64_t* rowptr_host, int64_t num_rows,
                                          int32_t parts, int64_t* cuts_host) {
  GM_REQUIRE(rowptr_host && cuts_host && parts >= 1 && num_rows >= 0, GM_ERR_INVALID_ARGUMENT,
             "gm_partition_rows_by_nnz: bad arguments");
  const int64_t nnz = rowptr_host[num_rows];
  cuts_host[0] = 0;
  for (int32_t p = 1; p < parts; ++p) {
    const int64_t target = (nnz * p + parts - 1) / parts;
    const int64_t* it = std::lower_bound(rowptr_host, rowptr_host + num_rows + 1, target);
    int64_t r = static_cast<int64_t>(it - rowptr_host);
    r = std::max<int64_t>(r, cuts_host[p - 1]);
    cuts_host[p] = std::min<int64_t>(r, num_rows);
  }
  cuts_host[parts] = num_rows;
  return GM_OK;
}

}  // extern "C"
