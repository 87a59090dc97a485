// spmm_bf16_v8.cu — __nv_bfloat16 / 8-byte-vector instantiation of the SpMM kernels
// (one TU per (dtype, vector width) so the kernel variants build in parallel).
#include "spmm_kernels.cuh"

namespace gm {
template gm_status dispatch_vb<__nv_bfloat16, 8>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
}  // namespace gm
