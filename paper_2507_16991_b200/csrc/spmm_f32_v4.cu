// spmm_f32_v4.cu — float / 4-byte-vector instantiation of the SpMM kernels
// (one TU per (dtype, vector width) so the kernel variants build in parallel).
#include "spmm_kernels.cuh"

namespace gm {
template gm_status dispatch_vb<float, 4>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
}  // namespace gm
