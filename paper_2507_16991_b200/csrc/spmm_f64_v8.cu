// spmm_f64_v8.cu — double / 8-byte-vector instantiation of the SpMM kernels
// (one TU per (dtype, vector width) so the kernel variants build in parallel).
#include "spmm_kernels.cuh"

namespace gm {
template gm_status dispatch_vb<double, 8>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
}  // namespace gm
