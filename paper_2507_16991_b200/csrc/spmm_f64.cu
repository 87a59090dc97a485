// spmm_f64.cu — double instantiations of the SpMM kernels (split for parallel builds).
#include "spmm_kernels.cuh"

namespace gm {

extern template gm_status dispatch_vb<double, 16>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
extern template gm_status dispatch_vb<double, 8>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);

gm_status spmm_dispatch_f64(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy, int64_t ns, int vb,
                            cudaStream_t st) {
  if (vb == 16) return dispatch_vb<double, 16>(p, maxmin, use_heavy, num_heavy, ns, st);
  return dispatch_vb<double, 8>(p, maxmin, use_heavy, num_heavy, ns, st);
}

}  // namespace gm
