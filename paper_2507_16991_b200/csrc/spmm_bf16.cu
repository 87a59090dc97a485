// spmm_bf16.cu — __nv_bfloat16 instantiations of the SpMM kernels (split for parallel builds).
#include "spmm_kernels.cuh"

namespace gm {

extern template gm_status dispatch_vb<__nv_bfloat16, 16>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
extern template gm_status dispatch_vb<__nv_bfloat16, 8>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
extern template gm_status dispatch_vb<__nv_bfloat16, 4>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);
extern template gm_status dispatch_vb<__nv_bfloat16, 2>(const SpmmArgs&, bool, bool, int64_t, int64_t, cudaStream_t);

gm_status spmm_dispatch_bf16(const SpmmArgs& p, bool maxmin, bool use_heavy, int64_t num_heavy, int64_t ns, int vb,
                            cudaStream_t st) {
  if (vb == 16) return dispatch_vb<__nv_bfloat16, 16>(p, maxmin, use_heavy, num_heavy, ns, st);
  if (vb == 8) return dispatch_vb<__nv_bfloat16, 8>(p, maxmin, use_heavy, num_heavy, ns, st);
  if (vb == 4) return dispatch_vb<__nv_bfloat16, 4>(p, maxmin, use_heavy, num_heavy, ns, st);
  return dispatch_vb<__nv_bfloat16, 2>(p, maxmin, false, 0, ns, st);
}

}  // namespace gm
