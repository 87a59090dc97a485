// placeholder, replaced by the tcgen05 kernel
#include "gm_common.cuh"
extern "C" {
GM_API size_t gm_segment_matmul_workspace(int64_t, int64_t, int64_t) { return 0; }
GM_API gm_status gm_segment_matmul(const void*, const int64_t*, int64_t, int64_t, int64_t, const void*,
                                   gm_dtype, void*, void*, size_t, gm_stream_t) {
  return gm::fail(GM_ERR_UNSUPPORTED, "segment_matmul: not built");
}
}
