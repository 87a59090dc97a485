// maxbwd.cu — backward of the max / min aggregation path
// (message_passing.hpp:508-514): the gradient of output (v, j) lands on the
// grouped position whose edge attained the extremum (aggregate.hpp:295-308,
// argpos scatter), then gather_rows' adjoint adds every grouped position's
// row into dx[src] in ascending grouped (CSC) position (tensor.hpp:510-524).
//
// Gather form, no atomics: per source s, its entries in ascending CSC
// position — the "source view" (rowptr by source, col = destination v,
// perm = COO edge id), i.e. the CSR by source ordered by (v, COO position)
// instead of COO position — and
//   dx[s][j] = sum_t (arg[v_t][j] == eid_t) ? g[v_t][j] : 0     in t order.
// Positions that did not win contribute exact zeros in the reference, which
// never change a sum started at +0 under round-to-nearest, so skipping them is
// bit-identical. Each output element is accumulated by one lane, sequentially.
//
// Traffic per edge: the argmax slice of the destination row (4 B per column),
// the gradient only where a column matches (sparse), plus col/eid.
#include <algorithm>

#include "vec.cuh"

namespace gm {
namespace mb {

constexpr int kU = 8;  // entries in flight per batch

template <typename S, int V>
struct Lane {  // V consecutive columns of one row
  using IV = typename std::conditional<V == 4, int4, typename std::conditional<V == 2, int2, int>::type>::type;
  using SV = typename std::conditional<
      V == 1, S, typename std::conditional<sizeof(S) == 4, typename std::conditional<V == 4, float4, float2>::type,
                                           double2>::type>::type;
};

template <typename T, int V>
__device__ __forceinline__ void unpack(const T& r, int32_t* out);
template <>
__device__ __forceinline__ void unpack<int4, 4>(const int4& r, int32_t* o) { o[0] = r.x; o[1] = r.y; o[2] = r.z; o[3] = r.w; }
template <>
__device__ __forceinline__ void unpack<int2, 2>(const int2& r, int32_t* o) { o[0] = r.x; o[1] = r.y; }
template <>
__device__ __forceinline__ void unpack<int, 1>(const int& r, int32_t* o) { o[0] = r; }

template <typename S, int V, typename SV>
__device__ __forceinline__ void unpack_s(const SV& r, S* o) {
  if constexpr (V == 1) {
    o[0] = r;
  } else if constexpr (V == 2) {
    o[0] = r.x;
    o[1] = r.y;
  } else {
    o[0] = r.x;
    o[1] = r.y;
    o[2] = r.z;
    o[3] = r.w;
  }
}

// Light rows: one warp per heavy-free window of consecutive source rows; lane
// l owns columns [(base + l) * V, +V) of every row, in passes of 32 lanes.
template <typename S, int V>
__global__ void __launch_bounds__(256) maxbwd_light_kernel(const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const int32_t* __restrict__ eid,
                                                           const int32_t* __restrict__ windows, int64_t num_windows,
                                                           const int32_t* __restrict__ arg, const S* __restrict__ g,
                                                           int64_t f, S* __restrict__ dx) {
  using IV = typename Lane<S, V>::IV;
  using SV = typename Lane<S, V>::SV;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_windows) return;
  const int r0 = windows[2 * w], r1 = windows[2 * w + 1];
  const int64_t nslot = f / V;
  for (int64_t base = 0; base < nslot; base += 32) {
    const int64_t slot = base + lane;
    const bool valid = slot < nslot;
    const int64_t c0 = slot * V;
    for (int r = r0; r < r1; ++r) {
      const int64_t kb = rowptr[r], ke = rowptr[r + 1];
      S acc[V];
#pragma unroll
      for (int x = 0; x < V; ++x) acc[x] = S(0);
      for (int64_t k0 = kb; k0 < ke; k0 += kU) {
        int32_t mv = 0, me = -2;
        if (lane < kU && k0 + lane < ke) {
          mv = col[k0 + lane];
          me = eid[k0 + lane];
        }
        const int nb = static_cast<int>(ke - k0 < kU ? ke - k0 : kU);
        IV a[kU];
        int32_t ev[kU];
        int32_t vv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          vv[u] = __shfl_sync(FULL, mv, u);
          ev[u] = __shfl_sync(FULL, me, u);
          if (valid && u < nb) a[u] = __ldg(reinterpret_cast<const IV*>(arg + static_cast<int64_t>(vv[u]) * f + c0));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (valid && u < nb) {
            int32_t ai[V];
            unpack<IV, V>(a[u], ai);
            bool any = false;
#pragma unroll
            for (int x = 0; x < V; ++x) any |= ai[x] == ev[u];
            if (any) {
              S gv[V];
              unpack_s<S, V, SV>(__ldg(reinterpret_cast<const SV*>(g + static_cast<int64_t>(vv[u]) * f + c0)), gv);
#pragma unroll
              for (int x = 0; x < V; ++x)
                if (ai[x] == ev[u]) acc[x] = add_rn(acc[x], gv[x]);
            }
          }
        }
      }
      if (valid) {
        S* o = dx + static_cast<int64_t>(r) * f + c0;
        if constexpr (V == 1) {
          o[0] = acc[0];
        } else {
          SV ov;
          if constexpr (V == 2) ov = SV{acc[0], acc[1]};
          else ov = SV{acc[0], acc[1], acc[2], acc[3]};
          *reinterpret_cast<SV*>(o) = ov;
        }
      }
    }
  }
}

// Hub rows (deg > the plan's threshold): one warp per (hub row, 32-column
// chunk), one column per lane, entries walked in order in batches of 32
// (metadata) x kU (loads in flight).
template <typename S>
__global__ void __launch_bounds__(128) maxbwd_hub_kernel(const int64_t* __restrict__ rowptr,
                                                         const int32_t* __restrict__ col,
                                                         const int32_t* __restrict__ eid,
                                                         const int32_t* __restrict__ heavy, int64_t num_heavy,
                                                         const int32_t* __restrict__ arg, const S* __restrict__ g,
                                                         int64_t f, S* __restrict__ dx) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t chunks = (f + 31) / 32;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= num_heavy * chunks) return;
  const int r = heavy[w / chunks];
  const int64_t c = (w % chunks) * 32 + lane;
  const bool valid = c < f;
  const int64_t kb = rowptr[r], ke = rowptr[r + 1];
  S acc = S(0);
  for (int64_t m0 = kb; m0 < ke; m0 += 32) {
    const bool has = m0 + lane < ke;
    const int32_t mv = has ? col[m0 + lane] : 0;
    const int32_t me = has ? eid[m0 + lane] : -2;
    const int n = static_cast<int>(ke - m0 < 32 ? ke - m0 : 32);
    for (int u0 = 0; u0 < n; u0 += kU) {
      int32_t a[kU], ev[kU], vv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        vv[u] = __shfl_sync(FULL, mv, u0 + u);
        ev[u] = __shfl_sync(FULL, me, u0 + u);
        a[u] = (valid && u0 + u < n) ? __ldg(arg + static_cast<int64_t>(vv[u]) * f + c) : -3;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (a[u] == ev[u]) acc = add_rn(acc, __ldg(g + static_cast<int64_t>(vv[u]) * f + c));
    }
  }
  if (valid) dx[static_cast<int64_t>(r) * f + c] = acc;
}

__global__ void widen_kernel(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void entry_rows64_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int64_t* __restrict__ out) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) out[k - rowptr[0]] = r;
}

__global__ void gather_ids_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ idx, int64_t n,
                                  int32_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = ids[idx[i]];
}

inline unsigned grid_of(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), kNumSMs * 32)));
}

struct SourceViewWs {
  int64_t* keys;
  int64_t* vals;
  int32_t* pos;
  unsigned char* build;
  size_t build_bytes;
  size_t bytes;
};

inline SourceViewWs source_view_layout(void* base, int64_t nnz, int64_t n_src) {
  SourceViewWs w{};
  unsigned char* p = static_cast<unsigned char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = p ? p + off : nullptr;
    off += align_up(std::max<size_t>(bytes, 1), 256);
    return q;
  };
  w.keys = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(nnz)));
  w.vals = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * static_cast<size_t>(nnz)));
  w.pos = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(nnz)));
  w.build_bytes = gm_build_compressed_workspace(nnz, n_src);
  w.build = take(w.build_bytes);
  w.bytes = off;
  return w;
}

template <typename S>
gm_status launch_bwd(const gm_csr* v, const gm_spmm_plan* plan, const int32_t* arg, const S* g, int64_t f, S* dx,
                     cudaStream_t st) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dx) |
                       reinterpret_cast<uintptr_t>(arg);
  const unsigned lgrid = static_cast<unsigned>(ceil_div(std::max<int64_t>(plan->num_light_windows, 1) * 32, 256));
  if (plan->num_light_windows > 0) {
    bool done = false;
    if constexpr (sizeof(S) == 4) {
      if (f % 4 == 0 && al % 16 == 0) {
        maxbwd_light_kernel<S, 4><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                         plan->num_light_windows, arg, g, f, dx);
        done = true;
      }
    }
    if (done) {
    } else if (f % 2 == 0 && al % (2 * sizeof(S)) == 0 && al % 8 == 0)
      maxbwd_light_kernel<S, 2><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                       plan->num_light_windows, arg, g, f, dx);
    else
      maxbwd_light_kernel<S, 1><<<lgrid, 256, 0, st>>>(v->rowptr, v->col, v->perm, plan->light_windows,
                                                       plan->num_light_windows, arg, g, f, dx);
    GM_CHECK_LAUNCH("maxbwd_light_kernel");
  }
  if (plan->num_heavy > 0) {
    const int64_t warps = plan->num_heavy * ceil_div(f, 32);
    maxbwd_hub_kernel<S><<<static_cast<unsigned>(ceil_div(warps * 32, 128)), 128, 0, st>>>(
        v->rowptr, v->col, v->perm, plan->heavy_rows, plan->num_heavy, arg, g, f, dx);
    GM_CHECK_LAUNCH("maxbwd_hub_kernel");
  }
  return GM_OK;
}

}  // namespace mb
}  // namespace gm

using namespace gm;

extern "C" {

GM_API size_t gm_source_view_workspace(int64_t nnz, int64_t n_src) {
  if (nnz < 0 || n_src < 0) return 0;
  return mb::source_view_layout(nullptr, nnz, n_src).bytes;
}

GM_API gm_status gm_source_view(const gm_csr* csc, int64_t n_src, int64_t* rowptr, int32_t* col, int32_t* eid,
                                void* workspace, size_t workspace_bytes, gm_stream_t stream) {
  GM_REQUIRE(csc && rowptr, GM_ERR_INVALID_ARGUMENT, "gm_source_view: null argument");
  GM_REQUIRE(csc->nnz >= 0 && n_src >= 0 && csc->num_rows >= 0, GM_ERR_INVALID_ARGUMENT,
             "gm_source_view: negative size");
  GM_REQUIRE(csc->nnz == 0 || csc->perm, GM_ERR_INVALID_ARGUMENT, "gm_source_view: csc->perm required");
  const mb::SourceViewWs need = mb::source_view_layout(nullptr, csc->nnz, n_src);
  GM_REQUIRE(workspace && workspace_bytes >= need.bytes, GM_ERR_INVALID_ARGUMENT,
             "gm_source_view: workspace too small");
  cudaStream_t st = as_stream(stream);
  const mb::SourceViewWs w = mb::source_view_layout(workspace, csc->nnz, n_src);
  const int64_t nnz = csc->nnz;
  if (nnz > 0) {
    // keys = the CSC's source ids, values = its destination rows, in CSC order
    int64_t k0 = 0;
    GM_TRY_CUDA(cudaMemcpyAsync(&k0, csc->rowptr, sizeof(k0), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    mb::widen_kernel<<<mb::grid_of(nnz), 256, 0, st>>>(csc->col + k0, nnz, w.keys);
    GM_CHECK_LAUNCH("widen_kernel");
    mb::entry_rows64_kernel<<<mb::grid_of(csc->num_rows), 256, 0, st>>>(csc->rowptr, csc->num_rows, w.vals);
    GM_CHECK_LAUNCH("entry_rows64_kernel");
  }
  // stable counting sort by source: per source, ascending CSC position
  gm_status s = gm_build_compressed(w.keys, w.vals, nnz, n_src, rowptr, col, w.pos, w.build, w.build_bytes, stream);
  if (s != GM_OK) return s;
  if (nnz > 0) {
    int64_t k0 = 0;
    GM_TRY_CUDA(cudaMemcpyAsync(&k0, csc->rowptr, sizeof(k0), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    mb::gather_ids_kernel<<<mb::grid_of(nnz), 256, 0, st>>>(csc->perm + k0, w.pos, nnz, eid);
    GM_CHECK_LAUNCH("gather_ids_kernel");
  }
  return GM_OK;
}

GM_API gm_status gm_spmm_max_backward(const gm_csr* source_view, const gm_spmm_plan* plan, gm_dtype dtype,
                                      const int32_t* arg, const void* g, int64_t f, void* dx, gm_stream_t stream) {
  GM_REQUIRE(source_view && plan, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: null view/plan");
  GM_REQUIRE(f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: negative feature width");
  GM_REQUIRE(dtype == GM_F32 || dtype == GM_F64, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: f32/f64 only");
  if (source_view->num_rows == 0 || f == 0) return GM_OK;
  GM_REQUIRE(arg && g && dx, GM_ERR_INVALID_ARGUMENT, "gm_spmm_max_backward: null pointer");
  GM_REQUIRE(source_view->nnz == 0 || source_view->perm, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_max_backward: the source view needs edge ids (perm)");
  cudaStream_t st = as_stream(stream);
  if (dtype == GM_F32)
    return mb::launch_bwd<float>(source_view, plan, arg, static_cast<const float*>(g), f, static_cast<float*>(dx), st);
  return mb::launch_bwd<double>(source_view, plan, arg, static_cast<const double*>(g), f, static_cast<double*>(dx), st);
}

}  // extern "C"
