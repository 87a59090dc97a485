// spmm.cu — CSR SpMM aggregation (sum / mean / max / min, optional edge
// scale or fused GCN norm, optional argmax) for sm_100a.
//
// Replaces, bit-exactly for f32/f64:
//   spmm / detail::spmm_forward     message_passing.hpp:47-85, 92-169
//   max path (fused, no E x F temp) message_passing.hpp:508-514 ->
//                                   dst_grouped_order 190-214, gather_rows
//                                   tensor.hpp:499-530, aggregate 197-215
//   GCN norm fused into the gather  message_passing.hpp:437-463, 490-495
//
// Exactness: every output element is accumulated by ONE thread, sequentially
// in compressed (CSC) order, with __fadd_rn/__fmul_rn (no FMA contraction) —
// the reference's `o[j] += w * xi[j]` loop order. Max/min: the first element
// initialises, then strict compare; ties keep the earlier edge.
//
// Scheduling (pure performance, never changes results):
//   * light rows (deg <= heavy_threshold): a group of LPR lanes owns one
//     nnz-balanced window of consecutive rows; lanes own VB-byte column
//     slices, U edges' gathers are in flight per batch (coalesced 128-bit
//     loads of whole feature rows, L1 no-allocate);
//   * heavy rows (power-law hubs): one CTA per row, longest first, on a forked
//     stream so hubs start before the light sweep; the CTA streams the row's
//     feature rows into a cp.async shared-memory ring (R stages of `se` edges)
//     while the owning threads accumulate each column in order.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "spmm_kernels.cuh"

namespace gm {

// ---------------------------------------------------------------------------
// Plan: nnz+row balanced windows and the hub list.
// ---------------------------------------------------------------------------
// Window size (edges + rows per light window). Larger windows amortise each
// warp's setup and row-boundary work; too few windows starve the machine. Auto:
// 1024, halved (down to 256) until the sweep has >= 8 waves of resident warps
// (148 SMs x 32). C4 same box, window 128 / 256 / 512 / 768 / 1024 / 2048 /
// 4096: sum 4.28 / 4.24 / 4.22 / 4.21 / 4.20 / 4.21 / 4.34 ms; C5 79.0 -> 76.3
// ms at 1024; the C3 relation SpMM (7.9 M entries) 0.60 -> 0.64 ms at 1024,
// hence the wave floor. Rows >= 1 KB wide (C2) keep 256 (plan_host->window_edges,
// set by the caller: C2 max 68.5 vs 70.1 ms at 1024).
constexpr int64_t kMinWindowCost = 256;
constexpr int64_t kMaxWindowCost = 1024;
static int64_t auto_window_cost(int64_t num_rows, int64_t nnz) {
  int64_t c = kMaxWindowCost;
  while (c > kMinWindowCost && (nnz + num_rows) / c < int64_t{kNumSMs} * 32 * 8) c /= 2;
  return c;
}
constexpr int64_t kHeavyThresholdDefault = 1024;
// Rows longer than this go to the CTA-per-row hub kernel (GM_HEAVY_THR overrides; tuning only).
static int64_t heavy_threshold() {
  static const int64_t thr = [] {
    const char* e = getenv("GM_HEAVY_THR");
    return e ? std::max<int64_t>(64, atoll(e)) : kHeavyThresholdDefault;
  }();
  return thr;
}

__global__ void plan_windows_kernel(const int64_t* __restrict__ rowptr, int64_t num_rows,
                                    int64_t num_windows, int64_t cost, int32_t* __restrict__ win_row) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g > num_windows) return;
  if (g == num_windows) {
    win_row[g] = static_cast<int32_t>(num_rows);
    return;
  }
  // rowptr may be a row slice of a larger CSR: offsets are relative to rowptr[0]
  const int64_t target = g * cost + rowptr[0];
  // first r in [0, num_rows] with rowptr[r] + r >= target
  int64_t lo = 0, hi = num_rows;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rowptr[mid] + mid >= target) hi = mid;
    else lo = mid + 1;
  }
  win_row[g] = static_cast<int32_t>(lo);
}

__global__ void plan_heavy_kernel(const int64_t* __restrict__ rowptr, int64_t num_rows,
                                  int64_t thr, int64_t cap, unsigned long long* __restrict__ keys,
                                  unsigned int* __restrict__ count) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= num_rows) return;
  const int64_t d = rowptr[r + 1] - rowptr[r];
  if (d > thr) {
    const unsigned int i = atomicAdd(count, 1u);
    if (i < cap) keys[i] = (static_cast<unsigned long long>(d) << 32) | static_cast<unsigned long long>(r);
  }
}

constexpr int kDegBuckets = 65536;  // out-degrees >= 65535 share the hottest bucket

__global__ void src_degree_kernel(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ deg) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&deg[col[k]], 1);
}
__global__ void deg_hist_kernel(const int32_t* __restrict__ deg, int64_t n, int32_t* __restrict__ hist) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&hist[min(deg[i], kDegBuckets - 1)], 1);
}
__global__ void src_class_kernel(const int32_t* __restrict__ col, int64_t nnz, const int32_t* __restrict__ deg,
                                 const uint8_t* __restrict__ table, uint8_t* __restrict__ cls) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cls[k] = table[min(deg[col[k]], kDegBuckets - 1)];
}

static int64_t plan_num_windows(int64_t num_rows, int64_t nnz, int64_t cost = kMinWindowCost) {
  return std::max<int64_t>(1, ceil_div(nnz + num_rows, cost));
}
static int64_t plan_heavy_cap(int64_t num_rows, int64_t nnz) {
  return std::min<int64_t>(num_rows, nnz / heavy_threshold() + 1);
}


static thread_local SideStream t_side;

gm_status side_stream(SideStream** out) {
  int dev = 0;
  GM_TRY_CUDA(cudaGetDevice(&dev));
  if (t_side.side == nullptr || t_side.device != dev) {
    GM_TRY_CUDA(cudaStreamCreateWithFlags(&t_side.side, cudaStreamNonBlocking));
    GM_TRY_CUDA(cudaEventCreateWithFlags(&t_side.fork, cudaEventDisableTiming));
    GM_TRY_CUDA(cudaEventCreateWithFlags(&t_side.join, cudaEventDisableTiming));
    t_side.device = dev;
  }
  *out = &t_side;
  return GM_OK;
}

}  // namespace gm

using namespace gm;

extern "C" {

GM_API size_t gm_spmm_plan_bytes(int64_t num_rows, int64_t num_cols, int64_t nnz) {
  if (num_rows < 0 || nnz < 0 || num_cols < 0) return 0;
  const int64_t g = plan_num_windows(num_rows, nnz);
  size_t b = align_up(static_cast<size_t>(g + 1) * sizeof(int32_t), 256);
  b += align_up(static_cast<size_t>(plan_heavy_cap(num_rows, nnz)) * sizeof(int32_t), 256);
  b += align_up(static_cast<size_t>(plan_heavy_cap(num_rows, nnz)) * sizeof(unsigned long long), 256);
  b += 256;  // counter
  b += align_up(static_cast<size_t>(2 * (g + plan_heavy_cap(num_rows, nnz))) * sizeof(int32_t), 256);
  b += align_up(static_cast<size_t>(num_cols) * sizeof(int32_t), 256);  // source out-degrees
  b += align_up(kDegBuckets * sizeof(int32_t), 256);                   // degree histogram
  b += align_up(kDegBuckets, 256);                                     // degree -> class
  b += align_up(static_cast<size_t>(nnz), 256);                        // per-entry class
  return b;
}

GM_API gm_status gm_spmm_plan_build(const gm_csr* csr, void* buffer, size_t buffer_bytes,
                                    gm_spmm_plan* plan, gm_stream_t stream) {
  GM_REQUIRE(csr && plan, GM_ERR_INVALID_ARGUMENT, "gm_spmm_plan_build: null argument");
  GM_REQUIRE(csr->num_rows >= 0 && csr->nnz >= 0 && csr->num_rows < INT32_MAX && csr->nnz < INT32_MAX,
             GM_ERR_INVALID_ARGUMENT, "gm_spmm_plan_build: sizes must be in [0, 2^31)");
  const size_t need = gm_spmm_plan_bytes(csr->num_rows, csr->num_cols, csr->nnz);
  GM_REQUIRE(buffer_bytes >= need, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_plan_build: buffer too small (" + std::to_string(buffer_bytes) + " < " +
                 std::to_string(need) + ")");
  cudaStream_t st = as_stream(stream);
  // a caller-set window size (plan_host->window_edges > 0, clamped to [256, 4096]) or the auto rule;
  // gm_spmm_plan_bytes sized every region for the smallest auto window
  const int64_t cost = plan->window_edges > 0 ? std::min<int64_t>(4096, std::max<int64_t>(kMinWindowCost, plan->window_edges))
                                              : auto_window_cost(csr->num_rows, csr->nnz);
  const int64_t g = plan_num_windows(csr->num_rows, csr->nnz, cost);
  // a caller-set threshold (>= the default) selects fewer hub rows
  const int64_t thr = std::max<int64_t>(heavy_threshold(), plan->heavy_threshold);
  const int64_t cap = plan_heavy_cap(csr->num_rows, csr->nnz);
  unsigned char* b = static_cast<unsigned char*>(buffer);
  int32_t* win_row = reinterpret_cast<int32_t*>(b);
  b += align_up(static_cast<size_t>(g + 1) * sizeof(int32_t), 256);
  int32_t* heavy_rows = reinterpret_cast<int32_t*>(b);
  b += align_up(static_cast<size_t>(cap) * sizeof(int32_t), 256);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(b);
  b += align_up(static_cast<size_t>(cap) * sizeof(unsigned long long), 256);
  unsigned int* count = reinterpret_cast<unsigned int*>(b);
  b += 256;
  int32_t* light = reinterpret_cast<int32_t*>(b);
  b += align_up(static_cast<size_t>(2 * (g + cap)) * sizeof(int32_t), 256);
  int32_t* sdeg = reinterpret_cast<int32_t*>(b);
  b += align_up(static_cast<size_t>(csr->num_cols) * sizeof(int32_t), 256);
  int32_t* dhist = reinterpret_cast<int32_t*>(b);
  b += align_up(kDegBuckets * sizeof(int32_t), 256);
  uint8_t* dtable = b;
  b += align_up(kDegBuckets, 256);
  uint8_t* cls = b;

  plan_windows_kernel<<<static_cast<unsigned>(ceil_div(g + 1, 256)), 256, 0, st>>>(
      csr->rowptr, csr->num_rows, g, cost, win_row);
  GM_CHECK_LAUNCH("plan_windows_kernel");
  GM_TRY_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned int), st));
  if (csr->num_rows > 0) {
    plan_heavy_kernel<<<static_cast<unsigned>(ceil_div(csr->num_rows, 256)), 256, 0, st>>>(
        csr->rowptr, csr->num_rows, thr, cap, keys, count);
    GM_CHECK_LAUNCH("plan_heavy_kernel");
  }
  unsigned int n_heavy = 0;
  GM_TRY_CUDA(cudaMemcpyAsync(&n_heavy, count, sizeof(n_heavy), cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> wr(static_cast<size_t>(g + 1));
  GM_TRY_CUDA(cudaMemcpyAsync(wr.data(), win_row, (g + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GM_TRY_CUDA(cudaStreamSynchronize(st));
  const int64_t nh = std::min<int64_t>(n_heavy, cap);
  std::vector<int32_t> heavy_sorted;
  if (nh > 0) {
    std::vector<unsigned long long> hk(static_cast<size_t>(nh));
    GM_TRY_CUDA(cudaMemcpyAsync(hk.data(), keys, nh * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    std::sort(hk.begin(), hk.end(), [](unsigned long long a, unsigned long long b) { return a > b; });
    std::vector<int32_t> rows(static_cast<size_t>(nh));
    for (int64_t i = 0; i < nh; ++i) rows[static_cast<size_t>(i)] = static_cast<int32_t>(hk[static_cast<size_t>(i)] & 0xffffffffull);
    GM_TRY_CUDA(cudaMemcpyAsync(heavy_rows, rows.data(), nh * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    heavy_sorted = rows;
    std::sort(heavy_sorted.begin(), heavy_sorted.end());
  }
  // heavy-free windows: split every window around the heavy rows inside it
  std::vector<int32_t> lw;
  lw.reserve(static_cast<size_t>(2 * (g + nh)));
  size_t hi = 0;
  for (int64_t w = 0; w < g; ++w) {
    int32_t a = wr[static_cast<size_t>(w)];
    const int32_t bnd = wr[static_cast<size_t>(w) + 1];
    while (hi < heavy_sorted.size() && heavy_sorted[hi] < a) ++hi;
    while (hi < heavy_sorted.size() && heavy_sorted[hi] < bnd) {
      const int32_t h = heavy_sorted[hi++];
      if (a < h) {
        lw.push_back(a);
        lw.push_back(h);
      }
      a = h + 1;
    }
    if (a < bnd) {
      lw.push_back(a);
      lw.push_back(bnd);
    }
  }
  if (!lw.empty()) {
    GM_TRY_CUDA(cudaMemcpyAsync(light, lw.data(), lw.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
  }
  plan->num_windows = g;
  plan->window_edges = cost;
  plan->num_heavy = nh;
  plan->heavy_threshold = thr;
  plan->win_row = win_row;
  plan->heavy_rows = heavy_rows;
  plan->num_light_windows = static_cast<int64_t>(lw.size() / 2);
  plan->light_windows = light;

  // source hotness classes for the L2 residency hint
  plan->src_class = nullptr;
  plan->l2_hot_bytes = 0;
  for (int c = 0; c < GM_PLAN_CLASSES; ++c) plan->hot_edge_frac[c] = 0.f;
  if (csr->num_cols > 0 && csr->nnz > 0) {
    GM_TRY_CUDA(cudaMemsetAsync(sdeg, 0, csr->num_cols * sizeof(int32_t), st));
    GM_TRY_CUDA(cudaMemsetAsync(dhist, 0, kDegBuckets * sizeof(int32_t), st));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(csr->nnz, 256), kNumSMs * 16));
    // a row slice's entries start at rowptr[0]
    int64_t k0 = 0;
    GM_TRY_CUDA(cudaMemcpyAsync(&k0, csr->rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    src_degree_kernel<<<grid, 256, 0, st>>>(csr->col + k0, csr->nnz, sdeg);
    GM_CHECK_LAUNCH("src_degree_kernel");
    deg_hist_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(csr->num_cols, 256), kNumSMs * 16)), 256, 0, st>>>(
        sdeg, csr->num_cols, dhist);
    GM_CHECK_LAUNCH("deg_hist_kernel");
    std::vector<int32_t> hist(kDegBuckets);
    GM_TRY_CUDA(cudaMemcpyAsync(hist.data(), dhist, kDegBuckets * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    std::vector<uint8_t> table(kDegBuckets);
    int64_t greater = 0;  // rows with a strictly larger out-degree
    for (int d = kDegBuckets - 1; d >= 0; --d) {
      const double c = std::floor(4.0 * std::log2(1.0 + static_cast<double>(greater)));
      table[static_cast<size_t>(d)] = static_cast<uint8_t>(std::min(255.0, c));
      greater += hist[static_cast<size_t>(d)];
    }
    // share of the entries whose source class is < c (the hint's L2 coverage)
    std::vector<double> cls_edges(256, 0.0);
    double all_edges = 0.0;
    for (int d = 0; d < kDegBuckets; ++d) {
      const double e = static_cast<double>(d) * hist[static_cast<size_t>(d)];
      cls_edges[table[static_cast<size_t>(d)]] += e;
      all_edges += e;
    }
    double run = 0.0;
    for (int c = 0; c < GM_PLAN_CLASSES; ++c) {
      plan->hot_edge_frac[c] = all_edges > 0 ? static_cast<float>(run / all_edges) : 0.f;
      run += cls_edges[static_cast<size_t>(c)];
    }
    GM_TRY_CUDA(cudaMemcpyAsync(dtable, table.data(), kDegBuckets, cudaMemcpyHostToDevice, st));
    src_class_kernel<<<grid, 256, 0, st>>>(csr->col + k0, csr->nnz, sdeg, dtable, cls + 0);
    GM_CHECK_LAUNCH("src_class_kernel");
    GM_TRY_CUDA(cudaStreamSynchronize(st));
    plan->src_class = cls - k0;  // indexed by global compressed position
    const char* env = getenv("GM_L2_HOT_MB");
    plan->l2_hot_bytes = (env ? atoll(env) : 64) << 20;
  }
  return GM_OK;
}

// GM_NARROW_8B=0 keeps 16-byte vectors for 129..256-byte rows (comparison only).
static bool narrow_rows_8b() {
  static const bool on = [] { const char* e = getenv("GM_NARROW_8B"); return !e || atoi(e) != 0; }();
  return on;
}

static gm_status spmm_impl(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype,
                           const void* x, int64_t f, const void* edge_weight,
                           const gm_gcn_norm* gcn, gm_reduce reduce, void* out, int32_t* arg_out,
                           int accum, const int32_t* mean_deg, gm_stream_t stream,
                           const gm_spmm_epilogue* ep = nullptr) {
  GM_REQUIRE(csr && plan, GM_ERR_INVALID_ARGUMENT, "gm_spmm: null csr/plan");
  GM_REQUIRE(f >= 0, GM_ERR_INVALID_ARGUMENT, "gm_spmm: negative feature width");
  GM_REQUIRE(!(edge_weight && gcn), GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: edge_weight and gcn norm are exclusive");
  const bool maxmin = reduce == GM_MAX || reduce == GM_MIN;
  GM_REQUIRE(reduce >= GM_SUM && reduce <= GM_MIN, GM_ERR_INVALID_ARGUMENT, "gm_spmm: bad reduce");
  GM_REQUIRE(!arg_out || maxmin, GM_ERR_INVALID_ARGUMENT, "gm_spmm: arg_out needs max/min");
  GM_REQUIRE(!arg_out || csr->perm || csr->nnz == 0, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: arg_out needs csr->perm");
  GM_REQUIRE(reinterpret_cast<uintptr_t>(arg_out) % 16 == 0, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: arg_out must be 16-byte aligned");
  GM_REQUIRE(!gcn || (gcn->deg_src && gcn->deg_dst), GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: gcn norm needs both degree arrays");
  GM_REQUIRE(!gcn || !(gcn->bias || gcn->relu) || reduce == GM_SUM || reduce == GM_MEAN, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: the bias/relu epilogue applies to sum/mean");
  const bool carry = ep && ep->carry_mode != GM_CARRY_NONE;
  const bool push = ep && ep->n_push > 0;
  GM_REQUIRE(!carry || (dtype == GM_BF16 && !maxmin && ep->carry && ep->carry_mode <= GM_CARRY_FINISH),
             GM_ERR_INVALID_ARGUMENT, "gm_spmm_ex: the fp32 carry applies to bf16 sum/mean");
  GM_REQUIRE(!carry || (ep->carry_mode == GM_CARRY_START) == (accum == 0), GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_ex: GM_CARRY_START starts the rows (accumulate = 0); CONTINUE/FINISH continue them");
  GM_REQUIRE(!push || (ep->n_push <= GM_MAX_PUSH && !gcn), GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_ex: push targets <= GM_MAX_PUSH peers (no fused GCN term)");
  GM_REQUIRE(!(carry && push && ep->carry_mode != GM_CARRY_FINISH), GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_ex: rows are pushed by the block that finishes them");
  GM_REQUIRE(!(carry || push) || !edge_weight, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_ex: the carry / push epilogue takes unweighted layers");
  if (csr->num_rows == 0 || f == 0) return GM_OK;
  GM_REQUIRE(x && out, GM_ERR_INVALID_ARGUMENT, "gm_spmm: null x/out");
  if (push)
    for (int q = 0; q < ep->n_push; ++q)
      GM_REQUIRE(ep->push_dst[q] != nullptr, GM_ERR_INVALID_ARGUMENT, "gm_spmm_ex: null push target");

  const size_t esz = dtype == GM_F64 ? 8 : dtype == GM_F32 ? 4 : 2;
  const size_t rowbytes = static_cast<size_t>(f) * esz;
  uintptr_t align = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out);
  if (push)
    for (int q = 0; q < ep->n_push; ++q) align |= reinterpret_cast<uintptr_t>(ep->push_dst[q]);
  int vb = 16;
  while (vb > static_cast<int>(esz) && (rowbytes % vb != 0 || align % vb != 0)) vb >>= 1;
  GM_REQUIRE(rowbytes % vb == 0 && align % vb == 0, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm: x/out must be element-aligned");
  // 129..256-byte rows (e.g. F=128 bf16, F=64 f32): 8-byte vectors put the row
  // on all 32 lanes (the flat kernel then keeps 16 edges in flight per batch)
  if (vb == 16 && rowbytes > 128 && rowbytes <= 256 && narrow_rows_8b()) vb = 8;
  const int64_t ns = static_cast<int64_t>(rowbytes / vb);

  SpmmArgs p{};
  p.rowptr = csr->rowptr;
  p.col = csr->col;
  p.perm = csr->perm;
  p.x = x;
  p.out = out;
  p.arg = arg_out;
  p.w = edge_weight;
  p.gdeg_src = gcn ? gcn->deg_src : nullptr;
  p.gdeg_dst = gcn ? gcn->deg_dst : nullptr;
  p.gcn_self = gcn ? gcn->self_loops : 0;
  p.bias = gcn ? gcn->bias : nullptr;
  p.relu = gcn ? gcn->relu : 0;
  p.mean = reduce == GM_MEAN;
  p.is_min = reduce == GM_MIN;
  p.accum = accum;
  p.mean_deg = mean_deg;
  if (carry) {
    p.carry = ep->carry;
    p.carry_out = ep->carry_mode == GM_CARRY_FINISH;
  }
  if (push) {
    p.n_push = ep->n_push;
    for (int q = 0; q < ep->n_push; ++q) p.push_dst[q] = ep->push_dst[q];
    p.push_row0 = ep->push_row0;
    p.push_mask = ep->push_mask;
  }
  p.num_rows = csr->num_rows;
  p.f = f;
  p.win_row = plan->win_row;
  p.num_windows = plan->num_windows;
  p.heavy_rows = plan->heavy_rows;
  p.light_windows = plan->light_windows;
  p.num_light_windows = plan->num_light_windows;
  // cp.async moves >= 4-byte granules: narrower rows keep hubs on the light path
  const bool use_heavy = plan->num_heavy > 0 && vb >= 4;
  p.heavy_thr = use_heavy ? plan->heavy_threshold : INT64_MAX;
  p.flat_ok = plan->num_heavy == 0 || use_heavy;
  p.src_class = nullptr;
  p.hot_class_limit = 0;
  // X much larger than L2 streams: every gather carries an eviction policy
  static const int stream_env = [] { const char* e = getenv("GM_STREAM_X"); return e ? atoi(e) : -1; }();
  p.stream_x = stream_env >= 0 ? stream_env
                               : static_cast<double>(csr->num_cols) * static_cast<double>(rowbytes) > 64.0 * (1 << 20);
  // L2 column blocking, an A/B variant (GM_L2_BLOCK_MB = budget in MB; unset/0
  // disables): when X is far larger than L2 but its rows are re-read many times
  // (E >= 16 x source rows) and a column block of >= 128 bytes per row fits the
  // budget, the columns are processed block by block so each block's gathers
  // can hit L2 after the first touch. Bit-identical, but on Reddit-shaped C2
  // (233k rows of 2408 bytes, 492 reads per row) mean 53.7 -> 84-128 ms and max
  // 64 -> 165-259 ms for budgets of 32-96 MB: a 256-byte block still misses L2
  // on 45% of its sectors (9.5 GB of DRAM per block) while every block repeats
  // the per-edge metadata and issue work of the sweep (profiles/r02l2b_*)
  static const double blk_mb = [] { const char* e = getenv("GM_L2_BLOCK_MB"); return e ? atof(e) : 0.0; }();
  if (blk_mb > 0 && p.stream_x && stream_env < 0 && csr->num_cols > 0 && csr->nnz >= 16 * csr->num_cols &&
      gcn == nullptr) {
    const int64_t fit = static_cast<int64_t>(blk_mb * (1 << 20) / static_cast<double>(csr->num_cols)) / vb;
    if (fit * vb >= 128 && fit < ns) {
      p.l2_block_slots = fit >= 32 ? fit / 32 * 32 : fit;
      p.stream_x = 0;  // block rows are meant to stay: default-priority gathers
    }
  }
  if (p.l2_block_slots == 0 && plan->src_class && plan->l2_hot_bytes > 0) {
    // rows that fit the budget: rank < hot_rows  <=>  class < floor(4*log2(1 + hot_rows))
    const double hot_rows = static_cast<double>(plan->l2_hot_bytes) / static_cast<double>(rowbytes);
    const int limit = static_cast<int>(std::floor(4.0 * std::log2(1.0 + hot_rows)));
    // the hint costs a class byte and a policy select per entry: only worth it
    // when the L2-resident rows serve a large share of the gathers
    static const double min_cover = [] {
      const char* e = getenv("GM_L2_MIN_COVER");
      return e ? atof(e) : 0.15;
    }();
    const double cover = plan->hot_edge_frac[std::min(limit, GM_PLAN_CLASSES - 1)];
    if (cover >= min_cover) {
      p.src_class = plan->src_class;
      p.hot_class_limit = limit;
    }
  }
  cudaStream_t st = as_stream(stream);

  switch (dtype) {
    case GM_F32: return spmm_dispatch_f32(p, maxmin, use_heavy, plan->num_heavy, ns, vb, st);
    case GM_F64: return spmm_dispatch_f64(p, maxmin, use_heavy, plan->num_heavy, ns, vb, st);
    case GM_BF16: return spmm_dispatch_bf16(p, maxmin, use_heavy && vb >= 4, plan->num_heavy, ns, vb, st);
  }
  return fail(GM_ERR_INVALID_ARGUMENT, "gm_spmm: unknown dtype");
}

GM_API gm_status gm_spmm(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype,
                         const void* x, int64_t f, const void* edge_weight,
                         const gm_gcn_norm* gcn, gm_reduce reduce, void* out, int32_t* arg_out,
                         gm_stream_t stream) {
  return spmm_impl(csr, plan, dtype, x, f, edge_weight, gcn, reduce, out, arg_out, 0, nullptr, stream);
}

GM_API gm_status gm_spmm_ex(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype, const void* x, int64_t f,
                            const void* edge_weight, gm_reduce reduce, int32_t accumulate, const int32_t* mean_deg,
                            const gm_spmm_epilogue* epilogue, void* out, int32_t* arg_out, gm_stream_t stream) {
  const bool maxmin = reduce == GM_MAX || reduce == GM_MIN;
  if (accumulate) {
    GM_REQUIRE(!maxmin || arg_out, GM_ERR_INVALID_ARGUMENT,
               "gm_spmm_ex: max/min continuation needs the running arg_out (ties break on COO id)");
    GM_REQUIRE(reduce != GM_MEAN || mean_deg, GM_ERR_INVALID_ARGUMENT,
               "gm_spmm_ex: a continued mean needs the full-row degrees");
    GM_REQUIRE(dtype != GM_BF16 || maxmin || (epilogue && epilogue->carry_mode != GM_CARRY_NONE),
               GM_ERR_INVALID_ARGUMENT, "gm_spmm_ex: continued bf16 sum/mean needs the fp32 carry");
  }
  return spmm_impl(csr, plan, dtype, x, f, edge_weight, nullptr, reduce, out, arg_out, accumulate ? 1 : 0,
                   accumulate ? mean_deg : nullptr, stream, epilogue);
}

GM_API gm_status gm_spmm_accumulate(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype,
                                    const void* x, int64_t f, const void* edge_weight, gm_reduce reduce,
                                    const int32_t* mean_deg, void* out, int32_t* arg_out,
                                    gm_stream_t stream) {
  const bool maxmin = reduce == GM_MAX || reduce == GM_MIN;
  GM_REQUIRE(dtype != GM_BF16 || maxmin, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_accumulate: bf16 sum/mean would round between blocks (use gm_spmm on the gathered x)");
  GM_REQUIRE(!maxmin || arg_out, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_accumulate: max/min needs the running arg_out (ties break on COO id)");
  GM_REQUIRE(reduce != GM_MEAN || mean_deg, GM_ERR_INVALID_ARGUMENT,
             "gm_spmm_accumulate: mean needs the full-row degrees");
  return spmm_impl(csr, plan, dtype, x, f, edge_weight, nullptr, reduce, out, arg_out, 1, mean_deg, stream);
}

}  // extern "C"
