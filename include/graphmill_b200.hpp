// graphmill_b200.hpp — header-only C++ mirror of the reference operator API
// (/root/reference/proj/include/graphmill/{edge_index,message_passing,
// aggregate,hetero}.hpp) over the C-ABI in graphmill_b200.h.
//
// Same names, argument meaning and exception behaviour as the reference:
//   EdgeIndex / EdgeIndexClaims / SortOrder / CsrView   edge_index.hpp:16-127
//   build_compressed                                    edge_index.hpp:120-121
//   spmm (sum | mean, optional edge weight)             message_passing.hpp:92-169
//   neighbor_aggregate (sum | mean | max | min)         message_passing.hpp:500-514
//   gcn_aggregate / gcn_layer / gcn_forward             message_passing.hpp:490-499, 578, 631-641
//   neighbor_aggregate_backward (max | min)             aggregate.hpp:295-308 + tensor.hpp:510-524
//   aggregate (edge rows by index)                      aggregate.hpp:154-215
//   grouped_matmul (bf16 and fp32, per-group tensors)   hetero.hpp:134-157
//   DistSpmm (dst-row partition over an ncclComm_t)
//   PushSpmm (exchange fused into the SpMM epilogue)
// Data lives on the device (DeviceMatrix / DeviceArray); std::invalid_argument,
// std::out_of_range and std::logic_error carry the reference's message shapes.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "graphmill_b200.h"

namespace b200 {

using Index = std::int64_t;
enum class SortOrder { unsorted, by_src, by_dst };
enum class AggKind { sum, mean, max, min };

struct EdgeIndexClaims {
  std::optional<SortOrder> sort_order;
  std::optional<bool> is_undirected;
};

// bf16 storage type for grouped_matmul operands.
struct bf16 {
  std::uint16_t bits = 0;
  static bf16 from_float(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);  // RNE (finite values)
    return bf16{static_cast<std::uint16_t>(u >> 16)};
  }
  float to_float() const {
    std::uint32_t u = static_cast<std::uint32_t>(bits) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
};

namespace detail {
inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
inline void check(gm_status st) {
  switch (st) {
    case GM_OK: return;
    case GM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(gm_last_error());
    case GM_ERR_OUT_OF_RANGE: throw std::out_of_range(gm_last_error());
    case GM_ERR_LOGIC: throw std::logic_error(gm_last_error());
    default: throw std::runtime_error(gm_last_error());
  }
}
inline cudaStream_t& stream_slot() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
template <class S>
constexpr gm_dtype dtype_of() {
  if constexpr (std::is_same_v<S, float>) return GM_F32;
  else if constexpr (std::is_same_v<S, double>) return GM_F64;
  else return GM_BF16;
}
}  // namespace detail

// All calls of this thread go to this stream (default: legacy stream).
inline void set_stream(cudaStream_t s) { detail::stream_slot() = s; }
inline cudaStream_t stream() { return detail::stream_slot(); }

// Caller-side owned device memory (shared, like the reference's shared storage).
template <class T>
class DeviceArray {
 public:
  DeviceArray() = default;
  explicit DeviceArray(std::size_t n) : n_(n) {
    if (n == 0) return;
    void* p = nullptr;
    detail::check_cuda(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    mem_ = std::shared_ptr<void>(p, [](void* q) { cudaFree(q); });
  }
  static DeviceArray from_host(const T* h, std::size_t n) {
    DeviceArray a(n);
    if (n) detail::check_cuda(cudaMemcpy(a.data(), h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    return a;
  }
  static DeviceArray from_host(const std::vector<T>& v) { return from_host(v.data(), v.size()); }
  std::vector<T> to_host() const {
    std::vector<T> v(n_);
    if (n_) {
      detail::check_cuda(cudaStreamSynchronize(stream()), "sync");
      detail::check_cuda(cudaMemcpy(v.data(), data(), n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
    return v;
  }
  T* data() const { return static_cast<T*>(mem_.get()); }
  std::size_t size() const { return n_; }

 private:
  std::shared_ptr<void> mem_;
  std::size_t n_ = 0;
};

template <class S>
class DeviceMatrix {
 public:
  DeviceMatrix() = default;
  DeviceMatrix(Index rows, Index cols) : rows_(rows), cols_(cols), buf_(static_cast<std::size_t>(rows * cols)) {}
  static DeviceMatrix from_host(Index rows, Index cols, const S* h) {
    DeviceMatrix m;
    m.rows_ = rows;
    m.cols_ = cols;
    m.buf_ = DeviceArray<S>::from_host(h, static_cast<std::size_t>(rows * cols));
    return m;
  }
  static DeviceMatrix from_host(Index rows, Index cols, const std::vector<S>& h) {
    if (static_cast<Index>(h.size()) != rows * cols)
      throw std::invalid_argument("tensor: data length does not match shape");
    return from_host(rows, cols, h.data());
  }
  std::vector<S> to_host() const { return buf_.to_host(); }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  S* data() const { return buf_.data(); }

 private:
  Index rows_ = 0, cols_ = 0;
  DeviceArray<S> buf_;
};

// Device CSR (edge_index.hpp:22-29) plus its cached scheduling plan.
class CsrView {
 public:
  DeviceArray<Index> rowptr;
  DeviceArray<std::int32_t> col;
  DeviceArray<std::int32_t> perm;
  Index num_cols = 0;

  Index num_rows() const { return static_cast<Index>(rowptr.size()) - 1; }
  Index num_entries() const { return static_cast<Index>(col.size()); }
  gm_csr c_struct() const {
    return gm_csr{num_rows(), num_cols, num_entries(), rowptr.data(), col.data(), perm.data()};
  }
  const gm_spmm_plan& plan() const {
    std::call_once(plan_->once, [&] {
      const gm_csr c = c_struct();
      const std::size_t bytes = gm_spmm_plan_bytes(c.num_rows, c.num_cols, c.nnz);
      plan_->buf = DeviceArray<unsigned char>(bytes ? bytes : 1);
      detail::check(gm_spmm_plan_build(&c, plan_->buf.data(), bytes, &plan_->plan, stream()));
    });
    return plan_->plan;
  }
  // Host copies in the reference's int64 layout.
  std::vector<Index> rowptr_host() const { return rowptr.to_host(); }
  std::vector<Index> col_host() const { return widen(col.to_host()); }
  std::vector<Index> perm_host() const { return widen(perm.to_host()); }

 private:
  static std::vector<Index> widen(const std::vector<std::int32_t>& v) { return {v.begin(), v.end()}; }
  struct PlanSlot {
    std::once_flag once;
    DeviceArray<unsigned char> buf;
    gm_spmm_plan plan{};
  };
  std::shared_ptr<PlanSlot> plan_ = std::make_shared<PlanSlot>();
};

// edge_index.cpp:45-62 on the device (bit-exact stable counting sort).
inline CsrView build_compressed(const DeviceArray<Index>& keys, const DeviceArray<Index>& values, Index num_rows,
                                Index num_cols = 0, Index count = -1) {
  const Index e = count < 0 ? static_cast<Index>(keys.size()) : count;
  CsrView v;
  v.rowptr = DeviceArray<Index>(static_cast<std::size_t>(num_rows + 1));
  v.col = DeviceArray<std::int32_t>(static_cast<std::size_t>(e));
  v.perm = DeviceArray<std::int32_t>(static_cast<std::size_t>(e));
  v.num_cols = num_cols;
  const std::size_t ws = gm_build_compressed_workspace(e, num_rows);
  DeviceArray<unsigned char> w(ws ? ws : 1);
  detail::check(gm_build_compressed(keys.data(), values.data(), e, num_rows, v.rowptr.data(), v.col.data(),
                                    v.perm.data(), w.data(), ws, stream()));
  return v;
}

// COO edge list with verified claims and demand-filled device CSR/CSC caches
// (edge_index.hpp:43-116). Value type: copies share storage and caches.
class EdgeIndex {
 public:
  EdgeIndex() : cache_(std::make_shared<CacheSlot>()) {}
  EdgeIndex(std::vector<Index> src, std::vector<Index> dst, Index num_src_nodes, Index num_dst_nodes,
            const EdgeIndexClaims& claims = {})
      : num_edges_(static_cast<Index>(src.size())),
        num_src_(num_src_nodes),
        num_dst_(num_dst_nodes),
        cache_(std::make_shared<CacheSlot>()) {
    if (src.size() != dst.size()) throw std::invalid_argument("EdgeIndex: src and dst lengths differ");
    if (num_src_nodes < 0 || num_dst_nodes < 0) throw std::invalid_argument("EdgeIndex: negative node count");
    src_ = DeviceArray<Index>::from_host(src);
    dst_ = DeviceArray<Index>::from_host(dst);
    verify_claims(claims, src, dst);
  }

  const DeviceArray<Index>& src() const { return src_; }
  const DeviceArray<Index>& dst() const { return dst_; }
  Index num_edges() const { return num_edges_; }
  Index num_src_nodes() const { return num_src_; }
  Index num_dst_nodes() const { return num_dst_; }
  SortOrder sort_order() const { return sort_order_; }
  bool is_undirected() const { return undirected_; }

  const CsrView& to_csr() const { return fill_cache(false); }
  const CsrView& to_csc() const { return fill_cache(true); }
  const CsrView& transpose_view() const { return undirected_ ? to_csr() : to_csc(); }
  bool has_csr_cache() const { return cache_->csr.load() != nullptr; }
  bool has_csc_cache() const { return cache_->csc.load() != nullptr; }
  int csr_build_count() const { return cache_->csr_builds.load(); }
  int csc_build_count() const { return cache_->csc_builds.load(); }

  // Effective GCN degrees of this index's FULL arrays, computed once and kept
  // beside its caches (they depend only on the immutable COO arrays).
  std::pair<const std::int32_t*, const std::int32_t*> gcn_degrees() const {
    std::call_once(cache_->gcn_once, [&] {
      const bool square = num_src_ == num_dst_;
      cache_->gcn_dst = DeviceArray<std::int32_t>(static_cast<std::size_t>(num_dst_));
      cache_->gcn_src = square ? cache_->gcn_dst : DeviceArray<std::int32_t>(static_cast<std::size_t>(num_src_));
      detail::check(gm_gcn_degrees(src_.data(), dst_.data(), num_edges_, num_src_, num_dst_, square,
                                   cache_->gcn_src.data(), cache_->gcn_dst.data(), stream()));
    });
    return {cache_->gcn_src.data(), cache_->gcn_dst.data()};
  }

  // Source view (gm_source_view): the gather order of the max/min backward.
  const CsrView& source_view() const {
    std::call_once(cache_->source_once, [&] {
      const CsrView& csc = to_csc();
      auto v = std::make_unique<CsrView>();
      v->rowptr = DeviceArray<Index>(static_cast<std::size_t>(num_src_ + 1));
      v->col = DeviceArray<std::int32_t>(static_cast<std::size_t>(num_edges_));
      v->perm = DeviceArray<std::int32_t>(static_cast<std::size_t>(num_edges_));
      v->num_cols = num_dst_;
      const gm_csr c = csc.c_struct();
      const std::size_t wsb = gm_source_view_workspace(num_edges_, num_src_);
      DeviceArray<unsigned char> w(wsb ? wsb : 1);
      detail::check(gm_source_view(&c, num_src_, v->rowptr.data(), v->col.data(), v->perm.data(), w.data(), wsb,
                                   stream()));
      detail::check_cuda(cudaStreamSynchronize(stream()), "sync");  // workspace dies here
      cache_->source = std::move(v);
    });
    return *cache_->source;
  }

  // Destination grouping used when the per-edge association matters on an
  // undirected index (the reference's COO sweep, message_passing.hpp:51-59):
  // built once, kept OUT of the public CSC cache like the reference.
  const CsrView& exact_dst_grouping() const {
    std::call_once(cache_->exact_once, [&] {
      cache_->exact = std::make_unique<CsrView>(build_compressed(dst_, src_, num_dst_, num_src_, num_edges_));
    });
    return *cache_->exact;
  }

 private:
  struct CacheSlot {
    std::atomic<const CsrView*> csr{nullptr};
    std::atomic<const CsrView*> csc{nullptr};
    std::atomic<int> csr_builds{0};
    std::atomic<int> csc_builds{0};
    std::once_flag exact_once;
    std::unique_ptr<CsrView> exact;
    std::once_flag gcn_once;
    DeviceArray<std::int32_t> gcn_src, gcn_dst;  // effective GCN degrees (message_passing.hpp:441-460)
    std::once_flag source_once;
    std::unique_ptr<CsrView> source;             // per source, entries in ascending CSC position
    ~CacheSlot() {
      delete csr.load();
      delete csc.load();
    }
  };

  const CsrView& fill_cache(bool by_dst) const {
    auto& slot = by_dst ? cache_->csc : cache_->csr;
    if (const CsrView* hit = slot.load(std::memory_order_acquire)) return *hit;
    const CsrView* built = new CsrView(by_dst ? build_compressed(dst_, src_, num_dst_, num_src_, num_edges_)
                                              : build_compressed(src_, dst_, num_src_, num_dst_, num_edges_));
    (by_dst ? cache_->csc_builds : cache_->csr_builds).fetch_add(1);
    const CsrView* expected = nullptr;
    // compute-then-publish (edge_index.cpp:121-136): at most one result wins
    if (!slot.compare_exchange_strong(expected, built, std::memory_order_acq_rel, std::memory_order_acquire)) {
      delete built;
      return *expected;
    }
    return *built;
  }

  static const char* name(SortOrder o) {
    return o == SortOrder::by_src ? "by_src" : o == SortOrder::by_dst ? "by_dst" : "unsorted";
  }

  void verify_claims(const EdgeIndexClaims& claims, const std::vector<Index>& hs, const std::vector<Index>& hd) {
    DeviceArray<unsigned char> ws(64);
    detail::check(gm_check_index_bounds(src_.data(), num_edges_, num_src_, "EdgeIndex: src", ws.data(), stream()));
    detail::check(gm_check_index_bounds(dst_.data(), num_edges_, num_dst_, "EdgeIndex: dst", ws.data(), stream()));
    if (claims.sort_order && *claims.sort_order != SortOrder::unsorted) {
      Index bad = -1;
      const auto& keys = *claims.sort_order == SortOrder::by_src ? src_ : dst_;
      detail::check(gm_first_unsorted(keys.data(), num_edges_, &bad, ws.data(), stream()));
      if (bad >= 0)
        throw std::invalid_argument(std::string("EdgeIndex: claim ") + name(*claims.sort_order) +
                                    " violated at position " + std::to_string(bad));
      sort_order_ = *claims.sort_order;
    }
    if (claims.is_undirected && *claims.is_undirected) {
      if (num_src_ != num_dst_)
        throw std::invalid_argument("EdgeIndex: is_undirected claim requires num_src_nodes == num_dst_nodes");
      // Multiset symmetry (edge_index.cpp:98-118) on the device: the first
      // position whose pair multiplicity differs from its reverse's
      const std::size_t wsb = gm_first_asymmetric_workspace(num_edges_);
      DeviceArray<unsigned char> aw(wsb ? wsb : 1);
      Index bad = -1;
      detail::check(gm_first_asymmetric(src_.data(), dst_.data(), num_edges_, num_src_, &bad, aw.data(), wsb, stream()));
      if (bad >= 0)
        throw std::invalid_argument("EdgeIndex: is_undirected claim violated at position " + std::to_string(bad) +
                                    " (edge " + std::to_string(hs[static_cast<std::size_t>(bad)]) + "->" +
                                    std::to_string(hd[static_cast<std::size_t>(bad)]) + " lacks a matching reverse)");
      undirected_ = true;
    }
  }

  DeviceArray<Index> src_, dst_;
  Index num_edges_ = 0, num_src_ = 0, num_dst_ = 0;
  SortOrder sort_order_ = SortOrder::unsorted;
  bool undirected_ = false;
  std::shared_ptr<CacheSlot> cache_;
};

namespace detail {
template <class S>
using Acc = std::conditional_t<std::is_same_v<S, double>, double, float>;

template <class S>
DeviceMatrix<S> run_spmm(const CsrView& g, const DeviceMatrix<S>& x, AggKind kind, const Acc<S>* w_csr,
                         const gm_gcn_norm* gcn, Index out_rows, DeviceArray<std::int32_t>* argmax) {
  DeviceMatrix<S> out(out_rows, x.cols());
  const gm_csr c = g.c_struct();
  const gm_reduce r = kind == AggKind::sum ? GM_SUM : kind == AggKind::mean ? GM_MEAN : kind == AggKind::max ? GM_MAX : GM_MIN;
  if (argmax) *argmax = DeviceArray<std::int32_t>(static_cast<std::size_t>(out_rows * x.cols()));
  check(gm_spmm(&c, &g.plan(), dtype_of<S>(), x.data(), x.cols(), w_csr, gcn, r, out.data(),
                argmax ? argmax->data() : nullptr, stream()));
  return out;
}

template <class S>
DeviceArray<Acc<S>> permute(const DeviceArray<Acc<S>>& w, const CsrView& g) {
  DeviceArray<Acc<S>> out(w.size());
  check(gm_permute_edge_values(dtype_of<Acc<S>>(), w.data(), g.perm.data(), static_cast<Index>(w.size()), out.data(),
                               stream()));
  return out;
}
}  // namespace detail

// message_passing.hpp:92-169 (forward). Weight in COO order, length E.
template <class S>
DeviceMatrix<S> spmm(const EdgeIndex& e, const DeviceMatrix<S>& x,
                     const std::optional<DeviceMatrix<detail::Acc<S>>>& edge_weight, AggKind reduce) {
  if (reduce != AggKind::sum && reduce != AggKind::mean)
    throw std::invalid_argument("spmm: reduce must be sum or mean");
  if (x.rows() != e.num_src_nodes()) throw std::invalid_argument("spmm: feature rows != num_src_nodes");
  if (edge_weight && edge_weight->rows() * edge_weight->cols() != e.num_edges())
    throw std::invalid_argument("spmm: edge weight length != num_edges");
  if (!edge_weight) return detail::run_spmm<S>(e.transpose_view(), x, reduce, nullptr, nullptr, e.num_dst_nodes(), nullptr);
  const CsrView& g = e.is_undirected() ? e.exact_dst_grouping() : e.transpose_view();
  DeviceArray<detail::Acc<S>> wc(static_cast<std::size_t>(e.num_edges()));
  detail::check(gm_permute_edge_values(detail::dtype_of<detail::Acc<S>>(), edge_weight->data(), g.perm.data(),
                                       e.num_edges(), wc.data(), stream()));
  return detail::run_spmm<S>(g, x, reduce, wc.data(), nullptr, e.num_dst_nodes(), nullptr);
}

// The fused segment path of layer_neighbor_aggregate for identity messages:
// sum/mean via spmm, max/min via dst_grouped_order + gather_rows + aggregate
// (no E x F temporary). argmax (optional): COO edge id, -1 for empty rows.
template <class S>
DeviceMatrix<S> neighbor_aggregate(const EdgeIndex& e, const DeviceMatrix<S>& x, AggKind kind,
                                   DeviceArray<std::int32_t>* argmax = nullptr) {
  if (x.rows() != e.num_src_nodes()) throw std::invalid_argument("propagate: h_src rows != num_src_nodes");
  const bool mm = kind == AggKind::max || kind == AggKind::min;
  return detail::run_spmm<S>(e.transpose_view(), x, kind, nullptr, nullptr, e.num_dst_nodes(), mm ? argmax : nullptr);
}

// GCN neighbour side after the transform (message_passing.hpp:490-495), with
// layer_update's bias (:578) and optionally the model's inter-layer relu (:637)
// fused into the aggregate's epilogue. Degrees are cached on the index.
template <class S>
DeviceMatrix<S> gcn_aggregate(const EdgeIndex& e, const DeviceMatrix<S>& xw,
                              const DeviceArray<detail::Acc<S>>* bias = nullptr, bool relu = false) {
  if (xw.rows() != e.num_src_nodes()) throw std::invalid_argument("spmm: feature rows != num_src_nodes");
  if (bias && static_cast<Index>(bias->size()) != xw.cols())
    throw std::invalid_argument("layer_update: bias length != feature width");
  const bool square = e.num_src_nodes() == e.num_dst_nodes();
  const auto deg = e.gcn_degrees();
  const gm_gcn_norm g{deg.first, deg.second, square ? 1 : 0, bias ? bias->data() : nullptr, relu ? 1 : 0};
  return detail::run_spmm<S>(e.to_csc(), xw, AggKind::sum, nullptr, &g, e.num_dst_nodes(), nullptr);
}

// layer_forward for LayerKind::gcn (message_passing.hpp:490-499, 578): the
// transform on the tcgen05 GEMM (fp32-accurate split route for float), then
// the fused aggregate + bias (+ relu).
inline DeviceMatrix<float> gcn_layer(const EdgeIndex& e, const DeviceMatrix<float>& h, const DeviceMatrix<float>& w,
                                     const DeviceArray<float>& bias, bool relu = false) {
  if (h.rows() != e.num_src_nodes() || e.num_src_nodes() != e.num_dst_nodes())
    throw std::invalid_argument("layer_forward: square index matching h required");
  if (w.rows() != h.cols()) throw std::invalid_argument("matmul: inner dimension mismatch");
  DeviceMatrix<float> xw(h.rows(), w.cols());
  const Index ptr[2] = {0, h.rows()};
  const std::size_t wsb = gm_segment_matmul_f32_workspace(h.rows(), 1, h.cols(), w.cols());
  DeviceArray<unsigned char> ws(wsb ? wsb : 1);
  detail::check(gm_segment_matmul_f32(h.data(), ptr, 1, h.cols(), w.cols(), w.data(), xw.data(), ws.data(), wsb,
                                      stream()));
  auto out = gcn_aggregate<float>(e, xw, &bias, relu);
  detail::check_cuda(cudaStreamSynchronize(stream()), "sync");  // the GEMM workspace dies here
  return out;
}

// Model::forward of a GCN stack (message_passing.hpp:631-641): relu between layers.
inline DeviceMatrix<float> gcn_forward(const EdgeIndex& e, const DeviceMatrix<float>& x,
                                       const std::vector<std::pair<DeviceMatrix<float>, DeviceArray<float>>>& layers) {
  DeviceMatrix<float> h = x;
  for (std::size_t i = 0; i < layers.size(); ++i)
    h = gcn_layer(e, h, layers[i].first, layers[i].second, i + 1 < layers.size());
  return h;
}

// Backward of neighbor_aggregate max/min: dx [num_src, F] from the output
// gradient and the argmax of the forward (aggregate.hpp:295-308, tensor.hpp:510-524).
template <class S>
DeviceMatrix<S> neighbor_aggregate_backward(const EdgeIndex& e, const DeviceMatrix<S>& grad_out,
                                            const DeviceArray<std::int32_t>& argmax) {
  static_assert(!std::is_same_v<S, bf16>, "f32/f64 only");
  if (grad_out.rows() != e.num_dst_nodes())
    throw std::invalid_argument("neighbor_aggregate_backward: grad_out must be [num_dst_nodes, F]");
  if (static_cast<Index>(argmax.size()) != grad_out.rows() * grad_out.cols())
    throw std::invalid_argument("neighbor_aggregate_backward: argmax must match grad_out");
  const CsrView& v = e.source_view();
  DeviceMatrix<S> dx(e.num_src_nodes(), grad_out.cols());
  const gm_csr c = v.c_struct();
  detail::check(gm_spmm_max_backward(&c, &v.plan(), detail::dtype_of<S>(), argmax.data(), grad_out.data(),
                                     grad_out.cols(), dx.data(), stream()));
  return dx;
}

// aggregate.hpp:154-215 for edge-level rows (sum/mean/max/min).
template <class S>
DeviceMatrix<S> aggregate(const DeviceMatrix<S>& values, const std::vector<Index>& index, Index num_groups,
                          AggKind kind) {
  if (values.rows() != static_cast<Index>(index.size()))
    throw std::invalid_argument("aggregate: values rows != index length");
  DeviceArray<Index> idx = DeviceArray<Index>::from_host(index);
  DeviceArray<unsigned char> ws(64);
  detail::check(gm_check_index_bounds(idx.data(), static_cast<Index>(index.size()), num_groups, "aggregate:",
                                      ws.data(), stream()));
  std::vector<Index> pos(index.size());
  for (std::size_t i = 0; i < pos.size(); ++i) pos[i] = static_cast<Index>(i);
  const CsrView g = build_compressed(idx, DeviceArray<Index>::from_host(pos), num_groups, values.rows());
  return detail::run_spmm<S>(g, values, kind, nullptr, nullptr, num_groups, nullptr);
}

// hetero.hpp:134-157: { H_T W_T } for W = [G, F, F'] over separate per-group
// tensors, one gm_grouped_matmul launch (per-group TMA maps: no concatenation,
// no copies). bf16 operands with fp32 output, or fp32 operands on the
// fp32-accurate route (the reference's grouped_matmul<float>).
namespace detail {
template <class X>
std::vector<DeviceMatrix<float>> grouped(const std::vector<DeviceMatrix<X>>& inputs, const void* w, Index groups,
                                         Index f_in, Index f_out) {
  if (static_cast<Index>(inputs.size()) != groups)
    throw std::invalid_argument("grouped_matmul: group count mismatch (" + std::to_string(inputs.size()) +
                                " inputs, " + std::to_string(groups) + " weight slabs)");
  std::vector<Index> rows;
  std::vector<const void*> xs;
  std::vector<void*> os;
  std::vector<DeviceMatrix<float>> outs;
  for (Index g = 0; g < groups; ++g) {
    const auto& h = inputs[static_cast<std::size_t>(g)];
    if (h.cols() != f_in)
      throw std::invalid_argument("grouped_matmul: group " + std::to_string(g) + " inner dimension mismatch");
    rows.push_back(h.rows());
    outs.emplace_back(h.rows(), f_out);
    xs.push_back(h.data());
    os.push_back(outs.back().data());
  }
  const gm_dtype dt = dtype_of<X>();
  const std::size_t wsb = gm_grouped_matmul_workspace(rows.data(), groups, f_in, f_out, dt, dt, GM_F32);
  DeviceArray<unsigned char> ws(wsb ? wsb : 1);
  check(gm_grouped_matmul(xs.data(), rows.data(), groups, f_in, f_out, w, dt, dt, os.data(), GM_F32, ws.data(), wsb,
                          stream()));
  check_cuda(cudaStreamSynchronize(stream()), "sync");  // the workspace dies here
  return outs;
}
}  // namespace detail

inline std::vector<DeviceMatrix<float>> grouped_matmul(const std::vector<DeviceMatrix<bf16>>& inputs,
                                                       const DeviceArray<bf16>& weights, Index groups, Index f_in,
                                                       Index f_out) {
  return detail::grouped<bf16>(inputs, weights.data(), groups, f_in, f_out);
}

inline std::vector<DeviceMatrix<float>> grouped_matmul(const std::vector<DeviceMatrix<float>>& inputs,
                                                       const DeviceArray<float>& weights, Index groups, Index f_in,
                                                       Index f_out) {
  return detail::grouped<float>(inputs, weights.data(), groups, f_in, f_out);
}

// One rank of the destination-row partitioned SpMM over a caller-owned NCCL
// communicator (gm_dist_spmm). EXACT mode: `rows` is the rank's row slice of
// the CSC with global source ids; every rank passes its X shard of
// shard_rows rows (row-sharded X, last shard zero-padded).
class DistSpmm {
 public:
  DistSpmm(const CsrView& rows, Index shard_rows, int rank, int world, ncclComm_t comm)
      : rows_(rows), comm_(comm) {
    layout_.rank = rank;
    layout_.world = world;
    layout_.mode = GM_DIST_EXACT;
    layout_.shard_rows = shard_rows;
    block_ = rows_.c_struct();
    detail::check_cuda(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "stream");
  }
  DistSpmm(const DistSpmm&) = delete;
  DistSpmm& operator=(const DistSpmm&) = delete;
  ~DistSpmm() { cudaStreamDestroy(comm_stream_); }

  template <class S>
  DeviceMatrix<S> operator()(const DeviceMatrix<S>& x_shard, AggKind kind, DeviceArray<std::int32_t>* argmax = nullptr) {
    if (x_shard.rows() != layout_.shard_rows) throw std::invalid_argument("DistSpmm: x_shard rows != shard_rows");
    plan_ = rows_.plan();
    layout_.blocks = &block_;
    layout_.plans = &plan_;
    const gm_dtype dt = detail::dtype_of<S>();
    const std::size_t wsb = gm_dist_spmm_workspace(&layout_, dt, x_shard.cols());
    if (ws_.size() < wsb) ws_ = DeviceArray<unsigned char>(wsb);
    DeviceMatrix<S> out(rows_.num_rows(), x_shard.cols());
    const bool mm = kind == AggKind::max || kind == AggKind::min;
    if (mm && argmax) *argmax = DeviceArray<std::int32_t>(static_cast<std::size_t>(out.rows() * out.cols()));
    const gm_reduce r = kind == AggKind::sum ? GM_SUM : kind == AggKind::mean ? GM_MEAN : kind == AggKind::max ? GM_MAX : GM_MIN;
    detail::check(gm_dist_spmm(&layout_, dt, x_shard.data(), x_shard.cols(), r, out.data(),
                               mm && argmax ? argmax->data() : nullptr, ws_.data(), ws_.size(), comm_, comm_stream_,
                               stream()));
    return out;
  }

 private:
  CsrView rows_;
  ncclComm_t comm_;
  gm_dist_layout layout_{};
  gm_csr block_{};
  gm_spmm_plan plan_{};
  cudaStream_t comm_stream_ = nullptr;
  DeviceArray<unsigned char> ws_;
};

// One rank of push mode (gm_spmm_ex push epilogue): the SpMM over rows
// [r0, r1) of `csc` (global source ids) reads this rank's replica of the layer
// input and stores every finished row into out_next (its rows r0..r1) and into
// each peer's replica of the next layer's input — device pointers mapped into
// this process, e.g. by gm_ipc_open_handle over NVLink. mask (optional, one
// word per local row): bit j = push to peers[j]. The caller orders the peers'
// reads after the call (a collective on the stream). Any unweighted
// aggregation; max/min also write this rank's argmax (local rows).
class PushSpmm {
 public:
  PushSpmm(const CsrView& csc, Index r0, Index r1, std::vector<void*> peers,
           const DeviceArray<std::uint32_t>* mask = nullptr)
      : csc_(csc), r0_(r0), r1_(r1), peers_(std::move(peers)), mask_(mask) {
    if (r0 < 0 || r1 < r0 || r1 > csc.num_rows()) throw std::invalid_argument("PushSpmm: bad row range");
    if (peers_.size() > GM_MAX_PUSH) throw std::invalid_argument("PushSpmm: at most GM_MAX_PUSH peers");
    const std::vector<Index> rp = csc.rowptr.to_host();
    slice_ = gm_csr{r1 - r0, csc.num_cols, rp[static_cast<std::size_t>(r1)] - rp[static_cast<std::size_t>(r0)],
                    csc.rowptr.data() + r0, csc.col.data(), csc.perm.data()};
    const std::size_t bytes = gm_spmm_plan_bytes(slice_.num_rows, slice_.num_cols, slice_.nnz);
    plan_buf_ = DeviceArray<unsigned char>(bytes ? bytes : 1);
    detail::check(gm_spmm_plan_build(&slice_, plan_buf_.data(), bytes, &plan_, stream()));
  }

  template <class S>
  void operator()(const DeviceMatrix<S>& x, DeviceMatrix<S>& out_next, AggKind kind,
                  DeviceArray<std::int32_t>* argmax = nullptr) const {
    const bool mm = kind == AggKind::max || kind == AggKind::min;
    if (mm && !argmax) throw std::invalid_argument("PushSpmm: max/min need the argmax of this rank's rows");
    if (x.rows() != csc_.num_cols || out_next.rows() != x.rows() || out_next.cols() != x.cols())
      throw std::invalid_argument("PushSpmm: x / out_next must be [num_nodes, F] replicas");
    gm_spmm_epilogue ep{};
    ep.n_push = static_cast<std::int32_t>(peers_.size());
    for (std::size_t q = 0; q < peers_.size(); ++q) ep.push_dst[q] = peers_[q];
    ep.push_row0 = r0_;
    ep.push_mask = mask_ ? mask_->data() : nullptr;
    if (mm) *argmax = DeviceArray<std::int32_t>(static_cast<std::size_t>((r1_ - r0_) * x.cols()));
    const gm_reduce r = kind == AggKind::sum ? GM_SUM : kind == AggKind::mean ? GM_MEAN
                        : kind == AggKind::max ? GM_MAX : GM_MIN;
    detail::check(gm_spmm_ex(&slice_, &plan_, detail::dtype_of<S>(), x.data(), x.cols(), nullptr, r, 0, nullptr, &ep,
                             out_next.data() + r0_ * x.cols(), mm ? argmax->data() : nullptr, stream()));
  }

 private:
  CsrView csc_;
  Index r0_, r1_;
  std::vector<void*> peers_;
  const DeviceArray<std::uint32_t>* mask_;
  gm_csr slice_{};
  gm_spmm_plan plan_{};
  DeviceArray<unsigned char> plan_buf_;
};

}  // namespace b200
