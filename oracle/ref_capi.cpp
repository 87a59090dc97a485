// ref_capi.cpp — C entry points over the UNMODIFIED reference
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/libgraphmill_ref.so). TEST INFRASTRUCTURE ONLY: used to pin the
// oracle restatement, to generate tests/golden/ fixtures, and as the
// "reference" CPU arm of bench.py. Every function calls the reference's own
// public API; nothing here re-implements its arithmetic.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <span>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "graphmill/aggregate.hpp"
#include "graphmill/edge_index.hpp"
#include "graphmill/hetero.hpp"
#include "graphmill/message_passing.hpp"

using namespace graphmill;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

EdgeIndex make_index(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src,
                     int64_t n_dst, int undirected) {
  EdgeIndexClaims claims;
  if (undirected) claims.is_undirected = true;
  return EdgeIndex(std::vector<Index>(src, src + e), std::vector<Index>(dst, dst + e), n_src,
                   n_dst, claims);
}

template <typename S>
Tensor<S> make_tensor(const S* p, int64_t rows, int64_t f) {
  return Tensor<S>::from_data({rows, f}, std::vector<S>(p, p + rows * f));
}

template <typename S>
int spmm_impl(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
              int undirected, const S* x, int64_t f, const S* w, int mean, S* out) {
  return guarded([&] {
    NoGradGuard ng;
    EdgeIndex ei = make_index(src, dst, e, n_src, n_dst, undirected);
    std::optional<Tensor<S>> wt;
    if (w) wt = Tensor<S>::from_data({e}, std::vector<S>(w, w + e));
    Tensor<S> o = spmm(ei, make_tensor(x, n_src, f), wt, mean ? AggKind::mean : AggKind::sum);
    std::memcpy(out, o.data().data(), sizeof(S) * static_cast<size_t>(n_dst * f));
  });
}

// The reference max path (message_passing.hpp:508-514) with argpos recovered
// from the reference's own backward (aggregate.hpp:295-308): the gradient of
// sum(out) lands exactly on the first attaining grouped position.
template <typename S>
int max_impl(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
             const S* x, int64_t f, int is_min, S* out, int64_t* arg) {
  return guarded([&] {
    EdgeIndex ei = make_index(src, dst, e, n_src, n_dst, 0);
    auto [order, grouped_dst] = detail::dst_grouped_order(ei, false);
    std::vector<Index> src_nodes(order.size());
    for (size_t i = 0; i < order.size(); ++i) src_nodes[i] = ei.src()[static_cast<size_t>(order[i])];
    Tensor<S> m;
    {
      NoGradGuard ng;
      Tensor<S> g = gather_rows(make_tensor(x, n_src, f), src_nodes);
      m = Tensor<S>::from_data(g.shape(), std::vector<S>(g.data().begin(), g.data().end()));
    }
    m.set_requires_grad(true);
    Tensor<S> o = aggregate(m, grouped_dst, n_dst, is_min ? AggKind::min : AggKind::max,
                            AggLayout::sorted_segments);
    std::memcpy(out, o.data().data(), sizeof(S) * static_cast<size_t>(n_dst * f));
    std::fill(arg, arg + n_dst * f, int64_t{-1});
    if (e == 0) return;
    backward(sum(o));
    Tensor<S> gm = m.grad();
    auto gd = gm.data();
    for (int64_t p = 0; p < e; ++p) {
      const Index v = grouped_dst[static_cast<size_t>(p)];
      for (int64_t j = 0; j < f; ++j)
        if (gd[static_cast<size_t>(p * f + j)] != S(0)) arg[v * f + j] = order[static_cast<size_t>(p)];
    }
  });
}

// Backward of the layer max/min path (message_passing.hpp:508-514) through the
// reference's own tape: x -> gather_rows(x, src in grouped order) (tracked) ->
// aggregate(max|min, sorted_segments) -> loss = sum(mul(out, G)); dx = x.grad()
// (aggregate.hpp:295-308 argpos scatter, then the gather_rows adjoint
// tensor.hpp:510-524).
template <typename S>
int max_bwd_impl(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst, const S* x,
                 int64_t f, int is_min, const S* G, S* dx) {
  return guarded([&] {
    EdgeIndex ei = make_index(src, dst, e, n_src, n_dst, 0);
    auto [order, grouped_dst] = detail::dst_grouped_order(ei, false);
    std::vector<Index> src_nodes(order.size());
    for (size_t i = 0; i < order.size(); ++i) src_nodes[i] = ei.src()[static_cast<size_t>(order[i])];
    Tensor<S> xt = make_tensor(x, n_src, f);
    xt.set_requires_grad(true);
    Tensor<S> m = gather_rows(xt, src_nodes);
    Tensor<S> o = aggregate(m, grouped_dst, n_dst, is_min ? AggKind::min : AggKind::max,
                            AggLayout::sorted_segments);
    backward(sum(mul(o, make_tensor(G, n_dst, f))));
    if (xt.has_grad()) {
      Tensor<S> gx = xt.grad();
      std::memcpy(dx, gx.data().data(), sizeof(S) * static_cast<size_t>(n_src * f));
    } else {
      std::fill(dx, dx + n_src * f, S(0));
    }
  });
}

// spmm backward through the reference's own tape: loss = sum(mul(spmm(e, x, w), G)),
// so the gradient entering spmm's closure is exactly G (test_message_passing.cpp:92-105).
template <typename S>
int spmm_bwd_impl(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst, int undirected,
                  const S* x, int64_t f, const S* w, int mean, const S* G, S* dx, S* dw) {
  return guarded([&] {
    EdgeIndex ei = make_index(src, dst, e, n_src, n_dst, undirected);
    Tensor<S> xt = make_tensor(x, n_src, f);
    xt.set_requires_grad(true);
    std::optional<Tensor<S>> wt;
    if (w) {
      wt = Tensor<S>::from_data({e}, std::vector<S>(w, w + e));
      wt->set_requires_grad(true);
    }
    Tensor<S> out = spmm(ei, xt, wt, mean ? AggKind::mean : AggKind::sum);
    Tensor<S> coeff = make_tensor(G, n_dst, f);
    backward(sum(mul(out, coeff)));
    if (xt.has_grad()) {
      Tensor<S> gx = xt.grad();
      std::memcpy(dx, gx.data().data(), sizeof(S) * static_cast<size_t>(n_src * f));
    } else {
      std::fill(dx, dx + n_src * f, S(0));
    }
    if (w && dw) {
      if (wt->has_grad()) {
        Tensor<S> gw = wt->grad();
        std::memcpy(dw, gw.data().data(), sizeof(S) * static_cast<size_t>(e));
      } else {
        std::fill(dw, dw + e, S(0));
      }
    }
  });
}

}  // namespace

extern "C" {

int ref_spmm_backward_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                          int undirected, const float* x, int64_t f, const float* w, int mean, const float* G,
                          float* dx, float* dw) {
  return spmm_bwd_impl<float>(src, dst, e, n_src, n_dst, undirected, x, f, w, mean, G, dx, dw);
}
int ref_spmm_backward_f64(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                          int undirected, const double* x, int64_t f, const double* w, int mean, const double* G,
                          double* dx, double* dw) {
  return spmm_bwd_impl<double>(src, dst, e, n_src, n_dst, undirected, x, f, w, mean, G, dx, dw);
}

// to_hetero(sage) + hetero_propagate(InterCombine::sum), segment_fused
// (hetero.hpp:217-365) with caller-given weights. Node types "n<i>" (ptr over a
// concatenated h), edge types (n<s>, r<i>, n<d>); outputs concatenated like h.
int ref_hetero_sage_f32(int32_t n_types, const int64_t* node_ptr, const float* h, int64_t f_in, int64_t f_out,
                        int32_t n_et, const int32_t* et_src, const int32_t* et_dst, const int64_t* e_ptr,
                        const int64_t* src, const int64_t* dst, const float* w_neigh, const float* w_self,
                        const float* bias, float* out) {
  return guarded([&] {
    NoGradGuard ng;
    HeteroGraph<float> g;
    std::map<std::string, Tensor<float>> hm;
    HeteroModel<float> model;
    model.kind = LayerKind::sage;
    model.in_dim = f_in;
    model.out_dim = f_out;
    model.combine = InterCombine::sum;
    auto name = [](int i) { return "n" + std::to_string(i); };
    for (int t = 0; t < n_types; ++t) {
      Tensor<float> ht = make_tensor(h + node_ptr[t] * f_in, node_ptr[t + 1] - node_ptr[t], f_in);
      g.add_node_type(name(t), ht);
      hm[name(t)] = ht;
      LayerParams<float> up;
      up.kind = LayerKind::sage;
      up.in_dim = f_in;
      up.out_dim = f_out;
      up.weights["w_self"] = make_tensor(w_self + t * f_in * f_out, f_in, f_out);
      up.weights["bias"] = Tensor<float>::from_data({f_out}, std::vector<float>(bias + t * f_out, bias + (t + 1) * f_out));
      model.node_update[name(t)] = up;
    }
    for (int i = 0; i < n_et; ++i) {
      EdgeType et{name(et_src[i]), "r" + std::to_string(i), name(et_dst[i])};
      const int64_t a = e_ptr[i], b = e_ptr[i + 1];
      g.add_edge_type(et, EdgeIndex(std::vector<Index>(src + a, src + b), std::vector<Index>(dst + a, dst + b),
                                    node_ptr[et_src[i] + 1] - node_ptr[et_src[i]],
                                    node_ptr[et_dst[i] + 1] - node_ptr[et_dst[i]]));
      LayerParams<float> rp;
      rp.kind = LayerKind::sage;
      rp.in_dim = f_in;
      rp.out_dim = f_out;
      rp.aggregation = AggregationSpec<float>::simple(AggKind::mean);
      rp.weights["w_neigh"] = make_tensor(w_neigh + i * f_in * f_out, f_in, f_out);
      model.replicas[et] = rp;
    }
    auto res = hetero_propagate(g, model, hm, ExecPath::segment_fused);
    for (int t = 0; t < n_types; ++t) {
      const Tensor<float>& o = res.at(name(t));
      std::memcpy(out + node_ptr[t] * f_out, o.data().data(), sizeof(float) * static_cast<size_t>(o.numel()));
    }
  });
}

const char* ref_last_error() { return g_err.c_str(); }

// edge_index.cpp:45-62
int ref_build_compressed(const int64_t* keys, const int64_t* values, int64_t e, int64_t num_rows,
                         int64_t* rowptr, int64_t* col, int64_t* perm) {
  return guarded([&] {
    CsrView v = build_compressed(std::span<const Index>(keys, static_cast<size_t>(e)),
                                 std::span<const Index>(values, static_cast<size_t>(e)), num_rows);
    std::copy(v.rowptr.begin(), v.rowptr.end(), rowptr);
    std::copy(v.col.begin(), v.col.end(), col);
    std::copy(v.perm.begin(), v.perm.end(), perm);
  });
}

// EdgeIndex ctor + verify_claims (edge_index.cpp:69-119): status + message.
int ref_edge_index_check(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src,
                         int64_t n_dst, int undirected, int sort_order) {
  return guarded([&] {
    EdgeIndexClaims claims;
    if (undirected) claims.is_undirected = true;
    if (sort_order == 1) claims.sort_order = SortOrder::by_src;
    if (sort_order == 2) claims.sort_order = SortOrder::by_dst;
    EdgeIndex ei(std::vector<Index>(src, src + e), std::vector<Index>(dst, dst + e), n_src, n_dst,
                 claims);
  });
}

// message_passing.hpp:92-169 (forward)
int ref_spmm_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                 int undirected, const float* x, int64_t f, const float* w, int mean, float* out) {
  return spmm_impl<float>(src, dst, e, n_src, n_dst, undirected, x, f, w, mean, out);
}
int ref_spmm_f64(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                 int undirected, const double* x, int64_t f, const double* w, int mean,
                 double* out) {
  return spmm_impl<double>(src, dst, e, n_src, n_dst, undirected, x, f, w, mean, out);
}

int ref_max_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                const float* x, int64_t f, int is_min, float* out, int64_t* arg) {
  return max_impl<float>(src, dst, e, n_src, n_dst, x, f, is_min, out, arg);
}
int ref_max_f64(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                const double* x, int64_t f, int is_min, double* out, int64_t* arg) {
  return max_impl<double>(src, dst, e, n_src, n_dst, x, f, is_min, out, arg);
}
int ref_max_backward_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                         const float* x, int64_t f, int is_min, const float* G, float* dx) {
  return max_bwd_impl<float>(src, dst, e, n_src, n_dst, x, f, is_min, G, dx);
}
int ref_max_backward_f64(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                         const double* x, int64_t f, int is_min, const double* G, double* dx) {
  return max_bwd_impl<double>(src, dst, e, n_src, n_dst, x, f, is_min, G, dx);
}

// aggregate.hpp:155-215 on edge-level values (a6): kind 0 sum, 1 mean, 2 max, 3 min.
int ref_aggregate_f32(const float* values, int64_t e, int64_t f, const int64_t* index,
                      int64_t n, int kind, float* out) {
  return guarded([&] {
    NoGradGuard ng;
    const AggKind k[] = {AggKind::sum, AggKind::mean, AggKind::max, AggKind::min};
    Tensor<float> o = aggregate(make_tensor(values, e, f),
                                std::span<const Index>(index, static_cast<size_t>(e)), n, k[kind]);
    std::memcpy(out, o.data().data(), sizeof(float) * static_cast<size_t>(n * f));
  });
}

// GCN fused branch (message_passing.hpp:490-495) after the transform:
// with_self_loops + gcn_norm + spmm(graph, xw, norm, sum). xw = h @ W given.
int ref_gcn_aggregate_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n,
                          const float* xw, int64_t f, float* out) {
  return guarded([&] {
    NoGradGuard ng;
    EdgeIndex ei = make_index(src, dst, e, n, n, 0);
    const EdgeIndex graph = with_self_loops(ei);
    Tensor<float> norm = detail::gcn_norm<float>(ei, graph, true);
    Tensor<float> o = spmm(graph, make_tensor(xw, n, f), norm, AggKind::sum);
    std::memcpy(out, o.data().data(), sizeof(float) * static_cast<size_t>(n * f));
  });
}

// Full reference GCN layer forward (message_passing.hpp:600-608, segment_fused):
// matmul(h, W) + GCN aggregate + bias. Used for the Cora 2-layer parity case.
int ref_gcn_layer_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n,
                      const float* h, int64_t f_in, const float* wgt, const float* bias,
                      int64_t f_out, float* out) {
  return guarded([&] {
    NoGradGuard ng;
    EdgeIndex ei = make_index(src, dst, e, n, n, 0);
    LayerParams<float> p;
    p.kind = LayerKind::gcn;
    p.in_dim = f_in;
    p.out_dim = f_out;
    p.weights["weight"] = make_tensor(wgt, f_in, f_out);
    p.weights["bias"] = Tensor<float>::from_data({f_out}, std::vector<float>(bias, bias + f_out));
    Tensor<float> o = layer_forward(p, ei, make_tensor(h, n, f_in), ExecPath::segment_fused);
    std::memcpy(out, o.data().data(), sizeof(float) * static_cast<size_t>(n * f_out));
  });
}

}  // extern "C"

// Model<S>::forward (message_passing.hpp:631-641) of a GCN stack: layer_forward
// per layer with relu in between, segment_fused path. layer l maps dims[l] ->
// dims[l+1]; weights/biases are concatenated in layer order.
template <typename S>
static int gcn_model_impl(const int64_t* src, const int64_t* dst, int64_t e, int64_t n, const S* h,
                          int32_t n_layers, const int64_t* dims, const S* weights, const S* biases, S* out) {
  return guarded([&] {
    NoGradGuard ng;
    EdgeIndex ei = make_index(src, dst, e, n, n, 0);
    Model<S> m;
    const S* w = weights;
    const S* b = biases;
    for (int32_t l = 0; l < n_layers; ++l) {
      LayerParams<S> p;
      p.kind = LayerKind::gcn;
      p.in_dim = dims[l];
      p.out_dim = dims[l + 1];
      p.weights["weight"] = make_tensor(w, dims[l], dims[l + 1]);
      p.weights["bias"] = Tensor<S>::from_data({dims[l + 1]}, std::vector<S>(b, b + dims[l + 1]));
      w += dims[l] * dims[l + 1];
      b += dims[l + 1];
      m.layers.push_back(std::move(p));
    }
    Tensor<S> o = m.forward(ei, make_tensor(h, n, dims[0]), ExecPath::segment_fused);
    std::memcpy(out, o.data().data(), sizeof(S) * static_cast<size_t>(n * dims[n_layers]));
  });
}

extern "C" {
int ref_gcn_model_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n, const float* h,
                      int32_t n_layers, const int64_t* dims, const float* weights, const float* biases,
                      float* out) {
  return gcn_model_impl<float>(src, dst, e, n, h, n_layers, dims, weights, biases, out);
}
int ref_gcn_model_f64(const int64_t* src, const int64_t* dst, int64_t e, int64_t n, const double* h,
                      int32_t n_layers, const int64_t* dims, const double* weights, const double* biases,
                      double* out) {
  return gcn_model_impl<double>(src, dst, e, n, h, n_layers, dims, weights, biases, out);
}
}  // extern "C"

// hetero.hpp:134-157 over segments of a concatenated x.
template <typename S>
static int gmm_impl(const S* x, const int64_t* ptr, int64_t groups, int64_t k, int64_t n,
                    const S* w, S* out) {
  return guarded([&] {
    NoGradGuard ng;
    std::vector<Tensor<S>> ins;
    for (int64_t g = 0; g < groups; ++g)
      ins.push_back(make_tensor(x + ptr[g] * k, ptr[g + 1] - ptr[g], k));
    Tensor<S> wt = Tensor<S>::from_data({groups, k, n}, std::vector<S>(w, w + groups * k * n));
    auto outs = grouped_matmul<S>(ins, wt);
    for (int64_t g = 0; g < groups; ++g)
      std::memcpy(out + ptr[g] * n, outs[static_cast<size_t>(g)].data().data(),
                  sizeof(S) * static_cast<size_t>((ptr[g + 1] - ptr[g]) * n));
  });
}
extern "C" {
int ref_grouped_matmul_f32(const float* x, const int64_t* ptr, int64_t groups, int64_t k,
                           int64_t n, const float* w, float* out) {
  return gmm_impl<float>(x, ptr, groups, k, n, w, out);
}
int ref_grouped_matmul_f64(const double* x, const int64_t* ptr, int64_t groups, int64_t k,
                           int64_t n, const double* w, double* out) {
  return gmm_impl<double>(x, ptr, groups, k, n, w, out);
}

// ---------------------------------------------------------------------------
// CPU arm of bench.py: the reference's own spmm<float> (sum) run by `threads`
// std::threads, each on the sub-EdgeIndex of a contiguous destination-row
// range (edges with dst in range, relative COO order kept, dst renumbered), so
// per-row results and order are those of the single-threaded reference.
// Sub-indices are built and their CSC caches filled OUTSIDE the timed region
// (steady state of repeated layer calls, edge_index.hpp:65-71). Returns the
// mean seconds per repeat over `repeat` timed calls after `warmup`, mirroring
// time_loop (message_passing.hpp:676-697). rows_limit > 0 restricts the run to
// the first rows_limit destination rows (a bounded sample); *edges_done gets
// the number of edges processed per repeat.
// ---------------------------------------------------------------------------
int ref_bench_spmm_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src,
                       int64_t n_dst, const float* x, int64_t f, int mean, int threads,
                       int64_t rows_limit, int warmup, int repeat, double* seconds,
                       int64_t* edges_done) {
  return guarded([&] {
    NoGradGuard ng;
    if (threads < 1) threads = 1;
    const int64_t rows = rows_limit > 0 ? std::min(rows_limit, n_dst) : n_dst;
    std::vector<int64_t> cut(static_cast<size_t>(threads) + 1);
    for (int t = 0; t <= threads; ++t) cut[static_cast<size_t>(t)] = rows * t / threads;
    std::vector<std::vector<Index>> ssrc(static_cast<size_t>(threads)), sdst(static_cast<size_t>(threads));
    for (int64_t i = 0; i < e; ++i) {
      if (dst[i] >= rows) continue;
      const int t = static_cast<int>(std::upper_bound(cut.begin(), cut.end(), dst[i]) - cut.begin()) - 1;
      ssrc[static_cast<size_t>(t)].push_back(src[i]);
      sdst[static_cast<size_t>(t)].push_back(dst[i] - cut[static_cast<size_t>(t)]);
    }
    int64_t total = 0;
    std::vector<EdgeIndex> subs;
    for (int t = 0; t < threads; ++t) {
      total += static_cast<int64_t>(ssrc[static_cast<size_t>(t)].size());
      subs.emplace_back(std::move(ssrc[static_cast<size_t>(t)]), std::move(sdst[static_cast<size_t>(t)]),
                        n_src, cut[static_cast<size_t>(t) + 1] - cut[static_cast<size_t>(t)]);
      subs.back().to_csc();
    }
    Tensor<float> xt = make_tensor(x, n_src, f);
    auto run_once = [&] {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
          Tensor<float> o = spmm(subs[static_cast<size_t>(t)], xt, std::nullopt,
                                 mean ? AggKind::mean : AggKind::sum);
          (void)o;
        });
      for (auto& th : pool) th.join();
    };
    BenchTiming bt = time_loop(run_once, repeat, warmup);
    *seconds = bt.mean_ms / 1000.0;
    *edges_done = total;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Synthetic inputs of the bench / parity configs, generated on
// the host for the reference arm WITHOUT the product library. The RNG is the
// reference's own (random.hpp:9-65: rng::mix, rng::derive, rng::Stream); the
// graph construction on top of it (Chung-Lu alpha = 0.5 by inverse CDF over a
// keyed Feistel permutation of node ids, 1-in-4 quantised feature rows) is the
// §8d generator, restated here so the CPU arm and the GPU arm see the same
// COO lists and features bit-for-bit (tests/test_oracle.py pins the two
// generators against each other). Built with -ffp-contract=off: every fp64
// operation rounds once, as on the device (__dadd_rn/__dmul_rn/__dsqrt_rn).
// ---------------------------------------------------------------------------
namespace synth {
enum : std::uint64_t {
  kTagSrc = 0x737263ull, kTagDst = 0x647374ull, kTagFeat = 0x66656174ull,
  kTagPerm = 0x7065726dull, kTagQuant = 0x7175616eull, kTagWgt = 0x776774ull,
};

// Bijection of [0, n): 4-round Feistel on the smallest even-bit power of two
// >= n, cycle-walking back into range.
std::uint64_t permute(std::uint64_t x, std::uint64_t n, std::uint64_t key) {
  if (n <= 1) return 0;
  int bits = 0;
  while ((std::uint64_t{1} << bits) < n) ++bits;
  if (bits & 1) ++bits;
  if (bits < 2) bits = 2;
  const int half = bits / 2;
  const std::uint64_t mask = (std::uint64_t{1} << half) - 1;
  do {
    std::uint64_t l = x >> half, r = x & mask;
    for (int round = 0; round < 4; ++round) {
      const std::uint64_t nl = r;
      r = l ^ (rng::mix(key ^ (r * 0x100000001b3ull) ^ static_cast<std::uint64_t>(round)) & mask);
      l = nl;
    }
    x = (l << half) | r;
  } while (x >= n);
  return x;
}

// Inverse CDF of the density (p+1)^-1/2 on [0, n): (1 + u(sqrt(n+1) - 1))^2 - 1.
std::uint64_t powerlaw_node(double u, std::uint64_t n, std::uint64_t perm_key) {
  const double s = std::sqrt(static_cast<double>(n + 1)) + -1.0;
  const double t = 1.0 + u * s;
  const double xpos = t * t + -1.0;
  std::uint64_t p = xpos <= 0.0 ? 0 : static_cast<std::uint64_t>(xpos);
  if (p >= n) p = n - 1;
  return permute(p, n, perm_key);
}

void edge(int kind, std::uint64_t seed, std::uint64_t i, std::uint64_t n_src, std::uint64_t n_dst,
          int64_t* s, int64_t* d) {
  rng::Stream ss(rng::derive(seed, kTagSrc, i));
  rng::Stream ds(rng::derive(seed, kTagDst, i));
  if (kind == 0) {
    *s = static_cast<int64_t>(ss.next_below(n_src));
    *d = static_cast<int64_t>(ds.next_below(n_dst));
  } else {
    *s = static_cast<int64_t>(powerlaw_node(ss.next_real(), n_src, rng::derive(seed, kTagPerm, 1)));
    *d = static_cast<int64_t>(powerlaw_node(ds.next_real(), n_dst, rng::derive(seed, kTagPerm, 2)));
  }
}

template <typename Fn>
void parallel_for(int64_t count, int threads, Fn&& fn) {
  if (threads < 1) threads = 1;
  if (count < 65536) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const int64_t lo = count * t / threads, hi = count * (t + 1) / threads;
      for (int64_t i = lo; i < hi; ++i) fn(i);
    });
  for (auto& th : pool) th.join();
}
}  // namespace synth

extern "C" {
int ref_synth_edges(int kind, uint64_t seed, int64_t first, int64_t count, int64_t n_src, int64_t n_dst,
                    int64_t* src, int64_t* dst, int threads) {
  return guarded([&] {
    synth::parallel_for(count, threads, [&](int64_t i) {
      synth::edge(kind, seed, static_cast<std::uint64_t>(first + i), static_cast<std::uint64_t>(n_src),
                  static_cast<std::uint64_t>(n_dst), src + i, dst + i);
    });
  });
}

// x[row][j] ~ U[-1, 1) from the row's stream (Tensor::rand_uniform,
// tensor.hpp:147-152, one stream per row); quantize: 1 row in 4 (by hash)
// snapped down to multiples of 1/8, a snapped zero is -0.0 in half of them.
int ref_synth_features_f32(uint64_t seed, int64_t first_row, int64_t rows, int64_t f, int quantize, float* x,
                           int threads) {
  return guarded([&] {
    synth::parallel_for(rows, threads, [&](int64_t i) {
      const std::uint64_t row = static_cast<std::uint64_t>(first_row + i);
      rng::Stream s(rng::derive(seed, synth::kTagFeat, row));
      const std::uint64_t h = rng::mix(rng::derive(seed, synth::kTagQuant, row));
      const bool snap = quantize && (h & 3) == 0, negzero = (h >> 2) & 1;
      for (int64_t j = 0; j < f; ++j) {
        double v = s.next_real(-1.0, 1.0);
        if (snap) {
          double q = static_cast<double>(static_cast<int64_t>(v * 8.0));
          if (q > v * 8.0) q = q + -1.0;
          v = q * 0.125;
          if (v == 0.0 && negzero) v = -0.0;
        }
        x[i * f + j] = static_cast<float>(v);
      }
    });
  });
}

// The reference's own build_compressed (edge_index.cpp:45-62) on the CSC keys,
// timed once (one thread: the reference has no parallel build).
int ref_bench_build_compressed(const int64_t* keys, const int64_t* values, int64_t e, int64_t num_rows,
                               double* seconds) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    CsrView v = build_compressed(std::span<const Index>(keys, static_cast<size_t>(e)),
                                 std::span<const Index>(values, static_cast<size_t>(e)), num_rows);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (v.rowptr.size() != static_cast<size_t>(num_rows + 1)) throw std::logic_error("bad rowptr");
  });
}

// The reference max path (message_passing.hpp:508-514: dst_grouped_order +
// gather_rows + aggregate(max, sorted_segments)) on the first rows_limit
// destination rows, timed once after the CSC cache is filled.
int ref_bench_max_f32(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_src, int64_t n_dst,
                      const float* x, int64_t f, int64_t rows_limit, double* seconds, int64_t* edges_done) {
  return guarded([&] {
    NoGradGuard ng;
    const int64_t rows = rows_limit > 0 ? std::min(rows_limit, n_dst) : n_dst;
    std::vector<Index> ss, dd;
    for (int64_t i = 0; i < e; ++i)
      if (dst[i] < rows) { ss.push_back(src[i]); dd.push_back(dst[i]); }
    *edges_done = static_cast<int64_t>(ss.size());
    EdgeIndex ei(std::move(ss), std::move(dd), n_src, rows);
    ei.to_csc();
    Tensor<float> xt = make_tensor(x, n_src, f);
    const auto t0 = std::chrono::steady_clock::now();
    auto [order, grouped_dst] = detail::dst_grouped_order(ei, false);
    std::vector<Index> src_nodes(order.size());
    for (size_t i = 0; i < order.size(); ++i) src_nodes[i] = ei.src()[static_cast<size_t>(order[i])];
    Tensor<float> m = gather_rows(xt, src_nodes);
    Tensor<float> o = aggregate(m, grouped_dst, rows, AggKind::max, AggLayout::sorted_segments);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    (void)o;
  });
}

}  // extern "C"
