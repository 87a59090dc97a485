// The reference's own hot-path test cases, restated against the C++ mirror
// (include/graphmill_b200.hpp) running on the B200 through the C-ABI.
// Each TEST_CASE cites the reference test it restates
// (/root/reference/proj/tests/...). Built and run by tests/test_gpu_cpp.py with
// the doctest stand-in used to pin the oracle (oracle/ref_shim/doctest_shim).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <algorithm>
#include <cmath>
#include <thread>

#include "graphmill_b200.hpp"
#include "synth.h"  // the reference RNG (random.hpp:9-65), for test_stream(salt)

using namespace b200;
using gm_synth::Stream;

namespace {

Stream test_stream(std::uint64_t salt) { return Stream(gm_synth::derive(0x746573747321ull, salt)); }

std::vector<double> random_values(std::size_t n, std::uint64_t salt, double lo = -1, double hi = 1) {
  Stream s = test_stream(salt);
  std::vector<double> v(n);
  for (auto& x : v) x = s.next_real(lo, hi);
  return v;
}

// test_edge_index.cpp:12-26 (counting-sort-free oracle)
struct HostCsr {
  std::vector<Index> rowptr, col, perm;
};
HostCsr oracle_compress(const std::vector<Index>& keys, const std::vector<Index>& values, Index num_rows) {
  HostCsr v;
  v.rowptr.assign(static_cast<std::size_t>(num_rows) + 1, 0);
  for (Index r = 0; r < num_rows; ++r) {
    v.rowptr[static_cast<std::size_t>(r) + 1] = v.rowptr[static_cast<std::size_t>(r)];
    for (std::size_t i = 0; i < keys.size(); ++i)
      if (keys[i] == r) {
        v.col.push_back(values[i]);
        v.perm.push_back(static_cast<Index>(i));
        ++v.rowptr[static_cast<std::size_t>(r) + 1];
      }
  }
  return v;
}

EdgeIndex diamond() { return EdgeIndex({0, 1, 1, 2}, {1, 0, 2, 1}, 3, 3); }

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  REQUIRE(a.size() == b.size());
  double w = 0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
  return w;
}

}  // namespace

TEST_CASE("claims are verified, not trusted (test_edge_index.cpp:34-54)") {
  EdgeIndexClaims by_src;
  by_src.sort_order = SortOrder::by_src;
  EdgeIndex ok({0, 1, 1, 2}, {1, 0, 2, 1}, 3, 3, by_src);
  CHECK(ok.sort_order() == SortOrder::by_src);
  EdgeIndexClaims by_dst;
  by_dst.sort_order = SortOrder::by_dst;
  CHECK_THROWS_WITH_AS(EdgeIndex({0, 1, 1, 2}, {1, 0, 2, 1}, 3, 3, by_dst), doctest::Contains("position 1"),
                       std::invalid_argument);
  EdgeIndexClaims undirected;
  undirected.is_undirected = true;
  EdgeIndex sym({0, 1}, {1, 0}, 2, 2, undirected);
  CHECK(sym.is_undirected());
  CHECK_THROWS_AS(EdgeIndex({0, 1}, {1, 2}, 3, 3, undirected), std::invalid_argument);
  CHECK_THROWS_AS(EdgeIndex({0, 0, 1}, {1, 1, 0}, 2, 2, undirected), std::invalid_argument);
  EdgeIndex dup({0, 0, 1, 1}, {1, 1, 0, 0}, 2, 2, undirected);
  CHECK(dup.is_undirected());
}

TEST_CASE("bounds are always validated (test_edge_index.cpp:56-61)") {
  CHECK_THROWS_AS(EdgeIndex({0, 3}, {1, 0}, 3, 3), std::out_of_range);
  CHECK_THROWS_AS(EdgeIndex({0, -1}, {1, 0}, 3, 3), std::out_of_range);
  CHECK_THROWS_AS(EdgeIndex({0}, {5}, 3, 3), std::out_of_range);
  CHECK_THROWS_AS(EdgeIndex({0, 1}, {1}, 2, 2), std::invalid_argument);
  CHECK_THROWS_WITH_AS(EdgeIndex({0, 3}, {1, 0}, 3, 3),
                       doctest::Contains("EdgeIndex: src index 3 at position 1 outside [0, 3)"), std::out_of_range);
}

TEST_CASE("csr/csc construction matches the counting oracle (test_edge_index.cpp:63-77)") {
  EdgeIndex e = diamond();
  const CsrView& csr = e.to_csr();
  CHECK(csr.rowptr_host() == std::vector<Index>{0, 1, 3, 4});
  CHECK(csr.col_host() == std::vector<Index>{1, 0, 2, 1});
  const CsrView& csc = e.to_csc();
  CHECK(csc.rowptr_host() == std::vector<Index>{0, 1, 3, 4});
  CHECK(csc.col_host() == std::vector<Index>{1, 0, 2, 1});
  const HostCsr ref = oracle_compress({0, 1, 1, 2}, {1, 0, 2, 1}, 3);
  CHECK(csr.rowptr_host() == ref.rowptr);
  CHECK(csr.col_host() == ref.col);
  CHECK(csr.perm_host() == ref.perm);
}

TEST_CASE("empty edge set compresses to all-zero rowptr (test_edge_index.cpp:79-84)") {
  EdgeIndex e({}, {}, 3, 3);
  const CsrView& csr = e.to_csr();
  CHECK(csr.rowptr_host() == std::vector<Index>{0, 0, 0, 0});
  CHECK(csr.col_host().empty());
}

TEST_CASE("caches fill once and are returned verbatim afterwards (test_edge_index.cpp:86-94)") {
  EdgeIndex e = diamond();
  CHECK(e.csr_build_count() == 0);
  const CsrView* first = &e.to_csr();
  CHECK(e.csr_build_count() == 1);
  CHECK(&e.to_csr() == first);
  CHECK(e.csr_build_count() == 1);
}

TEST_CASE("round-trip: perm expands any view back to the original pairs (test_edge_index.cpp:96-119)") {
  Stream stream = test_stream(21);
  const Index n = 17;
  std::vector<Index> src(120), dst(120);
  for (std::size_t i = 0; i < src.size(); ++i) {
    src[i] = static_cast<Index>(stream.next_below(n));
    dst[i] = static_cast<Index>(stream.next_below(n));
  }
  EdgeIndex e(src, dst, n, n);
  for (bool by_dst : {false, true}) {
    const CsrView& v = by_dst ? e.to_csc() : e.to_csr();
    const auto rp = v.rowptr_host(), col = v.col_host(), perm = v.perm_host();
    for (Index r = 0; r < n; ++r)
      for (Index k = rp[static_cast<std::size_t>(r)]; k < rp[static_cast<std::size_t>(r) + 1]; ++k) {
        const std::size_t orig = static_cast<std::size_t>(perm[static_cast<std::size_t>(k)]);
        CHECK((by_dst ? dst[orig] : src[orig]) == r);
        CHECK((by_dst ? src[orig] : dst[orig]) == col[static_cast<std::size_t>(k)]);
      }
  }
}

TEST_CASE("transpose_view of undirected graphs aliases the CSR cache (test_edge_index.cpp:121-131)") {
  EdgeIndexClaims undirected;
  undirected.is_undirected = true;
  EdgeIndex tri({0, 1, 1, 2, 2, 0}, {1, 0, 2, 1, 0, 2}, 3, 3, undirected);
  const CsrView* t = &tri.transpose_view();
  CHECK(t == &tri.to_csr());
  CHECK(tri.csc_build_count() == 0);
  CHECK_FALSE(tri.has_csc_cache());
}

TEST_CASE("transpose_view of a directed path groups by destination (test_edge_index.cpp:133-140)") {
  EdgeIndex path({0, 1}, {1, 2}, 3, 3);
  CHECK(path.transpose_view().rowptr_host() == std::vector<Index>{0, 0, 1, 2});
  const int builds = path.csc_build_count();
  path.transpose_view();
  CHECK(path.csc_build_count() == builds);
}

TEST_CASE("concurrent cache fill publishes exactly one consistent view (test_edge_index.cpp:227-245)") {
  Stream stream = test_stream(24);
  std::vector<Index> src(2000), dst(2000);
  for (std::size_t i = 0; i < src.size(); ++i) {
    src[i] = static_cast<Index>(stream.next_below(50));
    dst[i] = static_cast<Index>(stream.next_below(50));
  }
  EdgeIndex e(src, dst, 50, 50);
  std::vector<const CsrView*> seen(8, nullptr);
  std::vector<std::thread> workers;
  for (int t = 0; t < 8; ++t) workers.emplace_back([&, t] { seen[static_cast<std::size_t>(t)] = &e.to_csr(); });
  for (auto& w : workers) w.join();
  for (int t = 1; t < 8; ++t) CHECK(seen[static_cast<std::size_t>(t)] == seen[0]);
  const HostCsr ref = oracle_compress(src, dst, 50);
  CHECK(seen[0]->rowptr_host() == ref.rowptr);
  CHECK(seen[0]->col_host() == ref.col);
  CHECK(seen[0]->perm_host() == ref.perm);
}

TEST_CASE("spmm matches an explicit edge loop, with and without weights (test_message_passing.cpp:67-90)") {
  Stream stream = test_stream(61);
  std::vector<Index> src(40), dst(40);
  for (std::size_t i = 0; i < 40; ++i) {
    src[i] = static_cast<Index>(stream.next_below(12));
    dst[i] = static_cast<Index>(stream.next_below(12));
  }
  EdgeIndex e(src, dst, 12, 12);
  const auto xh = random_values(12 * 5, 62);
  const auto wh = random_values(40, 63);
  auto x = DeviceMatrix<double>::from_host(12, 5, xh);
  auto w = DeviceMatrix<double>::from_host(40, 1, wh);
  for (bool weighted : {false, true})
    for (AggKind reduce : {AggKind::sum, AggKind::mean}) {
      auto got = spmm<double>(e, x, weighted ? std::optional<DeviceMatrix<double>>(w) : std::nullopt, reduce)
                     .to_host();
      std::vector<double> want(12 * 5, 0.0);
      std::vector<Index> deg(12, 0);
      for (Index v : dst) ++deg[static_cast<std::size_t>(v)];
      for (std::size_t i = 0; i < 40; ++i)
        for (std::size_t j = 0; j < 5; ++j)
          want[static_cast<std::size_t>(dst[i]) * 5 + j] +=
              (weighted ? wh[i] : 1.0) * xh[static_cast<std::size_t>(src[i]) * 5 + j];
      if (reduce == AggKind::mean)
        for (std::size_t v = 0; v < 12; ++v)
          if (deg[v] > 0)
            for (std::size_t j = 0; j < 5; ++j) want[v * 5 + j] /= static_cast<double>(deg[v]);
      CHECK(max_abs_diff(got, want) <= 1e-12);
    }
  CHECK_THROWS_AS(spmm<double>(e, x, std::nullopt, AggKind::max), std::invalid_argument);
  CHECK_THROWS_AS(spmm<double>(e, DeviceMatrix<double>(3, 5), std::nullopt, AggKind::sum), std::invalid_argument);
}

TEST_CASE("spmm on an undirected index with asymmetric weights stays position-exact (test_message_passing.cpp:107-122)") {
  EdgeIndexClaims undirected;
  undirected.is_undirected = true;
  const std::vector<Index> src{0, 1, 1, 2, 2, 0}, dst{1, 0, 2, 1, 0, 2};
  EdgeIndex sym(src, dst, 3, 3, undirected);
  const auto xh = random_values(3 * 2, 68);
  const std::vector<double> wh{1, 10, 100, 1000, 10000, 100000};
  auto got = spmm<double>(sym, DeviceMatrix<double>::from_host(3, 2, xh), DeviceMatrix<double>::from_host(6, 1, wh),
                          AggKind::sum)
                 .to_host();
  std::vector<double> want(6, 0.0);
  for (std::size_t i = 0; i < 6; ++i)
    for (std::size_t j = 0; j < 2; ++j)
      want[static_cast<std::size_t>(dst[i]) * 2 + j] += wh[i] * xh[static_cast<std::size_t>(src[i]) * 2 + j];
  CHECK(max_abs_diff(got, want) == 0.0);
  CHECK(sym.csc_build_count() == 0);  // never materializes a CSC for undirected input
}

TEST_CASE("gcn on an edgeless graph keeps only the normalized self contribution (test_message_passing.cpp:199-207)") {
  EdgeIndex e({}, {}, 4, 4);
  const auto xh = random_values(4 * 3, 74);
  auto got = gcn_aggregate<double>(e, DeviceMatrix<double>::from_host(4, 3, xh)).to_host();
  CHECK(max_abs_diff(got, xh) <= 1e-14);  // deg = 1, norm = 1
}

TEST_CASE("hand-checked aggregations over two groups (test_aggregate.cpp:22-33)") {
  auto v = DeviceMatrix<double>::from_host(3, 1, std::vector<double>{1, 2, 3});
  const std::vector<Index> idx{0, 0, 1};
  CHECK(aggregate(v, idx, 2, AggKind::sum).to_host() == std::vector<double>{3.0, 3.0});
  CHECK(aggregate(v, idx, 2, AggKind::mean).to_host() == std::vector<double>{1.5, 3.0});
  CHECK(aggregate(v, idx, 2, AggKind::max).to_host() == std::vector<double>{2.0, 3.0});
}

TEST_CASE("empty groups yield zero; negatives keep the true extremum (test_aggregate.cpp:35-46)") {
  auto v = DeviceMatrix<double>::from_host(2, 1, std::vector<double>{4, -2});
  for (AggKind k : {AggKind::sum, AggKind::mean, AggKind::max, AggKind::min})
    CHECK(aggregate(v, {0, 0}, 3, k).to_host()[2] == 0.0);
  auto neg = DeviceMatrix<double>::from_host(2, 1, std::vector<double>{-4, -2});
  CHECK(aggregate(neg, {0, 0}, 3, AggKind::max).to_host()[0] == -2.0);
}

TEST_CASE("errors: bad index (test_aggregate.cpp:48-55)") {
  auto v = DeviceMatrix<double>::from_host(2, 1, std::vector<double>{1, 2});
  CHECK_THROWS_AS(aggregate(v, {0, 5}, 2, AggKind::sum), std::out_of_range);
}

TEST_CASE("max routes to the first attaining position (test_aggregate.cpp:127-134)") {
  EdgeIndex e({0, 1, 2}, {0, 0, 0}, 3, 1);
  DeviceArray<std::int32_t> arg;
  auto out = neighbor_aggregate(e, DeviceMatrix<double>::from_host(3, 1, std::vector<double>{5, 5, 1}), AggKind::max,
                                &arg);
  CHECK(out.to_host()[0] == 5.0);
  CHECK(arg.to_host()[0] == 0);
}

TEST_CASE("grouped_matmul equals independent per-group matmuls; empty groups; errors (test_hetero.cpp:61-92)") {
  const auto h0 = random_values(2 * 3, 201), h1 = random_values(4 * 3, 202), w = random_values(2 * 3 * 5, 203);
  auto to_bf = [](const std::vector<double>& v) {
    std::vector<bf16> o;
    for (double d : v) o.push_back(bf16::from_float(static_cast<float>(d)));
    return o;
  };
  const auto wb = to_bf(w);
  std::vector<DeviceMatrix<bf16>> ins{DeviceMatrix<bf16>::from_host(2, 3, to_bf(h0)),
                                      DeviceMatrix<bf16>::from_host(4, 3, to_bf(h1))};
  auto outs = grouped_matmul(ins, DeviceArray<bf16>::from_host(wb), 2, 3, 5);
  REQUIRE(outs.size() == 2);
  CHECK(outs[0].rows() == 2);
  CHECK(outs[1].rows() == 4);
  const std::vector<std::vector<double>*> hs{const_cast<std::vector<double>*>(&h0), const_cast<std::vector<double>*>(&h1)};
  for (std::size_t g = 0; g < 2; ++g) {
    const auto got = outs[g].to_host();
    const auto hb = to_bf(*hs[g]);
    for (Index r = 0; r < outs[g].rows(); ++r)
      for (Index j = 0; j < 5; ++j) {
        double want = 0, scale = 0;
        for (Index k = 0; k < 3; ++k) {
          const double a = hb[static_cast<std::size_t>(r * 3 + k)].to_float();
          const double b = wb[g * 15 + static_cast<std::size_t>(k * 5 + j)].to_float();
          want += a * b;
          scale += std::abs(a * b);
        }
        CHECK(std::abs(got[static_cast<std::size_t>(r * 5 + j)] - want) <= 1e-5 * scale + 1e-7);
      }
  }
  std::vector<DeviceMatrix<bf16>> with_empty{DeviceMatrix<bf16>(0, 3), ins[1]};
  CHECK(grouped_matmul(with_empty, DeviceArray<bf16>::from_host(wb), 2, 3, 5)[0].rows() == 0);
  CHECK_THROWS_AS(grouped_matmul({ins[0]}, DeviceArray<bf16>::from_host(wb), 2, 3, 5), std::invalid_argument);
  CHECK_THROWS_AS(grouped_matmul({ins[0], DeviceMatrix<bf16>(2, 4)}, DeviceArray<bf16>::from_host(wb), 2, 3, 5),
                  std::invalid_argument);
}

TEST_CASE("gcn layer: tcgen05 transform + fused bias/relu epilogue (message_passing.hpp:490-499, 578)") {
  // 3-node path with self loops: out = A_hat (h W) + b, relu when asked
  EdgeIndex e({0, 1, 1, 2}, {1, 0, 2, 1}, 3, 3);
  const std::vector<float> h{1, 2, -1, 0.5f, 3, -2}, w{0.5f, -1, 2, 0.25f}, b{0.1f, -5};
  auto hm = DeviceMatrix<float>::from_host(3, 2, h);
  auto wm = DeviceMatrix<float>::from_host(2, 2, w);
  auto bias = DeviceArray<float>::from_host(b);
  std::vector<double> xw(6, 0);
  for (int r = 0; r < 3; ++r)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k) xw[r * 2 + j] += double(h[r * 2 + k]) * w[k * 2 + j];
  const double deg[3] = {2, 3, 2};  // in-degree + self loop
  const std::vector<std::vector<int>> in{{1}, {0, 2}, {1}};
  const auto got = gcn_layer(e, hm, wm, bias).to_host();
  const auto got_relu = gcn_layer(e, hm, wm, bias, true).to_host();
  for (int v = 0; v < 3; ++v)
    for (int j = 0; j < 2; ++j) {
      double want = xw[v * 2 + j] / deg[v];
      for (int s : in[v]) want += xw[s * 2 + j] / std::sqrt(deg[s] * deg[v]);
      want += b[j];
      CHECK(std::abs(got[v * 2 + j] - want) <= 1e-5 * (std::abs(want) + 1));
      CHECK(got_relu[v * 2 + j] == (got[v * 2 + j] > 0 ? got[v * 2 + j] : 0.0f));
    }
}

TEST_CASE("fp32 grouped_matmul over separate tensors (hetero.hpp:134-157, grouped_matmul<float>)") {
  const auto h0 = random_values(300 * 128, 301), h1 = random_values(7 * 128, 302), w = random_values(2 * 128 * 64, 303);
  auto f = [](const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); };
  std::vector<DeviceMatrix<float>> ins{DeviceMatrix<float>::from_host(300, 128, f(h0)),
                                       DeviceMatrix<float>::from_host(7, 128, f(h1))};
  auto outs = grouped_matmul(ins, DeviceArray<float>::from_host(f(w)), 2, 128, 64);
  const std::vector<const std::vector<double>*> hs{&h0, &h1};
  for (std::size_t g = 0; g < 2; ++g) {
    const auto got = outs[g].to_host();
    for (Index r = 0; r < outs[g].rows(); ++r)
      for (Index j = 0; j < 64; ++j) {
        double want = 0, scale = 0;
        for (Index k = 0; k < 128; ++k) {
          const double a = float((*hs[g])[static_cast<std::size_t>(r * 128 + k)]);
          const double bb = float(w[g * 128 * 64 + static_cast<std::size_t>(k * 64 + j)]);
          want += a * bb;
          scale += std::abs(a * bb);
        }
        CHECK(std::abs(got[static_cast<std::size_t>(r * 64 + j)] - want) <= 1e-5 * scale + 1e-7);
      }
  }
}

TEST_CASE("max backward lands on the first attaining edge (aggregate.hpp:295-308)") {
  // destinations 0 and 1; edges (src -> dst): 0->0, 1->0, 2->0, 2->1, 0->1
  EdgeIndex e({0, 1, 2, 2, 0}, {0, 0, 0, 1, 1}, 3, 2);
  auto x = DeviceMatrix<double>::from_host(3, 1, std::vector<double>{5, 5, 1});
  DeviceArray<std::int32_t> arg;
  neighbor_aggregate(e, x, AggKind::max, &arg);
  auto g = DeviceMatrix<double>::from_host(2, 1, std::vector<double>{10, 7});
  const auto dx = neighbor_aggregate_backward(e, g, arg).to_host();
  // row 0: tie 5/5 -> edge 0 (src 0); row 1: max(1, 5) -> edge 4 (src 0)
  CHECK(dx == std::vector<double>{17, 0, 0});
}

TEST_CASE("DistSpmm over a 1-rank NCCL communicator equals the single-GPU spmm") {
  unsigned char id[128];
  REQUIRE(gm_nccl_unique_id(id) == GM_OK);
  ncclComm_t comm = nullptr;
  REQUIRE(gm_nccl_comm_init(1, id, 0, &comm) == GM_OK);
  {
    Stream s = test_stream(77);
    std::vector<Index> src(20000), dst(20000);
    for (std::size_t i = 0; i < src.size(); ++i) {
      src[i] = static_cast<Index>(s.next_below(3000));
      dst[i] = static_cast<Index>(s.next_below(3000));
    }
    EdgeIndex e(src, dst, 3000, 3000);
    const auto xh = random_values(3000 * 16, 78);
    auto x = DeviceMatrix<double>::from_host(3000, 16, xh);
    DistSpmm ds(e.to_csc(), 3000, 0, 1, comm);
    CHECK(ds(x, AggKind::sum).to_host() == neighbor_aggregate(e, x, AggKind::sum).to_host());
    DeviceArray<std::int32_t> a1, a2;
    CHECK(ds(x, AggKind::max, &a1).to_host() == neighbor_aggregate(e, x, AggKind::max, &a2).to_host());
    CHECK(a1.to_host() == a2.to_host());
  }
  CHECK(gm_nccl_comm_destroy(comm) == GM_OK);
}

TEST_CASE("PushSpmm: two virtual ranks push their rows into each other's next-layer replica") {
  Stream s = test_stream(91);
  const Index n = 4000;
  std::vector<Index> src(60000), dst(60000);
  for (std::size_t i = 0; i < src.size(); ++i) {
    src[i] = static_cast<Index>(s.next_below(n));
    dst[i] = static_cast<Index>(s.next_below(n));
  }
  EdgeIndex e(src, dst, n, n);
  const auto xh = random_values(static_cast<std::size_t>(n) * 8, 92);
  auto x0 = DeviceMatrix<float>::from_host(n, 8, std::vector<float>(xh.begin(), xh.end()));
  auto x1 = DeviceMatrix<float>::from_host(n, 8, std::vector<float>(xh.begin(), xh.end()));
  DeviceMatrix<float> b0(n, 8), b1(n, 8);
  const Index cut = 1700;
  PushSpmm rank0(e.to_csc(), 0, cut, {b1.data()});
  PushSpmm rank1(e.to_csc(), cut, n, {b0.data()});
  rank0(x0, b0, AggKind::mean);
  rank1(x1, b1, AggKind::mean);
  const auto want = neighbor_aggregate(e, x0, AggKind::mean).to_host();
  CHECK(b0.to_host() == want);
  CHECK(b1.to_host() == want);
  CHECK_THROWS_AS(rank0(x0, b0, AggKind::max), std::invalid_argument);  // max needs the argmax buffer
  DeviceArray<std::int32_t> arg0, arg1, want_arg;
  rank0(x0, b0, AggKind::max, &arg0);
  rank1(x1, b1, AggKind::max, &arg1);
  const auto want_max = neighbor_aggregate(e, x0, AggKind::max, &want_arg).to_host();
  CHECK(b0.to_host() == want_max);
  CHECK(b1.to_host() == want_max);
  auto wa = want_arg.to_host();
  auto a0 = arg0.to_host(), a1 = arg1.to_host();
  a0.insert(a0.end(), a1.begin(), a1.end());
  CHECK(a0 == wa);
}
