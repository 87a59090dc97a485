// ref_dataset_gen.cpp — TEST INFRASTRUCTURE ONLY. Writes small datasets with
// the REFERENCE's own writer (graphmill::save_dataset, dataset_io.hpp:69-112)
// so the device ingestion path (paper_2507_16991_b200/dataset.py) is pinned to
// the reference's on-disk format, not to our reading of it.
//   usage: ref_dataset_gen <out_dir_f32> <out_dir_f64>
#include <cstdio>

#include "graphmill/dataset_io.hpp"
#include "graphmill/hetero.hpp"
#include "graphmill/random.hpp"

using namespace graphmill;

template <typename S>
static void build(const char* dir, std::uint64_t salt) {
  rng::Stream st(rng::derive(0x6461746173657421ull, salt));
  HeteroGraph<S> g;
  const Index np = 53, na = 31, fp = 8, fa = 5;
  Timestamps tp(np);
  for (Index i = 0; i < np; ++i) tp[static_cast<std::size_t>(i)] = static_cast<std::int64_t>(st.next_below(1000)) - 100;
  g.add_node_type("paper", Tensor<S>::rand_uniform({np, fp}, -1.0, 1.0, st), tp);
  g.add_node_type("author", Tensor<S>::rand_uniform({na, fa}, -1.0, 1.0, st));
  auto edges = [&](Index e, Index ns, Index nd) {
    std::vector<Index> s(static_cast<std::size_t>(e)), d(static_cast<std::size_t>(e));
    for (Index i = 0; i < e; ++i) {
      s[static_cast<std::size_t>(i)] = static_cast<Index>(st.next_below(static_cast<std::uint64_t>(ns)));
      d[static_cast<std::size_t>(i)] = static_cast<Index>(st.next_below(static_cast<std::uint64_t>(nd)));
    }
    return EdgeIndex(std::move(s), std::move(d), ns, nd);
  };
  Timestamps tw(211);
  for (auto& t : tw) t = static_cast<std::int64_t>(st.next_below(5000));
  g.add_edge_type({"author", "writes", "paper"}, edges(211, na, np), std::nullopt, tw);
  g.add_edge_type({"paper", "cites", "paper"}, edges(157, np, np));
  g.add_edge_type({"author", "knows", "author"}, edges(0, na, na));  // empty edge type
  save_dataset(g, dir);
}

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s <out_dir_f32> <out_dir_f64>\n", argv[0]);
    return 2;
  }
  build<float>(argv[1], 1);
  build<double>(argv[2], 2);
  return 0;
}
