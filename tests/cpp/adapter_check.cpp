// adapter_check.cpp -- the reference's own types and checkers driving the
// B200 path through include/gcol_cuda.hpp (a reference user's drop-in).
//
// Built in the build container by __graft_entry__.build() (needs the
// reference headers); the binary travels to the GPU box and is run by
// tests/test_gpu_adapter.py.  Graphs are built with gcol::build_graph and
// checked with gcol::verify_coloring / gcol::count_colors from the
// reference; first_fit_sequential must match the reference bit for bit.
#include <cstdio>
#include <random>
#include <vector>

#include "gcol/coloring.hpp"
#include "gcol/graph.hpp"
#include "gcol/parallel.hpp"
#include "gcol/rmat.hpp"
#include "gcol_cuda.hpp"

namespace {

int failures = 0;

void check(bool ok, const char* what) {
  if (!ok) {
    std::printf("FAIL: %s\n", what);
    ++failures;
  }
}

// test_parallel.cpp:18-36 invariants, checked with the reference verifier.
void check_run(const gcol::Graph& g, const gcol::ColoringRun& run, unsigned threads) {
  check(run.coloring.complete(), "complete");
  check(gcol::verify_coloring(g, run.coloring).ok(), "proper (reference verify_coloring)");
  check(run.stats.num_colors == gcol::count_colors(run.coloring), "num_colors == count_colors");
  check(run.stats.num_colors <= g.max_degree() + 1, "<= max_degree + 1");
  check(run.stats.thread_count == threads, "thread_count recorded");
  check(run.stats.rounds >= 1, "rounds >= 1");
  check(run.stats.conflicts_per_round.size() == run.stats.rounds, "cpr size");
  std::uint64_t sum = 0;
  for (auto c : run.stats.conflicts_per_round) sum += c;
  check(run.stats.conflicts_total == sum, "conflicts_total");
  check(run.stats.conflicts_per_round.back() == 0, "last round clean");
  check(run.stats.barrier_events == run.stats.rounds + 1, "barrier_events == rounds + 1");
}

gcol::Graph random_graph(std::mt19937_64& rng, gcol::vertex_t n, double avg) {
  std::vector<std::pair<gcol::vertex_t, gcol::vertex_t>> e;
  if (n >= 2) {
    std::uniform_int_distribution<gcol::vertex_t> pick(0, n - 1);
    for (std::uint64_t i = 0; i < static_cast<std::uint64_t>(n * avg / 2); ++i)
      e.emplace_back(pick(rng), pick(rng));
  }
  return gcol::build_graph(std::move(e), n);
}

}  // namespace

int main() {
  std::mt19937_64 rng(606);
  for (int round = 0; round < 30; ++round) {
    const auto n = static_cast<gcol::vertex_t>(1 + rng() % 5000);
    const gcol::Graph g = random_graph(rng, n, 2.0 + static_cast<double>(rng() % 80) / 10.0);
    for (unsigned t : {1u, 16u}) check_run(g, gcol::cuda::color_rsoc(g, t), t);
    {
      const gcol::ColoringRun c = gcol::cuda::color_catalyurek(g, 4);
      check(c.coloring.complete() && gcol::verify_coloring(g, c.coloring).ok(), "catalyurek proper");
      check(c.stats.barrier_events == 2 * c.stats.rounds, "catalyurek barrier_events");
      check(c.stats.conflicts_per_round.back() == 0, "catalyurek last round clean");
    }
    const gcol::Coloring seq = gcol::first_fit_sequential(g);
    check(gcol::cuda::first_fit_sequential(g) == seq, "first_fit_sequential bit-identical");
    const gcol::ColoringRun s = gcol::cuda::run_coloring(g, gcol::Algorithm::seq, 1);
    check(s.coloring == seq && s.stats.rounds == 1, "run_coloring(seq)");
    check(gcol::cuda::count_colors(g, seq) == gcol::count_colors(seq), "count_colors");
    gcol::Coloring bad = seq;
    if (g.num_edges() > 0) {
      const auto& adj = g.adjacency();
      gcol::vertex_t u = 0;
      while (g.degree(u) == 0) ++u;
      bad.colors[adj[g.offsets()[u]]] = bad.colors[u];
      check(gcol::cuda::verify_coloring(g, bad).violations ==
                gcol::verify_coloring(g, bad).violations,
            "verify_coloring report identical");
    }
  }
  // K12, star, lone vertex, empty graph (test_parallel.cpp:63-116)
  std::vector<std::pair<gcol::vertex_t, gcol::vertex_t>> k;
  for (gcol::vertex_t u = 0; u < 12; ++u)
    for (gcol::vertex_t v = u + 1; v < 12; ++v) k.emplace_back(u, v);
  const gcol::Graph k12 = gcol::build_graph(k, 12);
  check(gcol::cuda::color_rsoc(k12, 4).stats.num_colors == 12, "K12 -> 12");
  const gcol::Graph empty = gcol::build_graph({}, 0);
  const auto er = gcol::cuda::color_rsoc(empty, 2);
  check(er.stats.rounds == 1 && er.stats.barrier_events == 2, "empty graph: one round");
  bool threw = false;
  try {
    gcol::cuda::color_rsoc(k12, 0);
  } catch (const gcol::input_error&) {
    threw = true;
  }
  check(threw, "thread_count 0 -> input_error");
  // an R-MAT from the reference's own generator, shuffled like the paper
  gcol::RmatParams p = *gcol::rmat_preset("rmat-b");
  p.scale = 14;
  p.edge_factor = 8;
  p.seed = 914;
  const auto [rg, perm] = gcol::shuffle_vertices(gcol::generate_rmat(p), 7);
  check_run(rg, gcol::cuda::color_rsoc(rg, 8), 8);
  std::printf(failures ? "adapter_check: %d failures\n" : "adapter_check: OK\n", failures);
  return failures ? 1 : 0;
}
