// gcol_cuda.hpp -- C++ adapter: the reference's coloring API on the B200 path.
//
// Header-only; include it next to the reference's headers
// (/root/reference/proj/include/gcol/*.hpp) and link libgcol_cuda.so.  It
// gives reference users the same call shapes, types and exceptions:
//
//   gcol::color_rsoc(g, T, opt)         parallel.hpp:253  ->  gcol::cuda::color_rsoc(g, T, opt)
//   gcol::color_catalyurek(g, T, opt)   parallel.hpp:183  ->  gcol::cuda::color_catalyurek(g, T, opt)
//   gcol::run_coloring(g, alg, T, opt)  bench.hpp:35      ->  gcol::cuda::run_coloring(g, alg, T, opt)
//   gcol::first_fit_sequential(g)       coloring.hpp:110  ->  gcol::cuda::first_fit_sequential(g)
//   gcol::verify_coloring(g, c)         coloring.hpp:159  ->  gcol::cuda::verify_coloring(g, c)
//   gcol::count_colors(c)               coloring.hpp:181  ->  gcol::cuda::count_colors(g, c)
//
// gcol::Graph stores uint64 offsets and uint32 neighbours (graph.hpp:91-92);
// for ids < 2^31 those are bit-identical to the ABI's int64 / int32 arrays,
// so the CSR is handed over without conversion.  Status codes come back as
// the reference's exception types (errors.hpp:11-52).  There is no CPU
// fallback: without a device the calls throw.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcol/coloring.hpp"
#include "gcol/errors.hpp"
#include "gcol/graph.hpp"
#include "gcol/parallel.hpp"
#include "gcol_cuda.h"

namespace gcol {
namespace cuda {

inline void throw_status(int rc) {
  if (rc == GCOL_OK) return;
  const std::string msg = gcol_cuda_last_error();
  switch (rc) {
    case GCOL_ERR_INVALID_ARGUMENT: throw gcol::input_error(msg);
    case GCOL_ERR_CAPACITY: throw gcol::capacity_error(msg);
    case GCOL_ERR_VERIFY: throw gcol::verification_error(msg);
    case GCOL_ERR_ROUND_CAP:
      throw std::runtime_error("round_cap reached (no CPU repair on the GPU path): " + msg);
    default: throw std::runtime_error("gcol_cuda: " + msg);
  }
}

// Device-side knobs beyond ParallelOptions (include/gcol_cuda.h).
struct CudaOptions {
  int priority = GCOL_PRIORITY_DEFAULT;
  int k1_blocks_per_sm = 0;
  bool k1_read_all = false;
  int k1_split_min_degree = 0;
  int k1_wide = 0;
  int k1_wait_polls = 0;
};

// A gcol::Graph uploaded once to the device (reuse it across runs, like the
// reference shares an immutable Graph across threads).
class DeviceGraph {
 public:
  explicit DeviceGraph(const gcol::Graph& g) {
    if (g.num_vertices() >= 0x7fffffffu)
      throw gcol::capacity_error("vertex ids do not fit the int32 column type");
    gcol_cuda_graph* h = nullptr;
    throw_status(gcol_cuda_graph_create(
        reinterpret_cast<const int64_t*>(g.offsets().data()),
        reinterpret_cast<const int32_t*>(g.adjacency().data()),
        static_cast<int64_t>(g.num_vertices()), static_cast<int64_t>(g.adjacency().size()),
        GCOL_MEM_HOST, -1, &h));
    h_.reset(h);
  }
  gcol_cuda_graph* get() const { return h_.get(); }

 private:
  struct Del {
    void operator()(gcol_cuda_graph* h) const { gcol_cuda_graph_destroy(h); }
  };
  std::unique_ptr<gcol_cuda_graph, Del> h_;
};

inline gcol_cuda_options to_c(unsigned thread_count, const ParallelOptions& opt,
                              const CudaOptions& co) {
  gcol_cuda_options o{};
  o.struct_size = sizeof o;
  o.thread_count = thread_count;
  o.chunk_size = opt.chunk_size;
  o.min_chunk_size = opt.min_chunk_size;
  o.round_cap = opt.round_cap;
  o.priority = co.priority;
  o.k1_blocks_per_sm = co.k1_blocks_per_sm;
  o.k1_read_all = co.k1_read_all ? 1 : 0;
  o.k1_split_min_degree = co.k1_split_min_degree;
  o.k1_wide = co.k1_wide;
  o.k1_wait_polls = co.k1_wait_polls;
  return o;
}

inline void fill_stats(ColoringRun& run, const gcol_cuda_stats& st,
                       const std::vector<uint64_t>& cpr) {
  run.stats.algorithm = static_cast<Algorithm>(st.algorithm);
  run.stats.thread_count = st.thread_count;
  run.stats.rounds = st.rounds;
  run.stats.conflicts_total = st.conflicts_total;
  run.stats.conflicts_per_round.assign(cpr.begin(),
                                       cpr.begin() + static_cast<std::ptrdiff_t>(st.cpr_len));
  run.stats.barrier_events = st.barrier_events;
  run.stats.num_colors = st.num_colors;
  run.stats.wall_time_ns = st.wall_time_ns;
  run.stats.fallback_triggered = st.fallback_triggered != 0;
}

inline ColoringRun run_coloring(const DeviceGraph& dg, std::size_t n, Algorithm algorithm,
                                unsigned thread_count, const ParallelOptions& opt = {},
                                const CudaOptions& co = {}) {
  if (thread_count < 1) throw gcol::input_error("thread_count must be at least 1");
  ColoringRun run{Coloring(n), {}};
  std::vector<uint64_t> cpr(static_cast<std::size_t>(opt.round_cap) + 1);
  gcol_cuda_stats st{};
  st.conflicts_per_round = cpr.data();
  st.cpr_cap = cpr.size();
  const gcol_cuda_options o = to_c(thread_count, opt, co);
  throw_status(gcol_cuda_run_coloring(dg.get(), static_cast<int32_t>(algorithm), &o,
                                      run.coloring.colors.data(), GCOL_MEM_HOST, &st));
  fill_stats(run, st, cpr);
  return run;
}

// RSOC on a host gcol::Graph in one call: the upload of the adjacency
// overlaps the initial pass (gcol_cuda_color_rsoc_csr).
inline ColoringRun color_rsoc_host(const gcol::Graph& g, unsigned thread_count,
                                   const ParallelOptions& opt = {}, const CudaOptions& co = {}) {
  if (thread_count < 1) throw gcol::input_error("thread_count must be at least 1");
  if (g.num_vertices() >= 0x7fffffffu)
    throw gcol::capacity_error("vertex ids do not fit the int32 column type");
  ColoringRun run{Coloring(g.num_vertices()), {}};
  std::vector<uint64_t> cpr(static_cast<std::size_t>(opt.round_cap) + 1);
  gcol_cuda_stats st{};
  st.conflicts_per_round = cpr.data();
  st.cpr_cap = cpr.size();
  const gcol_cuda_options o = to_c(thread_count, opt, co);
  throw_status(gcol_cuda_color_rsoc_csr(
      reinterpret_cast<const int64_t*>(g.offsets().data()),
      reinterpret_cast<const int32_t*>(g.adjacency().data()),
      static_cast<int64_t>(g.num_vertices()), static_cast<int64_t>(g.adjacency().size()), -1, &o,
      run.coloring.colors.data(), &st));
  fill_stats(run, st, cpr);
  return run;
}

inline ColoringRun run_coloring(const gcol::Graph& g, Algorithm algorithm,
                                unsigned thread_count, const ParallelOptions& opt = {},
                                const CudaOptions& co = {}) {
  if (algorithm == Algorithm::rsoc) return color_rsoc_host(g, thread_count, opt, co);
  DeviceGraph dg(g);
  return run_coloring(dg, g.num_vertices(), algorithm, thread_count, opt, co);
}

inline ColoringRun color_rsoc(const gcol::Graph& g, unsigned thread_count,
                              const ParallelOptions& opt = {}, const CudaOptions& co = {}) {
  return color_rsoc_host(g, thread_count, opt, co);
}

// gcol::color_catalyurek (parallel.hpp:183) on the device.
inline ColoringRun color_catalyurek(const gcol::Graph& g, unsigned thread_count,
                                    const ParallelOptions& opt = {}, const CudaOptions& co = {}) {
  return run_coloring(g, Algorithm::catalyurek, thread_count, opt, co);
}

inline Coloring first_fit_sequential(const gcol::Graph& g) {
  DeviceGraph dg(g);
  Coloring c(g.num_vertices());
  throw_status(gcol_cuda_first_fit_sequential(dg.get(), c.colors.data(), GCOL_MEM_HOST));
  return c;
}

inline ConflictReport verify_coloring(const gcol::Graph& g, const Coloring& c) {
  if (c.size() != g.num_vertices())
    throw gcol::input_error("verify_coloring: coloring has " + std::to_string(c.size()) +
                            " entries, graph has " + std::to_string(g.num_vertices()) +
                            " vertices");
  DeviceGraph dg(g);
  gcol_cuda_verify_report rep{};
  throw_status(gcol_cuda_verify_coloring(dg.get(), c.colors.data(),
                                         static_cast<int64_t>(c.size()), GCOL_MEM_HOST, &rep,
                                         nullptr, nullptr, nullptr, 0));
  ConflictReport out;
  if (rep.violations == 0) return out;
  std::vector<uint32_t> u(rep.violations), v(rep.violations);
  std::vector<int32_t> col(rep.violations);
  throw_status(gcol_cuda_verify_coloring(dg.get(), c.colors.data(),
                                         static_cast<int64_t>(c.size()), GCOL_MEM_HOST, &rep,
                                         u.data(), v.data(), col.data(),
                                         static_cast<int64_t>(rep.violations)));
  for (std::size_t i = 0; i < u.size(); ++i) out.violations.push_back({u[i], v[i], col[i]});
  return out;
}

inline std::uint32_t count_colors(const gcol::Graph& g, const Coloring& c) {
  DeviceGraph dg(g);
  uint32_t k = 0;
  throw_status(gcol_cuda_count_colors(dg.get(), c.colors.data(), static_cast<int64_t>(c.size()),
                                      GCOL_MEM_HOST, &k));
  return k;
}

}  // namespace cuda
}  // namespace gcol
