// ref_wrapper.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see gcol_oracle.h).  This file contains no
// reference code: it #includes the reference's header-only library from
// /root/reference/proj/include (path set by oracle/Makefile) and exposes the
// hot-path entry points with plain C types so tests/ and bench.py's
// reference arm can call the reference itself.  The build output lands in
// oracle/_ref/ (git-ignored, shipped to the GPU box like any built .so).
//
// Entry points wrapped (all /root/reference/proj/include/gcol/...):
//   build_graph            graph.hpp:98-138
//   color_rsoc             parallel.hpp:253-319
//   color_catalyurek       parallel.hpp:184-246
//   first_fit_sequential   coloring.hpp:110-116
//   smallest_available_color coloring.hpp:95-106
//   detect_conflicts       coloring.hpp:133-141
//   verify_coloring        coloring.hpp:159-177
//   count_colors           coloring.hpp:181-196
//   lockstep_color         lockstep.hpp:37-78
//   generate_rmat / shuffle_vertices  rmat.hpp:82-155
//   load_edge_list / save_edge_list / load_matrix_market  graph_io.hpp:83-221
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcol/coloring.hpp"
#include "gcol/graph.hpp"
#include "gcol/graph_io.hpp"
#include "gcol/lockstep.hpp"
#include "gcol/parallel.hpp"
#include "gcol/rmat.hpp"

#include "gcol_oracle.h"  // oracle_stats layout (shared with the C restatement)

namespace {
thread_local std::string g_err;

// Error codes: 0 ok, -1 input_error, -2 capacity_error, -3 logic_error,
// -4 other exception, -5 parse_error, -6 unsupported_format_error.
int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const gcol::parse_error*>(&e)) return -5;
  if (dynamic_cast<const gcol::unsupported_format_error*>(&e)) return -6;
  if (dynamic_cast<const gcol::input_error*>(&e)) return -1;
  if (dynamic_cast<const gcol::capacity_error*>(&e)) return -2;
  if (dynamic_cast<const std::logic_error*>(&e)) return -3;
  return -4;
}

void fill_stats(const gcol::ColoringStats& s, oracle_stats* st) {
  st->algorithm = static_cast<int32_t>(s.algorithm);
  st->thread_count = s.thread_count;
  st->rounds = s.rounds;
  st->conflicts_total = s.conflicts_total;
  st->barrier_events = s.barrier_events;
  st->num_colors = s.num_colors;
  st->fallback_triggered = s.fallback_triggered ? 1u : 0u;
  st->wall_time_ns = s.wall_time_ns;
  st->cpr_len = s.conflicts_per_round.size();
  for (std::size_t i = 0; i < s.conflicts_per_round.size() && i < st->cpr_cap; ++i)
    st->conflicts_per_round[i] = s.conflicts_per_round[i];
}

gcol::Coloring to_coloring(const int32_t* colors, int64_t n) {
  gcol::Coloring c(static_cast<std::size_t>(n));
  if (n > 0) std::memcpy(c.colors.data(), colors, sizeof(int32_t) * static_cast<std::size_t>(n));
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_build_graph(const uint32_t* pairs, int64_t num_pairs, uint32_t n, int* status) {
  try {
    std::vector<std::pair<gcol::vertex_t, gcol::vertex_t>> edges(static_cast<std::size_t>(num_pairs));
    for (int64_t i = 0; i < num_pairs; ++i) edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    *status = 0;
    return new gcol::Graph(gcol::build_graph(std::move(edges), n));
  } catch (const std::exception& e) {
    *status = code_of(e);
    return nullptr;
  }
}

// Builds the reference Graph for a canonical CSR by feeding its upper
// triangle to build_graph (the only constructor the reference offers).
void* ref_graph_from_csr(const uint64_t* off, const uint32_t* cols, uint32_t n, int* status) {
  try {
    std::vector<std::pair<gcol::vertex_t, gcol::vertex_t>> edges;
    edges.reserve(static_cast<std::size_t>(off[n] / 2));
    for (uint32_t v = 0; v < n; ++v)
      for (uint64_t i = off[v]; i < off[v + 1]; ++i)
        if (cols[i] > v) edges.emplace_back(v, cols[i]);
    *status = 0;
    return new gcol::Graph(gcol::build_graph(std::move(edges), n));
  } catch (const std::exception& e) {
    *status = code_of(e);
    return nullptr;
  }
}

void ref_graph_free(void* g) { delete static_cast<gcol::Graph*>(g); }

// The reference's text loaders on an in-memory source.  format 1: edge list
// (num_vertices < 0: from the ids), 2: Matrix Market.  *line = the
// parse_error's line (0 otherwise).
void* ref_parse_text(const char* text, uint64_t len, int format, int64_t num_vertices, int* status,
                     uint64_t* line) {
  *line = 0;
  try {
    std::istringstream in(std::string(text, static_cast<std::size_t>(len)));
    *status = 0;
    if (format == 2) return new gcol::Graph(gcol::load_matrix_market(in));
    std::optional<gcol::vertex_t> n;
    if (num_vertices >= 0) n = static_cast<gcol::vertex_t>(num_vertices);
    return new gcol::Graph(gcol::load_edge_list(in, n));
  } catch (const gcol::parse_error& e) {
    *line = e.line();
    *status = code_of(e);
    return nullptr;
  } catch (const std::exception& e) {
    *status = code_of(e);
    return nullptr;
  }
}

// save_edge_list into a caller buffer; returns the text length (call with
// cap = 0 to size it).
uint64_t ref_save_edge_list(const void* gp, char* out, uint64_t cap) {
  std::ostringstream os;
  gcol::save_edge_list(os, *static_cast<const gcol::Graph*>(gp));
  const std::string s = os.str();
  if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return s.size();
}

uint32_t ref_num_vertices(const void* g) { return static_cast<const gcol::Graph*>(g)->num_vertices(); }
uint64_t ref_num_adjacency(const void* g) { return static_cast<const gcol::Graph*>(g)->adjacency().size(); }
uint32_t ref_max_degree(const void* g) { return static_cast<const gcol::Graph*>(g)->max_degree(); }

void ref_graph_csr(const void* gp, uint64_t* offsets_out, uint32_t* cols_out) {
  const auto* g = static_cast<const gcol::Graph*>(gp);
  std::memcpy(offsets_out, g->offsets().data(), sizeof(uint64_t) * g->offsets().size());
  if (!g->adjacency().empty())
    std::memcpy(cols_out, g->adjacency().data(), sizeof(uint32_t) * g->adjacency().size());
}

// alg: 0 seq (run_coloring's seq branch, bench.hpp:35-60 restated as a plain
// call of first_fit_sequential), 1 catalyurek, 2 rsoc.
int ref_color(const void* gp, int alg, uint32_t threads, uint64_t chunk_size,
              uint64_t min_chunk_size, uint64_t round_cap, int32_t* colors_out, oracle_stats* st) {
  try {
    const auto& g = *static_cast<const gcol::Graph*>(gp);
    gcol::ParallelOptions opt;
    opt.chunk_size = chunk_size;
    opt.min_chunk_size = min_chunk_size;
    opt.round_cap = round_cap;
    gcol::ColoringRun run;
    if (alg == 1) {
      run = gcol::color_catalyurek(g, threads, opt);
    } else if (alg == 2) {
      run = gcol::color_rsoc(g, threads, opt);
    } else {
      if (threads < 1) throw gcol::input_error("thread_count must be at least 1");
      run.coloring = gcol::first_fit_sequential(g);
      run.stats.algorithm = gcol::Algorithm::seq;
      run.stats.thread_count = threads;
      run.stats.rounds = 1;
      run.stats.conflicts_per_round = {0};
      run.stats.num_colors = gcol::count_colors(run.coloring);
    }
    if (!run.coloring.colors.empty())
      std::memcpy(colors_out, run.coloring.colors.data(), sizeof(int32_t) * run.coloring.colors.size());
    fill_stats(run.stats, st);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int32_t ref_smallest_available_color(const void* gp, const int32_t* colors, uint32_t v) {
  const auto& g = *static_cast<const gcol::Graph*>(gp);
  gcol::Coloring c = to_coloring(colors, g.num_vertices());
  gcol::ForbiddenMarks marks(g.max_degree() + 1);
  return gcol::smallest_available_color(g, c, v, marks);
}

int64_t ref_detect_conflicts(const void* gp, const int32_t* colors, int64_t ncolors,
                             const uint32_t* pending, int64_t npending, uint32_t* out) {
  try {
    const auto& g = *static_cast<const gcol::Graph*>(gp);
    gcol::Worklist wl(pending, pending + npending);
    gcol::Worklist d = gcol::detect_conflicts(g, to_coloring(colors, ncolors), wl);
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = d[i];
    return static_cast<int64_t>(d.size());
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int64_t ref_verify_coloring(const void* gp, const int32_t* colors, int64_t ncolors, uint32_t* out_u,
                            uint32_t* out_v, int32_t* out_c, int64_t cap) {
  try {
    const auto& g = *static_cast<const gcol::Graph*>(gp);
    gcol::ConflictReport r = gcol::verify_coloring(g, to_coloring(colors, ncolors));
    for (std::size_t i = 0; i < r.violations.size() && static_cast<int64_t>(i) < cap; ++i) {
      out_u[i] = r.violations[i].u;
      out_v[i] = r.violations[i].v;
      out_c[i] = r.violations[i].color;
    }
    return static_cast<int64_t>(r.violations.size());
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int64_t ref_count_colors(const int32_t* colors, int64_t n) {
  try {
    return gcol::count_colors(to_coloring(colors, n));
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_first_fit_sequential(const void* gp, int32_t* out) {
  const auto& g = *static_cast<const gcol::Graph*>(gp);
  gcol::Coloring c = gcol::first_fit_sequential(g);
  if (!c.colors.empty()) std::memcpy(out, c.colors.data(), sizeof(int32_t) * c.colors.size());
  return 0;
}

int64_t ref_lockstep_color(const void* gp, const uint32_t* lanes, int64_t nlanes, uint64_t round_cap,
                           int32_t* trace_out, int32_t* converged) {
  try {
    const auto& g = *static_cast<const gcol::Graph*>(gp);
    std::vector<unsigned> lane_of(lanes, lanes + nlanes);
    gcol::LockstepOutcome o = gcol::lockstep_color(g, lane_of, round_cap);
    *converged = o.converged ? 1 : 0;
    for (std::size_t r = 0; r < o.color_trace.size(); ++r)
      if (g.num_vertices() > 0)
        std::memcpy(trace_out + r * g.num_vertices(), o.color_trace[r].colors.data(),
                    sizeof(int32_t) * g.num_vertices());
    return static_cast<int64_t>(o.rounds_executed);
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

void* ref_generate_rmat(unsigned scale, uint64_t edge_factor, double a, double b, double c,
                        double d, uint64_t seed, int* status) {
  try {
    gcol::RmatParams p;
    p.scale = scale;
    p.edge_factor = edge_factor;
    p.a = a; p.b = b; p.c = c; p.d = d;
    p.seed = seed;
    *status = 0;
    return new gcol::Graph(gcol::generate_rmat(p));
  } catch (const std::exception& e) {
    *status = code_of(e);
    return nullptr;
  }
}

void* ref_shuffle_vertices(const void* gp, uint64_t seed, uint32_t* perm_out) {
  const auto& g = *static_cast<const gcol::Graph*>(gp);
  auto [h, perm] = gcol::shuffle_vertices(g, seed);
  if (!perm.empty()) std::memcpy(perm_out, perm.data(), sizeof(uint32_t) * perm.size());
  return new gcol::Graph(std::move(h));
}

}  // extern "C"
