// gcol_io_abi.cpp -- extern "C" surface of include/gcol_io.hpp (declared in
// include/gcol_io.h).  Host only; built into libgcol_io.so by build.py.
#include "gcol_io.h"

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "gcol_io.hpp"

struct gcol_io_graph {
  gcol_io::HostCsr csr;
  std::int32_t max_degree = 0;
  std::string text;  // last format_edge_list result
};

namespace {

thread_local std::string t_err;
thread_local std::uint64_t t_line = 0;

template <class F>
int guarded(F&& f) {
  t_err.clear();
  t_line = 0;
  try {
    f();
    return GCOL_IO_OK;
  } catch (const gcol_io::error& e) {
    t_err = e.what();
    t_line = e.line();
    return static_cast<int>(e.kind());
  } catch (const std::bad_alloc&) {
    t_err = "out of host memory";
    return GCOL_IO_ERR_CAPACITY;
  } catch (const std::exception& e) {
    t_err = e.what();
    return GCOL_IO_ERR_INPUT;
  }
}

gcol_io_graph* wrap(gcol_io::HostCsr&& c) {
  auto* g = new gcol_io_graph;
  g->csr = std::move(c);
  g->max_degree = g->csr.max_degree();
  return g;
}

}  // namespace

extern "C" {

const char* gcol_io_last_error(void) { return t_err.c_str(); }
uint64_t gcol_io_last_error_line(void) { return t_line; }

int gcol_io_parse(const char* text, uint64_t len, int32_t format, int64_t num_vertices, gcol_io_graph** out) {
  return guarded([&] {
    if (!out || (!text && len)) throw gcol_io::error(gcol_io::ErrorKind::input, "null argument");
    const std::string_view sv(text ? text : "", static_cast<std::size_t>(len));
    *out = wrap(format == GCOL_IO_MM ? gcol_io::parse_matrix_market(sv) : gcol_io::parse_edge_list(sv, num_vertices));
  });
}

int gcol_io_load(const char* path, int32_t format, gcol_io_graph** out) {
  return guarded([&] {
    if (!out || !path) throw gcol_io::error(gcol_io::ErrorKind::input, "null argument");
    const char* f = format == GCOL_IO_MM ? "mm" : format == GCOL_IO_EDGELIST ? "edgelist" : "auto";
    *out = wrap(gcol_io::load_graph(path, f));
  });
}

int gcol_io_build_graph(const uint32_t* pairs, uint64_t num_pairs, uint64_t num_vertices, gcol_io_graph** out) {
  return guarded([&] {
    if (!out || (!pairs && num_pairs)) throw gcol_io::error(gcol_io::ErrorKind::input, "null argument");
    gcol_io::EdgeSink sink;
    sink.reserve(static_cast<std::size_t>(num_pairs));
    for (uint64_t i = 0; i < num_pairs; ++i) sink.add(pairs[2 * i], pairs[2 * i + 1]);
    *out = wrap(sink.build(num_vertices));
  });
}

void gcol_io_graph_free(gcol_io_graph* g) { delete g; }
int64_t gcol_io_num_vertices(const gcol_io_graph* g) { return g->csr.n; }
int64_t gcol_io_num_adjacency(const gcol_io_graph* g) { return g->csr.m(); }
int32_t gcol_io_max_degree(const gcol_io_graph* g) { return g->max_degree; }
const int64_t* gcol_io_offsets(const gcol_io_graph* g) { return g->csr.offsets.data(); }
const int32_t* gcol_io_cols(const gcol_io_graph* g) { return g->csr.cols.data(); }

uint64_t gcol_io_format_edge_list(gcol_io_graph* g, const char** text) {
  g->text = gcol_io::format_edge_list(g->csr);
  if (text) *text = g->text.data();
  return g->text.size();
}

int gcol_io_save_edge_list(gcol_io_graph* g, const char* path) {
  return guarded([&] {
    if (!g || !path) throw gcol_io::error(gcol_io::ErrorKind::input, "null argument");
    gcol_io::write_file(path, gcol_io::format_edge_list(g->csr));
  });
}

int gcol_io_parse_coloring(const char* text, uint64_t len, int32_t** colors, uint64_t* count) {
  return guarded([&] {
    if (!colors || !count || (!text && len)) throw gcol_io::error(gcol_io::ErrorKind::input, "null argument");
    const auto v = gcol_io::parse_coloring(std::string_view(text ? text : "", static_cast<std::size_t>(len)));
    auto* p = static_cast<int32_t*>(std::malloc(std::max<std::size_t>(1, v.size()) * sizeof(int32_t)));
    if (!p) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(int32_t));
    *colors = p;
    *count = v.size();
  });
}

void gcol_io_free(void* p) { std::free(p); }

}  // extern "C"
