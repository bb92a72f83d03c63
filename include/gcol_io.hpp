// gcol_io.hpp -- host-side text ingestion for the B200 colouring library:
// edge lists, Matrix Market coordinate files and colouring files, turned into
// the canonical CSR the C ABI takes (int64 offsets, int32 sorted columns).
//
// Replaces, for users of the reference's front-end:
//   load_edge_list      /root/reference/proj/include/gcol/graph_io.hpp:83-106
//   save_edge_list      graph_io.hpp:110-117
//   load_matrix_market  graph_io.hpp:124-221
//   build_graph         graph.hpp:98-138 (canonical form: loops dropped,
//                       duplicates in either orientation collapsed, ids < n)
//   read_coloring_file  /root/reference/proj/tools/gcol_main.cpp:72-108
// Same accepted grammar, same error classes, same "line N: ..." messages and
// line numbers; a different machine: the whole source is scanned in place
// from one buffer (no per-line strings or token vectors), edges are packed
// into 64-bit keys (lo << 32 | hi) and put in order by an LSD radix sort over
// the bytes that vary, and the CSR is filled from the sorted keys in two
// sweeps.  Header-only, standard library only; nothing here touches the GPU.
#pragma once

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace gcol_io {

// Error taxonomy of errors.hpp:11-52; `exit_code` is what the reference CLI
// returns for the class (gcol_main.cpp:20-23, :419-440).
enum class ErrorKind { input = 1, parse = 2, unsupported_format = 3, capacity = 4, io = 5 };

class error : public std::runtime_error {
 public:
  error(ErrorKind k, const std::string& msg, std::size_t line = 0)
      : std::runtime_error(line ? "line " + std::to_string(line) + ": " + msg : msg), kind_(k), line_(line) {}
  ErrorKind kind() const noexcept { return kind_; }
  std::size_t line() const noexcept { return line_; }  // 1-based; 0 = not tied to a line
  int exit_code() const noexcept { return kind_ == ErrorKind::io ? 4 : 2; }

 private:
  ErrorKind kind_;
  std::size_t line_;
};

// Canonical CSR (graph.hpp:15-19): rows ascending, symmetric, no loops.
struct HostCsr {
  std::int64_t n = 0;
  std::vector<std::int64_t> offsets{0};  // n + 1
  std::vector<std::int32_t> cols;        // 2 * undirected edges
  std::int64_t m() const { return static_cast<std::int64_t>(cols.size()); }
  std::int64_t num_edges() const { return m() / 2; }
  std::int32_t max_degree() const {
    std::int64_t d = 0;
    for (std::int64_t v = 0; v < n; ++v) d = std::max(d, offsets[v + 1] - offsets[v]);
    return static_cast<std::int32_t>(d);
  }
};

constexpr std::uint64_t kIdLimit = 0xFFFFFFFFull;  // kNoVertex (types.hpp:11): ids must be below it

namespace detail {

inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// One line of the buffer at a time, split into at most kMaxTok tokens in place.
struct LineScanner {
  static constexpr int kMaxTok = 8;
  const char* p;
  const char* end;
  std::size_t line_no = 0;
  std::string_view tok[kMaxTok];
  int ntok = 0;  // tokens on the line (counted past kMaxTok, stored up to it)

  LineScanner(const char* b, const char* e) : p(b), end(e) {}

  // Advances to the next line; false at end of input.
  bool next() {
    if (p >= end) return false;
    ++line_no;
    ntok = 0;
    const char* q = p;
    while (q < end && *q != '\n') {
      while (q < end && *q != '\n' && is_space(*q)) ++q;
      const char* t = q;
      while (q < end && !is_space(*q)) ++q;
      if (q > t) {
        if (ntok < kMaxTok) tok[ntok] = std::string_view(t, static_cast<std::size_t>(q - t));
        ++ntok;
      }
    }
    p = q < end ? q + 1 : end;
    return true;
  }
  bool blank_or(char comment) const { return ntok == 0 || tok[0].front() == comment; }
};

template <class T>
inline bool whole_number(std::string_view s, T& out) {
  const auto r = std::from_chars(s.data(), s.data() + s.size(), out);
  return r.ec == std::errc{} && r.ptr == s.data() + s.size();
}

inline std::string lower(std::string_view s) {
  std::string o(s);
  for (char& c : o) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return o;
}

// LSD radix sort of 64-bit keys, skipping every byte on which all keys agree.
inline void radix_sort(std::vector<std::uint64_t>& a) {
  if (a.size() < 2) return;
  if (a.size() < 2048) {
    std::sort(a.begin(), a.end());
    return;
  }
  std::uint64_t all_or = 0, all_and = ~0ull;
  for (const std::uint64_t k : a) {
    all_or |= k;
    all_and &= k;
  }
  const std::uint64_t varying = all_or ^ all_and;
  std::vector<std::uint64_t> b(a.size());
  std::uint64_t* src = a.data();
  std::uint64_t* dst = b.data();
  for (int byte = 0; byte < 8; ++byte) {
    const int sh = byte * 8;
    if (((varying >> sh) & 0xFFu) == 0) continue;
    std::size_t hist[257] = {0};
    for (std::size_t i = 0; i < a.size(); ++i) ++hist[((src[i] >> sh) & 0xFFu) + 1];
    for (int i = 0; i < 256; ++i) hist[i + 1] += hist[i];
    for (std::size_t i = 0; i < a.size(); ++i) dst[hist[(src[i] >> sh) & 0xFFu]++] = src[i];
    std::swap(src, dst);
  }
  if (src != a.data()) std::copy(src, src + a.size(), a.data());
}

}  // namespace detail

// Accumulates raw (u, v) pairs in any order and orientation.
class EdgeSink {
 public:
  void reserve(std::size_t k) {
    raw_u_.reserve(k);
    raw_v_.reserve(k);
  }
  void add(std::uint32_t u, std::uint32_t v) {
    max_id_ = std::max(max_id_, std::max(u, v));
    raw_u_.push_back(u);
    raw_v_.push_back(v);
  }
  std::size_t size() const { return raw_u_.size(); }
  std::uint32_t max_id() const { return max_id_; }

  // build_graph (graph.hpp:98-138): the first pair, in input order, that names
  // an id >= n is an input error; loops dropped; duplicates collapsed.
  HostCsr build(std::uint64_t n) {
    // the device library's ids are int32 (include/gcol_cuda.h: n < 2^31)
    if (n > 0x7FFFFFFFull)
      throw error(ErrorKind::capacity, "vertex count " + std::to_string(n) + " exceeds the 31-bit id space of the device CSR");
    for (std::size_t i = 0; i < raw_u_.size(); ++i)
      if (raw_u_[i] >= n || raw_v_[i] >= n)
        throw error(ErrorKind::input, "edge (" + std::to_string(raw_u_[i]) + ", " + std::to_string(raw_v_[i]) +
                                          ") references a vertex id >= " + std::to_string(n));
    keys_.clear();
    keys_.reserve(raw_u_.size());
    for (std::size_t i = 0; i < raw_u_.size(); ++i) {
      const std::uint32_t u = raw_u_[i], v = raw_v_[i];
      if (u == v) continue;
      keys_.push_back((static_cast<std::uint64_t>(std::min(u, v)) << 32) | std::max(u, v));
    }
    std::vector<std::uint32_t>().swap(raw_u_);
    std::vector<std::uint32_t>().swap(raw_v_);
    detail::radix_sort(keys_);
    keys_.erase(std::unique(keys_.begin(), keys_.end()), keys_.end());

    HostCsr g;
    g.n = static_cast<std::int64_t>(n);
    g.offsets.assign(static_cast<std::size_t>(n) + 1, 0);
    for (const std::uint64_t k : keys_) {
      ++g.offsets[(k >> 32) + 1];
      ++g.offsets[(k & 0xFFFFFFFFull) + 1];
    }
    for (std::size_t i = 1; i < g.offsets.size(); ++i) g.offsets[i] += g.offsets[i - 1];
    g.cols.resize(2 * keys_.size());
    // Keys ascend by (lo, hi): row r first receives its lower neighbours (as
    // the `hi` of keys whose lo < r, in ascending lo) and then its higher ones
    // (keys with lo == r, ascending hi) -- each row fills in ascending order.
    std::vector<std::int64_t> fill(g.offsets.begin(), g.offsets.end() - 1);
    for (const std::uint64_t k : keys_) {
      const std::uint32_t lo = static_cast<std::uint32_t>(k >> 32), hi = static_cast<std::uint32_t>(k);
      g.cols[static_cast<std::size_t>(fill[lo]++)] = static_cast<std::int32_t>(hi);
      g.cols[static_cast<std::size_t>(fill[hi]++)] = static_cast<std::int32_t>(lo);
    }
    std::vector<std::uint64_t>().swap(keys_);
    return g;
  }

 private:
  std::vector<std::uint32_t> raw_u_, raw_v_;
  std::vector<std::uint64_t> keys_;
  std::uint32_t max_id_ = 0;
};

// "u v" per line, '#' comments and blank lines skipped, 0-based ids
// (graph_io.hpp:79-106).  num_vertices < 0: 1 + the largest id (0 if none).
inline HostCsr parse_edge_list(std::string_view text, std::int64_t num_vertices = -1) {
  detail::LineScanner L(text.data(), text.data() + text.size());
  EdgeSink sink;
  bool any = false;
  auto vertex_id = [&](std::string_view t) -> std::uint32_t {
    std::uint64_t id = 0;
    if (!detail::whole_number(t, id))
      throw error(ErrorKind::parse, "expected a non-negative integer vertex id, got '" + std::string(t) + "'", L.line_no);
    if (id >= kIdLimit)
      throw error(ErrorKind::parse, "vertex id " + std::to_string(id) + " does not fit 32 bits", L.line_no);
    return static_cast<std::uint32_t>(id);
  };
  while (L.next()) {
    if (L.blank_or('#')) continue;
    if (L.ntok != 2)
      throw error(ErrorKind::parse, "expected two vertex ids, got " + std::to_string(L.ntok) + " token(s)", L.line_no);
    const std::uint32_t u = vertex_id(L.tok[0]);
    const std::uint32_t v = vertex_id(L.tok[1]);
    sink.add(u, v);
    any = true;
  }
  const std::uint64_t n = num_vertices >= 0 ? static_cast<std::uint64_t>(num_vertices)
                                            : (any ? static_cast<std::uint64_t>(sink.max_id()) + 1 : 0);
  return sink.build(n);
}

// Matrix Market coordinate source (graph_io.hpp:119-221): pattern / real /
// integer, general / symmetric; values parsed and discarded; diagonal
// dropped; n = max(rows, cols).
inline HostCsr parse_matrix_market(std::string_view text) {
  detail::LineScanner L(text.data(), text.data() + text.size());
  if (!L.next()) throw error(ErrorKind::parse, "empty Matrix Market source", 1);
  if (L.ntok != 5 || detail::lower(L.tok[0]) != "%%matrixmarket")
    throw error(ErrorKind::parse, "malformed Matrix Market banner", L.line_no);
  const std::string object = detail::lower(L.tok[1]), format = detail::lower(L.tok[2]),
                    field = detail::lower(L.tok[3]), symmetry = detail::lower(L.tok[4]);
  if (object != "matrix") throw error(ErrorKind::unsupported_format, "unsupported Matrix Market object: " + object);
  if (format == "array") throw error(ErrorKind::unsupported_format, "array format is not supported");
  if (format != "coordinate") throw error(ErrorKind::parse, "unknown Matrix Market format: " + format, L.line_no);
  if (field == "complex") throw error(ErrorKind::unsupported_format, "complex field is not supported");
  const bool pattern = field == "pattern", real = field == "real";
  if (!pattern && !real && field != "integer")
    throw error(ErrorKind::parse, "unknown Matrix Market field: " + field, L.line_no);
  if (symmetry == "skew-symmetric" || symmetry == "hermitian")
    throw error(ErrorKind::unsupported_format, "unsupported symmetry: " + symmetry);
  if (symmetry != "general" && symmetry != "symmetric")
    throw error(ErrorKind::parse, "unknown Matrix Market symmetry: " + symmetry, L.line_no);

  std::uint64_t rows = 0, cols = 0, entries = 0;
  bool sized = false;
  while (L.next()) {
    if (L.blank_or('%')) continue;
    if (L.ntok != 3 || !detail::whole_number(L.tok[0], rows) || !detail::whole_number(L.tok[1], cols) ||
        !detail::whole_number(L.tok[2], entries))
      throw error(ErrorKind::parse, "expected size line 'rows cols entries'", L.line_no);
    sized = true;
    break;
  }
  if (!sized) throw error(ErrorKind::parse, "missing size line", L.line_no);
  const std::uint64_t n = std::max(rows, cols);
  if (n > kIdLimit)
    throw error(ErrorKind::capacity, "matrix dimension " + std::to_string(n) + " exceeds the 32-bit vertex id space");

  const int want = pattern ? 2 : 3;
  EdgeSink sink;
  sink.reserve(static_cast<std::size_t>(std::min<std::uint64_t>(entries, std::uint64_t{1} << 32)));
  std::uint64_t seen = 0;
  while (seen < entries && L.next()) {
    if (L.blank_or('%')) continue;
    if (L.ntok != want)
      throw error(ErrorKind::parse,
                  "expected " + std::to_string(want) + " tokens per entry, got " + std::to_string(L.ntok), L.line_no);
    std::uint64_t i = 0, j = 0;
    if (!detail::whole_number(L.tok[0], i) || !detail::whole_number(L.tok[1], j))
      throw error(ErrorKind::parse, "malformed entry indices", L.line_no);
    if (!pattern) {
      if (real) {
        double x = 0;
        if (!detail::whole_number(L.tok[2], x))
          throw error(ErrorKind::parse, "malformed real value '" + std::string(L.tok[2]) + "'", L.line_no);
      } else {
        std::int64_t x = 0;
        if (!detail::whole_number(L.tok[2], x))
          throw error(ErrorKind::parse, "malformed integer value '" + std::string(L.tok[2]) + "'", L.line_no);
      }
    }
    if (i < 1 || i > rows || j < 1 || j > cols)
      throw error(ErrorKind::input, "entry (" + std::to_string(i) + ", " + std::to_string(j) + ") at line " +
                                        std::to_string(L.line_no) + " is outside the declared " +
                                        std::to_string(rows) + " x " + std::to_string(cols) + " shape");
    ++seen;
    if (i != j) sink.add(static_cast<std::uint32_t>(i - 1), static_cast<std::uint32_t>(j - 1));
  }
  if (seen < entries)
    throw error(ErrorKind::parse,
                "unexpected end of data: got " + std::to_string(seen) + " of " + std::to_string(entries) + " entries",
                L.line_no);
  while (L.next())
    if (!L.blank_or('%')) throw error(ErrorKind::parse, "unexpected content after the declared entries", L.line_no);
  return sink.build(n);
}

// One colour per line, blank lines skipped, -1 = uncoloured
// (gcol_main.cpp:72-108).
inline std::vector<std::int32_t> parse_coloring(std::string_view text) {
  detail::LineScanner L(text.data(), text.data() + text.size());
  std::vector<std::int32_t> out;
  while (L.next()) {
    if (L.ntok == 0) continue;
    if (L.ntok != 1) throw error(ErrorKind::parse, "expected one color per line", L.line_no);
    std::string_view t = L.tok[0];
    if (!t.empty() && t.front() == '+') t.remove_prefix(1);  // std::stol accepts a sign
    long long x = 0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), x);
    if (r.ec == std::errc::result_out_of_range) throw error(ErrorKind::parse, "color value out of range", L.line_no);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
      throw error(ErrorKind::parse, "expected an integer color, got '" + std::string(L.tok[0]) + "'", L.line_no);
    if (x < -1 || x > INT32_MAX) throw error(ErrorKind::parse, "color value out of range", L.line_no);
    out.push_back(static_cast<std::int32_t>(x));
  }
  return out;
}

// Edge list text readable by parse_edge_list: a comment with the counts, then
// "u v" with u < v, ascending (graph_io.hpp:108-117).
inline std::string format_edge_list(const HostCsr& g) {
  std::string s = "# " + std::to_string(g.n) + " vertices, " + std::to_string(g.num_edges()) + " edges\n";
  s.reserve(s.size() + static_cast<std::size_t>(g.num_edges()) * 14);
  char buf[48];
  for (std::int64_t v = 0; v < g.n; ++v)
    for (std::int64_t e = g.offsets[v]; e < g.offsets[v + 1]; ++e)
      if (g.cols[static_cast<std::size_t>(e)] > v) {
        const int k = std::snprintf(buf, sizeof buf, "%lld %d\n", static_cast<long long>(v),
                                    g.cols[static_cast<std::size_t>(e)]);
        s.append(buf, static_cast<std::size_t>(k));
      }
  return s;
}

// ---- files ----

inline std::string read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw error(ErrorKind::io, "cannot open '" + path + "' for reading");
  std::string s;
  char buf[1 << 16];
  std::size_t k;
  while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, k);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) throw error(ErrorKind::io, "failed reading '" + path + "'");
  return s;
}

inline void write_file(const std::string& path, std::string_view text) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw error(ErrorKind::io, "cannot open '" + path + "' for writing");
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  if (std::fclose(f) != 0 || !ok) throw error(ErrorKind::io, "failed writing '" + path + "'");
}

// load_graph of gcol_main.cpp:25-35: format "auto" picks Matrix Market for
// .mtx / .mm, an edge list otherwise.
inline HostCsr load_graph(const std::string& path, const std::string& format = "auto") {
  std::string f = format;
  if (f == "auto") {
    const std::size_t dot = path.find_last_of('.'), slash = path.find_last_of('/');
    const std::string ext = dot != std::string::npos && (slash == std::string::npos || dot > slash) ? path.substr(dot) : "";
    f = (ext == ".mtx" || ext == ".mm") ? "mm" : "edgelist";
  }
  const std::string text = read_file(path);
  return f == "mm" ? parse_matrix_market(text) : parse_edge_list(text);
}

}  // namespace gcol_io
