// gcol_b200 -- command-line front-end of the B200 colouring library: the
// `color`, `verify` and `bench` subcommands of the reference's tool
// (/root/reference/proj/tools/gcol_main.cpp:140-298) over the C ABI
// (include/gcol_cuda.h) and the text loaders (include/gcol_io.hpp).
//
// Same arguments, same output (stats JSON of bench.hpp:164-176, report JSON
// :178-205, CSV :207-227, the summary table and speed-up lines of
// gcol_main.cpp:270-296), same exit codes (gcol_main.cpp:20-23: 0 ok, 2 input
// / parse / format / capacity errors, 3 verification failure, 4 I/O).  What
// differs is underneath: every algorithm runs on the GPU (`seq` is the exact
// device First-Fit), `--threads` is recorded in the stats only, and
// verification is the device's verify_coloring.  With no usable GPU the
// library reports GCOL_ERR_NO_DEVICE and the tool exits 1: there is no CPU
// fallback.  `generate` and `lockstep` are not part of this path
// (paper_1505_04086_b200/graphs.py generates the workloads on the device).
// Arguments are parsed by hand: the reference's CLI11 is not vendored here.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "gcol_cuda.h"
#include "gcol_io.hpp"

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitInput = 2, kExitVerify = 3, kExitIo = 4;

struct CliError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw CliError{code, msg}; }

const char* const kAlgNames[3] = {"seq", "catalyurek", "rsoc"};

int algorithm_id(const std::string& name) {
  for (int i = 0; i < 3; ++i)
    if (name == kAlgNames[i]) return i;
  fail(kExitInput, "unknown algorithm '" + name + "' (expected seq, catalyurek, or rsoc)");
}

// GCOL_CHUNK_SIZE (gcol_main.cpp:48-60): validated as the reference does,
// then passed through (the device ignores chunk sizes).
gcol_cuda_options options_from_env() {
  gcol_cuda_options o;
  std::memset(&o, 0, sizeof o);
  o.struct_size = sizeof o;
  if (const char* raw = std::getenv("GCOL_CHUNK_SIZE")) {
    char* end = nullptr;
    const unsigned long long v = std::strtoull(raw, &end, 10);
    if (end == raw || *end != '\0' || v == 0)
      fail(kExitInput, "GCOL_CHUNK_SIZE must be a positive integer, got '" + std::string(raw) + "'");
    o.chunk_size = v;
  }
  return o;
}

// Library status -> exit code (the adapter's exception mapping, include/gcol_cuda.hpp).
[[noreturn]] void fail_status(int rc) {
  const std::string msg = gcol_cuda_last_error();
  switch (rc) {
    case GCOL_ERR_INVALID_ARGUMENT:
    case GCOL_ERR_CAPACITY:
      fail(kExitInput, msg);
    case GCOL_ERR_VERIFY:
    case GCOL_ERR_ROUND_CAP:
      fail(kExitVerify, msg);
    case GCOL_ERR_NO_DEVICE:
      fail(kExitUsage, "no usable CUDA device (this tool has no CPU fallback): " + msg);
    default:
      fail(kExitUsage, msg);
  }
}

struct DeviceGraph {
  gcol_cuda_graph* h = nullptr;
  explicit DeviceGraph(const gcol_io::HostCsr& g) {
    const int rc = gcol_cuda_graph_create(g.offsets.data(), g.cols.data(), g.n, g.m(), GCOL_MEM_HOST, -1, &h);
    if (rc != GCOL_OK) fail_status(rc);
  }
  ~DeviceGraph() {
    if (h) gcol_cuda_graph_destroy(h);
  }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
};

struct Run {
  gcol_cuda_stats s;
  std::vector<std::uint64_t> cpr;
  std::vector<std::int32_t> colors;
};

Run run_coloring(DeviceGraph& dg, std::int64_t n, int alg, unsigned threads, gcol_cuda_options opt) {
  if (threads < 1) fail(kExitInput, "thread_count must be at least 1");
  Run r;
  std::memset(&r.s, 0, sizeof r.s);
  r.cpr.assign(4096, 0);
  r.colors.assign(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)), -1);
  opt.thread_count = threads;
  r.s.conflicts_per_round = r.cpr.data();
  r.s.cpr_cap = r.cpr.size();
  const int rc = gcol_cuda_run_coloring(dg.h, alg, &opt, r.colors.data(), GCOL_MEM_HOST, &r.s);
  if (rc != GCOL_OK) fail_status(rc);
  r.colors.resize(static_cast<std::size_t>(n));
  r.cpr.resize(static_cast<std::size_t>(std::min<std::uint64_t>(r.s.cpr_len, r.cpr.size())));
  return r;
}

// ---- JSON in nlohmann's dump(2) layout: keys in alphabetical order, arrays
// one element per line (what the reference's to_json(...).dump(2) prints) ----

std::string pad(int k) { return std::string(static_cast<std::size_t>(k), ' '); }

std::string json_number(double x) {
  char buf[64];
  if (x == static_cast<double>(static_cast<long long>(x)) && std::abs(x) < 1e15)
    std::snprintf(buf, sizeof buf, "%.1f", x);
  else
    std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

template <class T>
std::string json_array(const std::vector<T>& v, int ind) {
  if (v.empty()) return "[]";
  std::string s = "[\n";
  for (std::size_t i = 0; i < v.size(); ++i)
    s += pad(ind + 2) + std::to_string(v[i]) + (i + 1 < v.size() ? ",\n" : "\n");
  return s + pad(ind) + "]";
}

std::string graph_stats_json(const gcol_io::HostCsr& g, std::int32_t max_degree, int ind) {
  return "{\n" + pad(ind + 2) + "\"max_degree\": " + std::to_string(max_degree) + ",\n" + pad(ind + 2) +
         "\"num_edges\": " + std::to_string(g.num_edges()) + ",\n" + pad(ind + 2) +
         "\"num_vertices\": " + std::to_string(g.n) + "\n" + pad(ind) + "}";
}

// to_json(ColoringStats), bench.hpp:164-176; extra = further top-level members
// (key, rendered value) merged in alphabetical order.
std::string stats_json(const Run& r, int ind, std::vector<std::pair<std::string, std::string>> extra = {}) {
  std::vector<std::pair<std::string, std::string>> kv = {
      {"algorithm", std::string("\"") + kAlgNames[r.s.algorithm] + "\""},
      {"barrier_events", std::to_string(r.s.barrier_events)},
      {"conflicts_per_round", json_array(r.cpr, ind + 2)},
      {"conflicts_total", std::to_string(r.s.conflicts_total)},
      {"fallback_triggered", r.s.fallback_triggered ? "true" : "false"},
      {"num_colors", std::to_string(r.s.num_colors)},
      {"rounds", std::to_string(r.s.rounds)},
      {"thread_count", std::to_string(r.s.thread_count)},
      {"wall_time_ns", std::to_string(r.s.wall_time_ns)},
  };
  for (auto& e : extra) kv.push_back(std::move(e));
  std::sort(kv.begin(), kv.end());
  std::string s = "{\n";
  for (std::size_t i = 0; i < kv.size(); ++i)
    s += pad(ind + 2) + "\"" + kv[i].first + "\": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
  return s + pad(ind) + "}";
}

// ---- argument cursor ----

struct Args {
  std::vector<std::string> v;
  std::size_t i = 0;
  bool done() const { return i >= v.size(); }
  const std::string& peek() const { return v[i]; }
  std::string take() { return v[i++]; }
  // "--name value" or "--name=value"
  bool option(const std::string& name, std::string& out) {
    const std::string& a = v[i];
    if (a == name) {
      if (i + 1 >= v.size()) fail(kExitUsage, name + " needs a value");
      out = v[i + 1];
      i += 2;
      return true;
    }
    if (a.rfind(name + "=", 0) == 0) {
      out = a.substr(name.size() + 1);
      ++i;
      return true;
    }
    return false;
  }
};

unsigned long long positive_number(const std::string& s, const std::string& what) {
  unsigned long long x = 0;
  if (!gcol_io::detail::whole_number(std::string_view(s), x) || x == 0)
    fail(kExitUsage, what + " must be a positive number, got '" + s + "'");
  return x;
}

std::vector<std::string> split_commas(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ','))
    if (!t.empty()) out.push_back(t);
  return out;
}

void check_format(const std::string& f) {
  if (f != "auto" && f != "mm" && f != "edgelist") fail(kExitUsage, "--format must be one of auto, mm, edgelist");
}

// ---- color (gcol_main.cpp:140-187) ----

int cmd_color(Args& a) {
  std::string input, format = "auto", algorithm = "seq", output, coloring_output, t;
  unsigned threads = 1;
  while (!a.done()) {
    if (a.option("--format", format)) check_format(format);
    else if (a.option("--algorithm", algorithm)) {}
    else if (a.option("--threads", t)) threads = static_cast<unsigned>(positive_number(t, "--threads"));
    else if (a.option("--output", output)) {}
    else if (a.option("--coloring-output", coloring_output)) {}
    else if (a.peek().rfind("--", 0) == 0) fail(kExitUsage, "unknown option " + a.peek());
    else if (input.empty()) input = a.take();
    else fail(kExitUsage, "unexpected argument " + a.peek());
  }
  if (input.empty()) fail(kExitUsage, "color: input is required");

  const gcol_io::HostCsr g = gcol_io::load_graph(input, format);
  const int alg = algorithm_id(algorithm);
  const gcol_cuda_options opt = options_from_env();
  DeviceGraph dg(g);
  const Run run = run_coloring(dg, g.n, alg, threads, opt);

  gcol_cuda_verify_report rep;
  std::memset(&rep, 0, sizeof rep);
  const int rc = gcol_cuda_verify_coloring(dg.h, run.colors.data(), g.n, GCOL_MEM_HOST, &rep, nullptr, nullptr, nullptr, 0);
  if (rc != GCOL_OK) fail_status(rc);
  if (rep.violations != 0) {
    std::cerr << "verification failed: " << rep.violations << " violation(s)\n";
    return kExitVerify;
  }
  const std::string stats =
      stats_json(run, 0, {{"graph_stats", graph_stats_json(g, g.max_degree(), 2)}});
  if (!coloring_output.empty()) {
    std::string s;
    for (const std::int32_t c : run.colors) s += std::to_string(c) + "\n";
    gcol_io::write_file(coloring_output, s);
  }
  if (output.empty()) {
    std::cout << stats << "\n";
  } else {
    gcol_io::write_file(output, stats + "\n");
    std::cout << "colored " << g.n << " vertices with " << run.s.num_colors << " colors in "
              << run.s.wall_time_ns / 1000000.0 << " ms (" << run.s.rounds << " round(s), " << run.s.conflicts_total
              << " conflict(s))\n";
  }
  return kExitOk;
}

// ---- verify (gcol_main.cpp:189-225) ----

int cmd_verify(Args& a) {
  std::string input, format = "auto", coloring;
  while (!a.done()) {
    if (a.option("--format", format)) check_format(format);
    else if (a.option("--coloring", coloring)) {}
    else if (a.peek().rfind("--", 0) == 0) fail(kExitUsage, "unknown option " + a.peek());
    else if (input.empty()) input = a.take();
    else fail(kExitUsage, "unexpected argument " + a.peek());
  }
  if (input.empty() || coloring.empty()) fail(kExitUsage, "verify: input and --coloring are required");

  const gcol_io::HostCsr g = gcol_io::load_graph(input, format);
  const std::vector<std::int32_t> colors = gcol_io::parse_coloring(gcol_io::read_file(coloring));
  if (static_cast<std::int64_t>(colors.size()) != g.n)
    fail(kExitInput, "coloring has " + std::to_string(colors.size()) + " entries but the graph has " +
                         std::to_string(g.n) + " vertices");
  DeviceGraph dg(g);
  constexpr std::int64_t kMaxShown = 20;
  std::uint32_t u[kMaxShown], v[kMaxShown];
  std::int32_t c[kMaxShown];
  gcol_cuda_verify_report rep;
  std::memset(&rep, 0, sizeof rep);
  int rc = gcol_cuda_verify_coloring(dg.h, colors.data(), g.n, GCOL_MEM_HOST, &rep, u, v, c, kMaxShown);
  if (rc != GCOL_OK) fail_status(rc);
  if (rep.violations == 0) {
    std::uint32_t k = 0;
    rc = gcol_cuda_count_colors(dg.h, colors.data(), g.n, GCOL_MEM_HOST, &k);
    if (rc != GCOL_OK) fail_status(rc);
    std::cout << "proper coloring with " << k << " colors\n";
    return kExitOk;
  }
  const std::int64_t shown = std::min<std::int64_t>(kMaxShown, static_cast<std::int64_t>(rep.violations));
  for (std::int64_t i = 0; i < shown; ++i) {
    if (v[i] == 0xFFFFFFFFu)
      std::cout << "vertex " << u[i] << " is uncolored\n";
    else
      std::cout << "edge (" << u[i] << ", " << v[i] << "): both endpoints have color " << c[i] << "\n";
  }
  if (static_cast<std::int64_t>(rep.violations) > kMaxShown)
    std::cout << "... and " << rep.violations - kMaxShown << " more\n";
  std::cout << rep.violations << " violation(s)\n";
  return kExitVerify;
}

// ---- bench (gcol_main.cpp:227-298; run_benchmark bench.hpp:115-150) ----

struct Aggregate {  // bench.hpp:63-71, :87-110
  unsigned thread_count = 1;
  double wall_mean = 0, conflicts_mean = 0, rounds_mean = 0;
  std::uint64_t wall_min = 0, wall_max = 0;
  std::uint32_t colors_median = 0;
};

struct Report {
  int alg = 0;
  std::vector<unsigned> threads;
  std::uint32_t repeats = 0;
  std::vector<Run> runs;
  std::vector<Aggregate> agg;
};

Report run_benchmark(DeviceGraph& dg, const gcol_io::HostCsr& g, int alg, const std::vector<unsigned>& threads,
                     std::uint32_t repeats, const gcol_cuda_options& opt) {
  Report rep;
  rep.alg = alg;
  rep.threads = threads;
  rep.repeats = repeats;
  for (const unsigned tc : threads) {
    Aggregate A;
    A.thread_count = tc;
    A.wall_min = UINT64_MAX;
    std::vector<std::uint32_t> colors;
    for (std::uint32_t r = 0; r < repeats; ++r) {
      Run run = run_coloring(dg, g.n, alg, tc, opt);
      gcol_cuda_verify_report vr;
      std::memset(&vr, 0, sizeof vr);
      const int rc = gcol_cuda_verify_coloring(dg.h, run.colors.data(), g.n, GCOL_MEM_HOST, &vr, nullptr, nullptr, nullptr, 0);
      if (rc != GCOL_OK) fail_status(rc);
      if (vr.violations != 0)
        fail(kExitVerify, std::string("benchmark run produced an improper coloring (") + kAlgNames[alg] + ", " +
                              std::to_string(tc) + " threads)");
      A.wall_mean += static_cast<double>(run.s.wall_time_ns);
      A.conflicts_mean += static_cast<double>(run.s.conflicts_total);
      A.rounds_mean += static_cast<double>(run.s.rounds);
      A.wall_min = std::min<std::uint64_t>(A.wall_min, run.s.wall_time_ns);
      A.wall_max = std::max<std::uint64_t>(A.wall_max, run.s.wall_time_ns);
      colors.push_back(run.s.num_colors);
      std::vector<std::int32_t>().swap(run.colors);
      rep.runs.push_back(std::move(run));
    }
    A.wall_mean /= repeats;
    A.conflicts_mean /= repeats;
    A.rounds_mean /= repeats;
    std::sort(colors.begin(), colors.end());
    A.colors_median = colors[(colors.size() - 1) / 2];  // lower median
    rep.agg.push_back(A);
  }
  return rep;
}

std::string report_json(const Report& R, const std::string& name, const gcol_io::HostCsr& g) {
  std::string s = "{\n  \"aggregate\": ";
  if (R.agg.empty()) s += "[]";
  else {
    s += "[\n";
    for (std::size_t i = 0; i < R.agg.size(); ++i) {
      const Aggregate& a = R.agg[i];
      s += "    {\n      \"conflicts_total_mean\": " + json_number(a.conflicts_mean) +
           ",\n      \"num_colors_median\": " + std::to_string(a.colors_median) +
           ",\n      \"rounds_mean\": " + json_number(a.rounds_mean) +
           ",\n      \"thread_count\": " + std::to_string(a.thread_count) +
           ",\n      \"wall_time_ns_max\": " + std::to_string(a.wall_max) +
           ",\n      \"wall_time_ns_mean\": " + json_number(a.wall_mean) +
           ",\n      \"wall_time_ns_min\": " + std::to_string(a.wall_min) + "\n    }" +
           (i + 1 < R.agg.size() ? ",\n" : "\n");
    }
    s += "  ]";
  }
  s += std::string(",\n  \"algorithm\": \"") + kAlgNames[R.alg] + "\"";
  s += ",\n  \"graph_name\": \"" + name + "\"";
  s += ",\n  \"graph_stats\": " + graph_stats_json(g, g.max_degree(), 2);
  s += ",\n  \"repeats\": " + std::to_string(R.repeats);
  s += ",\n  \"runs\": ";
  if (R.runs.empty()) s += "[]";
  else {
    s += "[\n";
    for (std::size_t i = 0; i < R.runs.size(); ++i)
      s += "    " + stats_json(R.runs[i], 4) + (i + 1 < R.runs.size() ? ",\n" : "\n");
    s += "  ]";
  }
  s += ",\n  \"thread_counts\": " + json_array(R.threads, 2);
  return s + "\n}";
}

int cmd_bench(Args& a) {
  std::string input, format = "auto", output, csv, t;
  std::vector<std::string> algorithms{"seq", "catalyurek", "rsoc"};
  std::vector<unsigned> threads{1};
  std::uint32_t repeats = 10;
  while (!a.done()) {
    if (a.option("--format", format)) check_format(format);
    else if (a.option("--algorithms", t)) algorithms = split_commas(t);
    else if (a.option("--threads", t)) {
      threads.clear();
      for (const std::string& x : split_commas(t)) {
        unsigned long long k = 0;
        if (!gcol_io::detail::whole_number(std::string_view(x), k)) fail(kExitUsage, "--threads: bad count '" + x + "'");
        threads.push_back(static_cast<unsigned>(k));
      }
    } else if (a.option("--repeats", t)) repeats = static_cast<std::uint32_t>(positive_number(t, "--repeats"));
    else if (a.option("--output", output)) {}
    else if (a.option("--csv", csv)) {}
    else if (a.peek().rfind("--", 0) == 0) fail(kExitUsage, "unknown option " + a.peek());
    else if (input.empty()) input = a.take();
    else fail(kExitUsage, "unexpected argument " + a.peek());
  }
  if (input.empty()) fail(kExitUsage, "bench: input is required");

  const gcol_io::HostCsr g = gcol_io::load_graph(input, format);
  const gcol_cuda_options opt = options_from_env();
  const std::size_t slash = input.find_last_of('/');
  const std::string name = slash == std::string::npos ? input : input.substr(slash + 1);
  if (threads.empty()) fail(kExitInput, "run_benchmark: need at least one thread count");
  for (const unsigned tc : threads)
    if (tc < 1) fail(kExitInput, "run_benchmark: thread counts must be at least 1");

  DeviceGraph dg(g);
  std::vector<Report> reports;
  for (const std::string& n : algorithms) reports.push_back(run_benchmark(dg, g, algorithm_id(n), threads, repeats, opt));

  if (!output.empty()) {
    for (const Report& R : reports) {
      std::string path = output;
      if (reports.size() > 1) {  // stem-<algorithm>.ext
        const std::size_t sl = path.find_last_of('/');
        const std::size_t dot = path.find_last_of('.');
        const bool has_ext = dot != std::string::npos && (sl == std::string::npos || dot > sl + 1);
        const std::string ext = has_ext ? path.substr(dot) : "";
        path = (has_ext ? path.substr(0, dot) : path) + "-" + kAlgNames[R.alg] + ext;
      }
      gcol_io::write_file(path, report_json(R, name, g) + "\n");
    }
  }
  if (!csv.empty()) {
    std::string s = "algorithm,threads,run_index,rounds,conflicts_total,num_colors,wall_time_ns\n";
    for (const Report& R : reports) {
      std::size_t i = 0;
      for (const unsigned tc : R.threads)
        for (std::uint32_t r = 0; r < R.repeats; ++r, ++i) {
          const gcol_cuda_stats& st = R.runs[i].s;
          s += std::string(kAlgNames[st.algorithm]) + "," + std::to_string(tc) + "," + std::to_string(r) + "," +
               std::to_string(st.rounds) + "," + std::to_string(st.conflicts_total) + "," +
               std::to_string(st.num_colors) + "," + std::to_string(st.wall_time_ns) + "\n";
        }
    }
    gcol_io::write_file(csv, s);
  }

  std::printf("graph %s: %lld vertices, %lld edges, max degree %d\n", name.c_str(), static_cast<long long>(g.n),
              static_cast<long long>(g.num_edges()), g.max_degree());
  std::printf("%-12s%9s%14s%12s%12s%10s\n", "algorithm", "threads", "mean ms", "rounds", "conflicts", "colors");
  for (const Report& R : reports)
    for (const Aggregate& A : R.agg)
      std::printf("%-12s%9u%14.3f%12.2f%12.1f%10u\n", kAlgNames[R.alg], A.thread_count, A.wall_mean / 1e6, A.rounds_mean,
                  A.conflicts_mean, A.colors_median);
  // relative_speedup (bench.hpp:152-162): mean wall time of j over that of i
  for (std::size_t j = 0; j < reports.size(); ++j)
    for (std::size_t i = j + 1; i < reports.size(); ++i)
      for (const Aggregate& ta : reports[i].agg)
        for (const Aggregate& tb : reports[j].agg)
          if (ta.thread_count == tb.thread_count && ta.wall_mean > 0)
            std::printf("speedup of %s over %s at %u thread(s): %.3f\n", kAlgNames[reports[i].alg],
                        kAlgNames[reports[j].alg], ta.thread_count, tb.wall_mean / ta.wall_mean);
  return kExitOk;
}

const char* const kUsage =
    "B200 graph colouring toolkit (RSOC of arXiv 1505.04086 on the GPU)\n"
    "usage: gcol_b200 <subcommand> [options]\n"
    "  color  <graph> [--format auto|mm|edgelist] [--algorithm seq|catalyurek|rsoc] [--threads N]\n"
    "         [--output stats.json] [--coloring-output colors.txt]\n"
    "  verify <graph> --coloring colors.txt [--format ...]\n"
    "  bench  <graph> [--format ...] [--algorithms a,b,c] [--threads t1,t2] [--repeats K]\n"
    "         [--output report.json] [--csv runs.csv]\n"
    "exit codes: 0 ok, 2 bad input, 3 verification failed, 4 I/O error\n"
    "(generate and lockstep of the reference tool are not part of the GPU path)\n";

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) a.v.emplace_back(argv[i]);
  if (a.done()) {
    std::cerr << kUsage;
    return kExitUsage;
  }
  const std::string sub = a.take();
  if (sub == "--help" || sub == "-h" || sub == "help") {
    std::cout << kUsage;
    return kExitOk;
  }
  try {
    if (sub == "color") return cmd_color(a);
    if (sub == "verify") return cmd_verify(a);
    if (sub == "bench") return cmd_bench(a);
    std::cerr << "unknown subcommand '" << sub << "'\n" << kUsage;
    return kExitUsage;
  } catch (const gcol_io::error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return e.exit_code();
  } catch (const CliError& e) {
    std::cerr << "error: " << e.msg << "\n";
    return e.code;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}
