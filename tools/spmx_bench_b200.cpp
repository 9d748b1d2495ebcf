// spmx_bench_b200 — the reference's benchmark driver (tools/bench.cpp: `spmx_bench`) for the
// B200 path: same options, same report fields and column order (JSON or CSV), same exit codes
// (0 ok, 1 usage/runtime error, 2 verification failure), plus the GPU-side fields
// bytes_algorithmic, gbs, roofline_frac, n_chunks, gpus. SURVEY.md §8 row f1.
//
//   spmx_bench_b200 [--matrix f.mtx|f.jspm | --synthetic ROWS [--avg-nnz A] [--skew S]
//                    | --config c1..c5 [--scale S | --rows R]]   (BASELINE.json's configurations,
//                                                                 host/spmx_workloads.hpp; X and d come with them)
//                   [--cols D] [--strategy row|nnz|merge] [--dispatch static|dynamic]
//                   [--backend native|interp] [--threads T] [--batch-size B] [--trials K]
//                   [--seed S] [--verify] [--no-jit] [--format json|csv] [--report FILE]
//                   [--save-cache f.jspm] [--peak-gbs G] [--gpus G] [--shards S] [--shard-by nnz|merge]
//   spmx_bench_b200 sweep [common options] [--d-list 16 32 ...] [--strategies row nnz merge]
//                   [--backends native interp] [--dispatch static|dynamic]
//
// backend "native" = default device mode; "interp" = exact-order mode (bitwise equal to the
// reference's result, so y_checksum can be compared with a report of the reference's CLI).
// --tier, --counters, --dump-plan, --dump-code are x86-only and rejected with a usage error.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../paper_2312_05639_b200/host/spmx_b200.hpp"
#include "../paper_2312_05639_b200/host/spmx_io.hpp"
#include "../paper_2312_05639_b200/host/spmx_workloads.hpp"

using namespace spmx;

namespace {

struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };

struct Cli {
  std::string matrix_path;
  int64_t synthetic_rows = 0;
  double avg_nnz = 16.0, skew = 0.0;
  int cols = 16;
  bool cols_given = false;
  std::string config;  // BASELINE.json configuration c1 .. c5
  int scale = 0;
  int64_t rows = 0;
  std::string strategy = "row", dispatch = "dynamic", backend = "native";
  unsigned threads = 0, trials = 1;
  uint64_t batch_size = 128, seed = 42;
  bool verify = false, jit = true;
  std::string format = "json", report_path, save_cache_path;
  double peak_gbs = 6551.0;  // measured HBM copy peak of this pool's B200s (MEASURED_PEAKS.json)
  unsigned gpus = 1, shards = 0;  // row-shard A over G GPUs (the library's multi-GPU driver)
  std::string shard_by = "nnz";
  bool sweep = false;
  std::vector<int> d_list{16, 32};
  std::vector<std::string> strategies{"row", "nnz", "merge"}, backends{"native", "interp"};
};

struct Row {  // one report entry; values already formatted as JSON scalars / arrays
  std::vector<std::pair<std::string, std::string>> kv;
  void num(const std::string& k, double v) { char b[64]; std::snprintf(b, sizeof b, "%.17g", v); kv.emplace_back(k, b); }
  void integer(const std::string& k, long long v) { kv.emplace_back(k, std::to_string(v)); }
  void u64(const std::string& k, uint64_t v) { kv.emplace_back(k, std::to_string(v)); }
  void str(const std::string& k, const std::string& v) {
    std::string e = "\"";
    for (char c : v) { if (c == '"' || c == '\\') e.push_back('\\'); e.push_back(c); }
    kv.emplace_back(k, e + "\"");
  }
  const std::string* find(const std::string& k) const {
    for (const auto& p : kv) if (p.first == k) return &p.second;
    return nullptr;
  }
  std::string json(int indent) const {
    std::string pad(size_t(indent), ' '), s = "{\n";
    for (size_t i = 0; i < kv.size(); ++i)
      s += pad + "  \"" + kv[i].first + "\": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
    return s + pad + "}";
  }
};

// same column order as the reference's report (tools/bench.cpp:109-113), GPU columns appended
const char* const kColumns[] = {"matrix", "m", "n", "nnz", "d", "strategy", "backend", "tier", "threads",
                                "batch_size", "trials", "times_s", "mean_s", "codegen_s", "codegen_pct",
                                "gflops", "memory_loads", "stores", "branches", "vector_arith",
                                "scalar_arith", "instructions", "y_checksum", "max_rel_err", "status",
                                "bytes_algorithmic", "gbs", "roofline_frac", "n_chunks", "gpus"};

std::string csv_header() {
  std::string s;
  for (const char* c : kColumns) s += std::string(s.empty() ? "" : ",") + c;
  return s + "\n";
}

std::string csv_row(const Row& r) {
  std::string s;
  bool first = true;
  for (const char* c : kColumns) {
    if (!first) s += ",";
    first = false;
    const std::string* v = r.find(c);
    if (!v) { if (std::string(c) == "status") s += "ok"; continue; }
    std::string t = *v;
    if (!t.empty() && t.front() == '"') t = t.substr(1, t.size() - 2);     // strings unquoted
    if (!t.empty() && t.front() == '[') {                                  // times_s: ';'-separated
      t = t.substr(1, t.size() - 2);
      for (char& ch : t) if (ch == ',') ch = ';';
      t.erase(std::remove(t.begin(), t.end(), ' '), t.end());
    }
    s += t;
  }
  return s + "\n";
}

Strategy parse_strategy(const std::string& s) {
  if (s == "row") return Strategy::RowSplit;
  if (s == "nnz") return Strategy::NnzSplit;
  if (s == "merge") return Strategy::MergeSplit;
  throw UsageError("--strategy: unknown strategy: " + s);
}

RunConfig make_run_config(const Cli& c) {
  RunConfig cfg;
  cfg.strategy = parse_strategy(c.strategy);
  if (c.dispatch != "static" && c.dispatch != "dynamic") throw UsageError("--dispatch: expected static or dynamic");
  cfg.dynamic_dispatch = c.dispatch == "dynamic" && cfg.strategy == Strategy::RowSplit;
  cfg.threads = c.threads;
  if (c.backend == "native") cfg.backend = Backend::Native;
  else if (c.backend == "interp") cfg.backend = Backend::Interp;
  else throw UsageError("--backend: unknown backend: " + c.backend);
  cfg.batch_size = c.batch_size;
  cfg.verify = c.verify;
  cfg.trials = c.trials;
  cfg.jit_width = c.jit;
  cfg.gpus = c.gpus;
  cfg.shards = c.shards;
  if (c.shard_by != "nnz" && c.shard_by != "merge") throw UsageError("--shard-by: expected nnz or merge");
  cfg.shard_by_merge = c.shard_by == "merge";
  return cfg;
}

workloads::Dist config_x_dist(const std::string& config) {
  return config == "c3" ? workloads::Dist::Normal : workloads::Dist::UniformPm1;
}

CsrMatrix load_input(const Cli& c, std::string& name) {
  if (!c.config.empty()) {
    name = c.config + (c.scale ? "@scale" + std::to_string(c.scale) : "") +
           (c.rows ? "@rows" + std::to_string(c.rows) : "");
    return workloads::make_config(c.config, c.scale, c.rows).a;
  }
  if (!c.matrix_path.empty()) {
    name = c.matrix_path;
    const std::string& p = c.matrix_path;
    if (p.size() > 5 && p.compare(p.size() - 5, 5, ".jspm") == 0) return load_csr_cache(p);
    return load_matrix_market(p);
  }
  if (c.synthetic_rows > 0) {
    name = "synthetic(" + std::to_string(c.synthetic_rows) + ")";
    return random_csr(c.synthetic_rows, c.avg_nnz, c.skew, c.seed ^ 0x5157a7e5u);  // as the reference
  }
  throw UsageError("--matrix: need --matrix or --synthetic");
}

Row report_row(const std::string& matrix, const CsrMatrix& a, int d, const RunConfig& cfg, const RunReport& rep,
               uint64_t y_checksum, double peak_gbs) {
  Row r;
  r.str("matrix", matrix);
  r.integer("m", a.m); r.integer("n", a.n); r.integer("nnz", a.nnz); r.integer("d", d);
  r.str("strategy", std::string(strategy_name(cfg.strategy)) + (cfg.dynamic_dispatch ? "+dynamic" : ""));
  r.str("backend", backend_name(cfg.backend));
  r.str("tier", "sm_100a");
  r.integer("threads", rep.threads);
  r.u64("batch_size", cfg.batch_size);
  r.integer("trials", cfg.trials);
  std::string ts = "[";
  for (size_t i = 0; i < rep.times_s.size(); ++i) {
    char b[64]; std::snprintf(b, sizeof b, "%.9g", rep.times_s[i]);
    ts += std::string(i ? ", " : "") + b;
  }
  r.kv.emplace_back("times_s", ts + "]");
  r.num("mean_s", rep.mean_s);
  r.num("codegen_s", rep.codegen_s);
  r.num("codegen_pct", rep.mean_s > 0 ? 100.0 * rep.codegen_s / rep.mean_s : 0.0);
  r.num("gflops", rep.gflops);
  r.u64("y_checksum", y_checksum);
  if (rep.max_rel_err) r.num("max_rel_err", *rep.max_rel_err);
  const double bytes = 8.0 * double(a.nnz) + 4.0 * double(a.m + 1) + 4.0 * double(a.n) * d + 4.0 * double(a.m) * d;
  r.num("bytes_algorithmic", bytes);
  r.num("gbs", rep.mean_s > 0 ? bytes / rep.mean_s / 1e9 : 0.0);
  r.num("roofline_frac", rep.mean_s > 0 ? bytes / rep.mean_s / 1e9 / peak_gbs : 0.0);
  r.u64("n_chunks", rep.n_chunks);
  r.integer("gpus", rep.gpus);
  if (rep.gpus > 1 || !rep.shard_rows.empty()) {
    r.num("x_broadcast_s", rep.x_broadcast_s);
    r.num("roofline_frac_all_gpus", rep.mean_s > 0 ? bytes / rep.mean_s / 1e9 / (peak_gbs * rep.gpus) : 0.0);
    std::string sr = "[";
    for (size_t i = 0; i < rep.shard_rows.size(); ++i)
      sr += std::string(i ? ", " : "") + "[" + std::to_string(rep.shard_rows[i].begin) + ", " +
            std::to_string(rep.shard_rows[i].end) + "]";
    r.kv.emplace_back("shard_rows", sr + "]");
  }
  return r;
}

void write_report(const Cli& c, const std::string& text) {
  if (c.report_path.empty()) { std::cout << text; return; }
  std::ofstream out(c.report_path);
  if (!out) throw std::runtime_error("cannot write report: " + c.report_path);
  out << text;
}

DenseMatrix dense_operand(const Cli& c, const CsrMatrix& a, int d, uint64_t seed) {
  if (!c.config.empty())  // the configuration's own X (its seed and distribution), d columns
    return workloads::dense(a.n, d, workloads::make_config_seed(c.config), config_x_dist(c.config));
  DenseMatrix x = random_dense(a.n > 0 ? a.n : 1, d, seed);
  if (a.n == 0) x.rows = 0;
  return x;
}

int run_single(const Cli& c) {
  std::string name;
  CsrMatrix a = load_input(c, name);
  if (!c.save_cache_path.empty()) save_csr_cache(a, c.save_cache_path);
  const int cols = (!c.config.empty() && !c.cols_given) ? workloads::config_width(c.config) : c.cols;
  const DenseMatrix x = dense_operand(c, a, cols, c.seed);
  const RunConfig cfg = make_run_config(c);
  auto [y, rep] = run_spmm(a, x, cfg);
  const Row r = report_row(name, a, cols, cfg, rep, checksum(y), c.peak_gbs);
  write_report(c, c.format == "csv" ? csv_header() + csv_row(r) : r.json(0) + "\n");
  if (rep.max_rel_err && *rep.max_rel_err > kVerifyTolerance) {
    std::cerr << "verification FAILED: max_rel_err = " << *rep.max_rel_err << "\n";
    return 2;
  }
  return 0;
}

int run_sweep(const Cli& c) {
  std::string name;
  CsrMatrix a = load_input(c, name);
  std::vector<Row> rows;
  bool failed = false;
  for (const std::string& strat : c.strategies)
    for (int d : c.d_list)
      for (const std::string& backend : c.backends) {
        Cli cell = c;
        cell.strategy = strat; cell.cols = d; cell.backend = backend;
        try {
          const RunConfig cfg = make_run_config(cell);
          const DenseMatrix x = dense_operand(c, a, d, c.seed);
          auto [y, rep] = run_spmm(a, x, cfg);
          Row r = report_row(name, a, d, cfg, rep, checksum(y), c.peak_gbs);
          r.str("status", "ok");
          if (rep.max_rel_err && *rep.max_rel_err > kVerifyTolerance) failed = true;
          rows.push_back(std::move(r));
        } catch (const std::exception& e) {
          Row r;
          r.str("matrix", name); r.integer("d", d); r.str("strategy", strat); r.str("backend", backend);
          r.str("status", std::string("skipped: ") + e.what());
          rows.push_back(std::move(r));
        }
      }
  std::string text;
  if (c.format == "csv") {
    text = csv_header();
    for (const Row& r : rows) text += csv_row(r);
  } else {
    text = "[\n";
    for (size_t i = 0; i < rows.size(); ++i) text += "  " + rows[i].json(2) + (i + 1 < rows.size() ? ",\n" : "\n");
    text += "]\n";
  }
  write_report(c, text);
  return failed ? 2 : 0;
}

Cli parse(int argc, char** argv) {
  Cli c;
  std::vector<std::string> args(argv + 1, argv + argc);
  size_t i = 0;
  if (!args.empty() && args[0] == "sweep") { c.sweep = true; i = 1; }
  auto is_opt = [](const std::string& s) { return s.size() > 2 && s[0] == '-' && s[1] == '-'; };
  while (i < args.size()) {
    std::string key = args[i++], inline_val;
    bool has_inline = false;
    if (!is_opt(key)) throw UsageError("unexpected argument: " + key);
    const size_t eq = key.find('=');
    if (eq != std::string::npos) { inline_val = key.substr(eq + 1); key = key.substr(0, eq); has_inline = true; }
    auto value = [&]() -> std::string {
      if (has_inline) return inline_val;
      if (i >= args.size() || is_opt(args[i])) throw UsageError(key + ": value expected");
      return args[i++];
    };
    auto values = [&]() {
      std::vector<std::string> v;
      if (has_inline) v.push_back(inline_val);
      while (i < args.size() && !is_opt(args[i])) v.push_back(args[i++]);
      if (v.empty()) throw UsageError(key + ": value expected");
      return v;
    };
    auto positive = [&](const std::string& s) {
      char* end = nullptr;
      const long long v = std::strtoll(s.c_str(), &end, 10);
      if (end == s.c_str() || *end || v <= 0) throw UsageError(key + ": positive number expected");
      return v;
    };
    if (key == "--matrix") c.matrix_path = value();
    else if (key == "--synthetic") c.synthetic_rows = std::atoll(value().c_str());
    else if (key == "--avg-nnz") c.avg_nnz = std::atof(value().c_str());
    else if (key == "--skew") c.skew = std::atof(value().c_str());
    else if (key == "--threads") c.threads = unsigned(std::strtoul(value().c_str(), nullptr, 10));
    else if (key == "--batch-size") c.batch_size = uint64_t(positive(value()));
    else if (key == "--trials") c.trials = unsigned(positive(value()));
    else if (key == "--seed") c.seed = std::strtoull(value().c_str(), nullptr, 10);
    else if (key == "--verify") c.verify = true;
    else if (key == "--jit") c.jit = true;
    else if (key == "--no-jit") c.jit = false;
    else if (key == "--format") { c.format = value(); if (c.format != "json" && c.format != "csv") throw UsageError("--format: json|csv"); }
    else if (key == "--report") c.report_path = value();
    else if (key == "--peak-gbs") c.peak_gbs = std::atof(value().c_str());
    else if (key == "--dispatch") c.dispatch = value();
    else if (key == "--gpus") c.gpus = unsigned(positive(value()));
    else if (key == "--shards") c.shards = unsigned(positive(value()));
    else if (key == "--shard-by") c.shard_by = value();
    else if (!c.sweep && key == "--cols") { c.cols = int(positive(value())); c.cols_given = true; }
    else if (key == "--config") c.config = value();
    else if (key == "--scale") c.scale = int(positive(value()));
    else if (key == "--rows") c.rows = positive(value());
    else if (!c.sweep && key == "--strategy") c.strategy = value();
    else if (!c.sweep && key == "--backend") c.backend = value();
    else if (!c.sweep && key == "--save-cache") c.save_cache_path = value();
    else if (c.sweep && key == "--d-list") { c.d_list.clear(); for (auto& s : values()) c.d_list.push_back(int(positive(s))); }
    else if (c.sweep && key == "--strategies") c.strategies = values();
    else if (c.sweep && key == "--backends") c.backends = values();
    else if (key == "--tier" || key == "--counters" || key == "--dump-plan" || key == "--dump-code")
      throw UsageError(key + ": x86-only option of the reference, not available on the B200 path");
    else if (key == "--help") { std::cout << "see the header of tools/spmx_bench_b200.cpp\n"; std::exit(0); }
    else throw UsageError("unknown option: " + key);
  }
  return c;
}

}  // namespace

int main(int argc, char** argv) {
  Cli c;
  try {
    c = parse(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n";
    return 1;
  }
  try {
    return c.sweep ? run_sweep(c) : run_single(c);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
