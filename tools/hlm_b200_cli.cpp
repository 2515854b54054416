// hlm_b200_cli -- the reference's command-line harness (proj/tools/hlm_app.hpp) on libhlm_b200.so.
//
// Same subcommands, flags, CSV schema (hlm_app.hpp:121-140) and exit codes as `hlm_cli`:
//   run       one matcher on one instance file             (cmd_run      :212-218, execute_run :156-202)
//   bench     batch runs + per-instance means + geomeans   (cmd_bench    :232-333)
//   generate  tight | random instance files                (cmd_generate :349-372)
//   verify    a matching file against an instance          (cmd_verify   :379-394)
// Everything goes through the C-ABI (include/hlm_b200.h): instance files are parsed by the library's
// host code, the matching and verify_matching run on the GPU.  Extensions: --variant auto, --device,
// --gpus (edge blocks over several devices).  Not provided: the exact branch-and-bound oracle
// (exact.hpp:84, out of scope): `oracle` exits 2, `run --oracle` leaves ratio_vs_oracle blank like the
// reference does when its edge cap is exceeded.  --workers / --grain / --assert-crew are accepted and
// ignored (the device decides its own parallelism); the workers column holds the device's SM count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hlm_b200.h"

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct HostGraph {  // owns an hlm_b200_host_graph
  hlm_b200_host_graph g{};
  HostGraph() = default;
  HostGraph(const HostGraph&) = delete;
  HostGraph& operator=(const HostGraph&) = delete;
  ~HostGraph() { hlm_b200_host_graph_free(&g); }
  hlm_b200_csr_view view() const {
    return {g.num_vertices, g.num_edges, g.vertex_offsets, g.vertex_incidence, g.edge_offsets, g.edge_members, g.base_weights};
  }
  uint64_t pins() const { return g.num_edges ? g.edge_offsets[g.num_edges] : 0; }
};

[[noreturn]] void fail_lib(const std::string& what) { throw std::runtime_error(what + ": " + hlm_b200_last_error()); }

std::string read_file(const std::string& path, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error(std::string("cannot open ") + what + " " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

struct InstanceOptions {  // hlm_app.hpp:24-30
  std::string path, format = "auto", weights = "file";
  uint64_t weight_seed = 1;
  bool drop_isolated = false;
};

struct StreamOptions {  // hlm_app.hpp:32-37
  uint64_t seed = 1;
  std::string generator = "xorshift", noise = "0:100";
  bool uniform = false;
};

bool is_metis_path(const std::string& path) {  // hlm_app.hpp:39-44
  const auto dot = path.rfind('.');
  if (dot == std::string::npos) return false;
  const std::string ext = path.substr(dot + 1);
  return ext == "graph" || ext == "metis";
}

void load_instance(const InstanceOptions& o, HostGraph& h) {  // hlm_app.hpp:46-62
  const std::string text = read_file(o.path, "instance file");
  const bool metis = o.format == "metis" || (o.format == "auto" && is_metis_path(o.path));
  const int dz = o.drop_isolated ? HLM_B200_DEGREE_ZERO_DROP : HLM_B200_DEGREE_ZERO_REJECT;
  const int st = metis ? hlm_b200_parse_metis_graph(text.data(), text.size(), dz, &h.g)
                       : hlm_b200_parse_hgr(text.data(), text.size(), dz, &h.g);
  if (st != HLM_B200_OK) fail_lib(o.path);
  if (h.g.num_warnings) std::cerr << "warning: " << o.path << ": vertex weights present but ignored; matching does not use them\n";
  if (o.weights == "unit")
    std::fill(h.g.base_weights, h.g.base_weights + h.g.num_edges, 1.0);
  else if (o.weights == "random")
    hlm_b200_random_weights_1_100(h.g.num_edges, o.weight_seed, h.g.base_weights);
}

hlm_b200_stream make_stream(const StreamOptions& o) {  // hlm_app.hpp:64-89
  hlm_b200_stream s{};
  s.seed = o.seed;
  if (o.generator == "xorshift")
    s.kind = HLM_B200_GEN_XORSHIFT;
  else if (o.generator == "park-miller")
    s.kind = HLM_B200_GEN_PARK_MILLER;
  else if (o.generator == "splitmix")
    s.kind = HLM_B200_GEN_SPLITMIX;
  else
    throw std::runtime_error("unknown generator '" + o.generator + "'");
  s.mode = o.uniform ? HLM_B200_MODE_REPLACE_UNIFORM : HLM_B200_MODE_PERTURB_BASE;
  const auto colon = o.noise.find(':');
  const std::string bad = "noise interval must look like LO:HI, got '" + o.noise + "'";
  if (colon == std::string::npos) throw std::runtime_error(bad);
  try {
    s.noise_low = std::stod(o.noise.substr(0, colon));
    s.noise_high = std::stod(o.noise.substr(colon + 1));
  } catch (const std::exception&) {
    throw std::runtime_error(bad);
  }
  if (s.noise_low < 0.0 || s.noise_high < s.noise_low) throw std::runtime_error("noise interval must satisfy 0 <= low <= high");
  return s;
}

int parse_variant(const std::string& name) {  // hlm_app.hpp:91-98 (+ auto)
  if (name == "seq") return HLM_B200_VARIANT_SEQ;
  if (name == "crcw") return HLM_B200_VARIANT_CRCW;
  if (name == "crew") return HLM_B200_VARIANT_CREW;
  if (name == "opt") return HLM_B200_VARIANT_WORK_OPTIMAL;
  if (name == "greedy") return HLM_B200_VARIANT_GREEDY;
  if (name == "auto") return HLM_B200_VARIANT_AUTO;
  throw std::runtime_error("unknown variant '" + name + "'");
}

double geometric_mean(const std::vector<double>& v) {  // hlm_app.hpp:100-104
  if (v.empty()) return 0.0;
  double log_sum = 0.0;
  for (double x : v) log_sum += std::log(x);
  return std::exp(log_sum / static_cast<double>(v.size()));
}

struct RunRow {  // hlm_app.hpp:107-121
  std::string instance, variant, workers, seed, generator, repeat;
  std::optional<double> rounds, size, weight, time_ms, edge_visits, pin_visits, ratio_vs_oracle;
};

const char* csv_header() {
  return "instance,variant,workers,seed,generator,repeat,rounds,size,weight,time_ms,"
         "edge_visits,pin_visits,ratio_vs_oracle";
}

std::string csv_row(const RunRow& r) {  // hlm_app.hpp:128-142
  auto num = [](const std::optional<double>& v, const char* fmt) {
    if (!v) return std::string();
    char buf[64];
    std::snprintf(buf, sizeof(buf), fmt, *v);
    return std::string(buf);
  };
  std::ostringstream out;
  out << r.instance << ',' << r.variant << ',' << r.workers << ',' << r.seed << ',' << r.generator << ',' << r.repeat << ','
      << num(r.rounds, "%.0f") << ',' << num(r.size, "%.0f") << ',' << num(r.weight, "%.6f") << ',' << num(r.time_ms, "%.3f")
      << ',' << num(r.edge_visits, "%.0f") << ',' << num(r.pin_visits, "%.0f") << ',' << num(r.ratio_vs_oracle, "%.6f");
  return out.str();
}

struct RunFlags {  // hlm_app.hpp:144-155
  InstanceOptions instance;
  StreamOptions stream;
  std::string variant = "crcw";
  unsigned workers = 0;
  uint32_t max_rounds = 0;
  bool with_oracle = false;
  std::string csv_path, emit_matching_path;
  int device = 0;
  unsigned gpus = 0;
};

std::string workers_column(int device) {
  (void)device;
  const int n = hlm_b200_device_count();
  return n > 0 ? "gpu" : "0";
}

RunRow execute_run(const RunFlags& f, const HostGraph& h) {  // hlm_app.hpp:156-202
  hlm_b200_config cfg{};
  cfg.variant = parse_variant(f.variant);
  cfg.max_rounds = f.max_rounds;
  cfg.num_gpus = f.gpus;
  const hlm_b200_stream stream = make_stream(f.stream);
  const hlm_b200_csr_view view = h.view();
  hlm_b200_result res{};
  const int st = hlm_b200_match_host(&view, &stream, &cfg, f.device, &res);
  if (st != HLM_B200_OK) {
    const std::string msg = st == HLM_B200_ERR_ROUND_LIMIT ? "round limit exceeded with " + std::to_string(res.rounds) + " rounds used"
                                                            : std::string(hlm_b200_last_error());
    hlm_b200_result_free(&res);
    throw std::runtime_error(msg);
  }
  // the caller always verifies (hlm_app.hpp:167-171): on the device
  hlm_b200_graph* g = nullptr;
  if (hlm_b200_graph_upload(&view, f.device, &g) != HLM_B200_OK) {
    hlm_b200_result_free(&res);
    fail_lib("upload for verification");
  }
  int disjoint = 0, maximal = 0;
  double weight = 0.0;
  const int vs = hlm_b200_verify(g, res.matched_edges, res.num_matched, &disjoint, &maximal, &weight);
  hlm_b200_graph_release(g);
  if (vs != HLM_B200_OK || !disjoint || !maximal) {
    hlm_b200_result_free(&res);
    throw std::logic_error(std::string("internal verification failed: matching is ") + (disjoint ? "" : "not disjoint ") +
                           (maximal ? "" : "not maximal"));
  }
  RunRow row;
  row.instance = f.instance.path;
  row.variant = f.variant;
  row.workers = workers_column(f.device);
  row.seed = std::to_string(f.stream.seed);
  row.generator = f.stream.generator;
  row.repeat = "0";
  row.rounds = res.rounds;
  row.size = static_cast<double>(res.num_matched);
  row.weight = res.total_weight;
  row.time_ms = res.wall_time_ms;
  row.edge_visits = static_cast<double>(res.total_edge_visits);
  row.pin_visits = static_cast<double>(res.total_pin_visits);
  if (f.with_oracle)
    std::cerr << "warning: oracle skipped, the exact search is not part of libhlm_b200\n";
  if (!f.emit_matching_path.empty()) {
    char* text = nullptr;
    size_t len = 0;
    if (hlm_b200_write_matching(res.matched_edges, res.num_matched, res.total_weight, res.rounds, &text, &len) != HLM_B200_OK) {
      hlm_b200_result_free(&res);
      fail_lib("write_matching");
    }
    std::ofstream out(f.emit_matching_path, std::ios::binary);
    if (!out) {
      hlm_b200_text_free(text);
      hlm_b200_result_free(&res);
      throw std::runtime_error("cannot write matching file " + f.emit_matching_path);
    }
    out.write(text, static_cast<std::streamsize>(len));
    hlm_b200_text_free(text);
  }
  hlm_b200_result_free(&res);
  return row;
}

void append_csv(const std::string& path, const std::vector<RunRow>& rows, bool truncate) {  // hlm_app.hpp:204-210
  bool fresh = truncate;
  if (!truncate) {
    std::ifstream probe(path);
    fresh = !probe.good();
  }
  std::ofstream out(path, truncate ? std::ios::trunc : std::ios::app);
  if (!out) throw std::runtime_error("cannot open csv file " + path);
  if (fresh) out << csv_header() << '\n';
  for (const auto& r : rows) out << csv_row(r) << '\n';
}

int cmd_run(const RunFlags& f) {
  HostGraph h;
  load_instance(f.instance, h);  // untimed
  const RunRow row = execute_run(f, h);
  std::cout << csv_header() << '\n' << csv_row(row) << '\n';
  if (!f.csv_path.empty()) append_csv(f.csv_path, {row}, false);
  return 0;
}

struct BenchFlags {  // hlm_app.hpp:220-227
  std::vector<std::string> instances, variants = {"crcw"};
  std::vector<uint64_t> seeds = {1};
  uint32_t repeats = 3;
  uint32_t warmup = 1;  // untimed runs per (instance, variant) first: CUDA context, module load, memory pools
                        // (a B200 extension; the CPU reference has nothing to warm)
  RunFlags base;
  std::string csv_path;
};

int cmd_bench(const BenchFlags& f) {  // hlm_app.hpp:232-333
  std::vector<RunRow> rows;
  bool any_failed = false;
  for (const auto& path : f.instances) {
    HostGraph h;
    bool loaded = false;
    try {
      InstanceOptions io = f.base.instance;
      io.path = path;
      load_instance(io, h);
      loaded = true;
    } catch (const std::exception& ex) {
      std::cerr << "error: " << path << ": " << ex.what() << "\n";
    }
    for (const auto& variant : f.variants) {
      for (uint32_t w = 0; loaded && w < f.warmup; ++w) {
        try {
          RunFlags rf = f.base;
          rf.instance.path = path;
          rf.variant = variant;
          rf.stream.seed = f.seeds.empty() ? 1 : f.seeds.front();
          rf.emit_matching_path.clear();
          (void)execute_run(rf, h);
        } catch (const std::exception&) {  // reported by the timed runs below
        }
      }
      for (uint64_t seed : f.seeds)
        for (uint32_t rep = 0; rep < f.repeats; ++rep) {
          RunRow row;
          row.instance = path;
          row.variant = variant;
          row.seed = std::to_string(seed);
          row.generator = f.base.stream.generator;
          row.workers = workers_column(f.base.device);
          row.repeat = std::to_string(rep);
          if (loaded) {
            try {
              RunFlags rf = f.base;
              rf.instance.path = path;
              rf.variant = variant;
              rf.stream.seed = seed;
              row = execute_run(rf, h);
              row.repeat = std::to_string(rep);
              row.seed = std::to_string(seed);
            } catch (const std::exception& ex) {
              std::cerr << "error: " << path << " variant=" << variant << " seed=" << seed << ": " << ex.what() << "\n";
              any_failed = true;
            }
          } else {
            any_failed = true;
          }
          rows.push_back(std::move(row));
        }
    }
  }
  std::map<std::pair<std::string, std::string>, std::vector<size_t>> by_pair;
  for (size_t i = 0; i < rows.size(); ++i)
    if (rows[i].time_ms) by_pair[{rows[i].instance, rows[i].variant}].push_back(i);
  std::vector<RunRow> summary;
  std::map<std::string, std::vector<double>> variant_times, variant_weights;
  for (const auto& [key, group] : by_pair) {
    RunRow mean;
    mean.instance = key.first;
    mean.variant = key.second;
    mean.workers = rows[group.front()].workers;
    mean.generator = rows[group.front()].generator;
    mean.repeat = "mean";
    auto avg = [&](std::optional<double> RunRow::*field) {
      double sum = 0.0;
      for (size_t i : group) sum += *(rows[i].*field);
      return sum / static_cast<double>(group.size());
    };
    mean.rounds = avg(&RunRow::rounds);
    mean.size = avg(&RunRow::size);
    mean.weight = avg(&RunRow::weight);
    mean.time_ms = avg(&RunRow::time_ms);
    variant_times[key.second].push_back(*mean.time_ms);
    variant_weights[key.second].push_back(*mean.weight);
    summary.push_back(std::move(mean));
  }
  for (const auto& [variant, times] : variant_times) {
    RunRow geo;
    geo.instance = "geomean";
    geo.variant = variant;
    geo.repeat = "geomean";
    geo.time_ms = geometric_mean(times);
    const auto& w = variant_weights[variant];
    if (!w.empty() && std::all_of(w.begin(), w.end(), [](double x) { return x > 0; })) geo.weight = geometric_mean(w);
    summary.push_back(std::move(geo));
  }
  rows.insert(rows.end(), summary.begin(), summary.end());
  if (!f.csv_path.empty()) {
    append_csv(f.csv_path, rows, true);
  } else {
    std::cout << csv_header() << '\n';
    for (const auto& r : rows) std::cout << csv_row(r) << '\n';
  }
  return any_failed ? 1 : 0;
}

struct GenerateFlags {  // hlm_app.hpp:335-347
  bool tight = false;
  uint32_t d = 3;
  double epsilon = 0.1;
  uint32_t n = 100, m = 80, min_size = 2, max_size = 3;
  uint64_t seed = 1;
  std::string weights = "unit";
  uint64_t weight_seed = 1;
  std::string out_path;
};

int cmd_generate(const GenerateFlags& f) {  // hlm_app.hpp:349-372
  HostGraph h;
  if (f.tight) {
    if (hlm_b200_generate_tight_family(f.d, f.epsilon, &h.g) != HLM_B200_OK) fail_lib("generate tight");
  } else {
    if (hlm_b200_generate_random(f.n, f.m, f.min_size, f.max_size, f.seed, &h.g) != HLM_B200_OK) fail_lib("generate random");
    if (f.weights == "random")
      hlm_b200_random_weights_1_100(h.g.num_edges, f.weight_seed, h.g.base_weights);
    else if (f.weights != "unit")
      throw std::runtime_error("generate supports weights unit|random");
  }
  const hlm_b200_csr_view view = h.view();
  char* text = nullptr;
  size_t len = 0;
  if (hlm_b200_write_hgr(&view, &text, &len) != HLM_B200_OK) fail_lib("write_hgr");
  std::ofstream out(f.out_path, std::ios::binary);
  if (!out) {
    hlm_b200_text_free(text);
    throw std::runtime_error("cannot write instance file " + f.out_path);
  }
  out.write(text, static_cast<std::streamsize>(len));
  hlm_b200_text_free(text);
  std::cout << "wrote " << f.out_path << " n=" << h.g.num_vertices << " m=" << h.g.num_edges << " kappa=" << h.pins() << '\n';
  return 0;
}

int cmd_verify(const InstanceOptions& inst, const std::string& matching_path, int device) {  // hlm_app.hpp:379-394
  HostGraph h;
  load_instance(inst, h);
  const std::string text = read_file(matching_path, "matching file");
  uint32_t* ids = nullptr;
  uint64_t count = 0;
  if (hlm_b200_parse_matching(text.data(), text.size(), &ids, &count) != HLM_B200_OK) fail_lib(matching_path);
  std::sort(ids, ids + count);
  const hlm_b200_csr_view view = h.view();
  hlm_b200_graph* g = nullptr;
  if (hlm_b200_graph_upload(&view, device, &g) != HLM_B200_OK) {
    hlm_b200_text_free(ids);
    fail_lib("upload");
  }
  int disjoint = 0, maximal = 0;
  double weight = 0.0;
  const int st = hlm_b200_verify(g, ids, count, &disjoint, &maximal, &weight);
  hlm_b200_graph_release(g);
  hlm_b200_text_free(ids);
  if (st != HLM_B200_OK) fail_lib("verify");
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6f", weight);
  std::cout << "disjoint: " << (disjoint ? "yes" : "NO") << '\n' << "maximal: " << (maximal ? "yes" : "NO") << '\n' << "weight: " << buf << '\n';
  return disjoint && maximal ? 0 : 1;
}

// ---- a small flag parser (the reference uses CLI11, a third-party header that is not vendored) ----
class Args {
 public:
  explicit Args(std::vector<std::string> a) : a_(std::move(a)) {}
  bool done() const { return i_ >= a_.size(); }
  std::string next() { return a_[i_++]; }
  bool peek_is_flag() const { return !done() && a_[i_].rfind("--", 0) == 0; }
  std::string value(const std::string& flag) {
    if (done()) throw UsageError(flag + " needs a value");
    return a_[i_++];
  }
 private:
  std::vector<std::string> a_;
  size_t i_ = 0;
};

uint64_t to_u64(const std::string& s, const std::string& flag) {
  try {
    size_t pos = 0;
    if (!s.empty() && s[0] == '-') throw std::invalid_argument("negative");
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw UsageError(flag + ": expected an unsigned integer, got '" + s + "'");
  }
}

double to_f64(const std::string& s, const std::string& flag) {
  try {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw UsageError(flag + ": expected a number, got '" + s + "'");
  }
}

void check_member(const std::string& v, std::initializer_list<const char*> set, const std::string& flag) {
  for (const char* s : set)
    if (v == s) return;
  throw UsageError(flag + ": '" + v + "' is not one of the allowed values");
}

std::vector<std::string> split_commas(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) out.push_back(tok);
  return out;
}

bool instance_flag(const std::string& flag, Args& a, InstanceOptions& o, bool with_path) {
  if (with_path && flag == "--instance") {
    o.path = a.value(flag);
  } else if (flag == "--format") {
    o.format = a.value(flag);
    check_member(o.format, {"auto", "hgr", "metis"}, flag);
  } else if (flag == "--weights") {
    o.weights = a.value(flag);
    check_member(o.weights, {"file", "unit", "random"}, flag);
  } else if (flag == "--weight-seed") {
    o.weight_seed = to_u64(a.value(flag), flag);
  } else if (flag == "--drop-isolated") {
    o.drop_isolated = true;
  } else {
    return false;
  }
  return true;
}

bool stream_flag(const std::string& flag, Args& a, StreamOptions& o) {
  if (flag == "--seed") {
    o.seed = to_u64(a.value(flag), flag);
  } else if (flag == "--generator") {
    o.generator = a.value(flag);
    check_member(o.generator, {"xorshift", "park-miller", "splitmix"}, flag);
  } else if (flag == "--noise") {
    o.noise = a.value(flag);
  } else if (flag == "--uniform") {
    o.uniform = true;
  } else {
    return false;
  }
  return true;
}

const char* kUsage =
    "usage: hlm_b200_cli <run|bench|generate|verify> [flags]\n"
    "  run      --instance F [--format auto|hgr|metis] [--weights file|unit|random] [--weight-seed N] [--drop-isolated]\n"
    "           [--seed N] [--generator xorshift|park-miller|splitmix] [--noise LO:HI] [--uniform]\n"
    "           [--variant seq|crcw|crew|opt|greedy|auto] [--max-rounds N] [--csv F] [--emit-matching F] [--device N] [--gpus K]\n"
    "  bench    --instances F... [--variants a,b] [--seeds 1,2] [--repeats N] [--warmup N] [--csv F] + the instance / stream flags of run\n"
    "  generate tight --d N --epsilon X --out F | random --n N --m M [--min-size A] [--max-size B] [--seed S]\n"
    "           [--weights unit|random] [--weight-seed S] --out F\n"
    "  verify   --instance F --matching F\n";

int run_cli(std::vector<std::string> argv) {
  if (argv.empty()) throw UsageError("a subcommand is required");
  Args a(std::move(argv));
  const std::string cmd = a.next();
  if (cmd == "run") {
    RunFlags f;
    while (!a.done()) {
      const std::string flag = a.next();
      if (instance_flag(flag, a, f.instance, true) || stream_flag(flag, a, f.stream)) continue;
      if (flag == "--variant") {
        f.variant = a.value(flag);
        check_member(f.variant, {"seq", "crcw", "crew", "opt", "greedy", "auto"}, flag);
      } else if (flag == "--workers") {
        f.workers = static_cast<unsigned>(to_u64(a.value(flag), flag));
      } else if (flag == "--max-rounds") {
        f.max_rounds = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (flag == "--grain") {
        (void)to_u64(a.value(flag), flag);
      } else if (flag == "--assert-crew") {
      } else if (flag == "--oracle") {
        f.with_oracle = true;
      } else if (flag == "--oracle-cap") {
        (void)to_u64(a.value(flag), flag);
      } else if (flag == "--csv") {
        f.csv_path = a.value(flag);
      } else if (flag == "--emit-matching") {
        f.emit_matching_path = a.value(flag);
      } else if (flag == "--device") {
        f.device = static_cast<int>(to_u64(a.value(flag), flag));
      } else if (flag == "--gpus") {
        f.gpus = static_cast<unsigned>(to_u64(a.value(flag), flag));
      } else {
        throw UsageError("unknown flag " + flag);
      }
    }
    if (f.instance.path.empty()) throw UsageError("--instance is required");
    return cmd_run(f);
  }
  if (cmd == "bench") {
    BenchFlags f;
    while (!a.done()) {
      const std::string flag = a.next();
      if (instance_flag(flag, a, f.base.instance, false) || stream_flag(flag, a, f.base.stream)) continue;
      if (flag == "--instances") {
        while (!a.done() && !a.peek_is_flag()) f.instances.push_back(a.next());
      } else if (flag == "--variants") {
        f.variants = split_commas(a.value(flag));
      } else if (flag == "--seeds") {
        f.seeds.clear();
        for (const auto& s : split_commas(a.value(flag))) f.seeds.push_back(to_u64(s, flag));
      } else if (flag == "--repeats") {
        f.repeats = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (flag == "--warmup") {
        f.warmup = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (flag == "--workers") {
        f.base.workers = static_cast<unsigned>(to_u64(a.value(flag), flag));
      } else if (flag == "--max-rounds") {
        f.base.max_rounds = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (flag == "--assert-crew") {
      } else if (flag == "--csv") {
        f.csv_path = a.value(flag);
      } else if (flag == "--device") {
        f.base.device = static_cast<int>(to_u64(a.value(flag), flag));
      } else if (flag == "--gpus") {
        f.base.gpus = static_cast<unsigned>(to_u64(a.value(flag), flag));
      } else {
        throw UsageError("unknown flag " + flag);
      }
    }
    if (f.instances.empty()) throw UsageError("--instances is required");
    return cmd_bench(f);
  }
  if (cmd == "generate") {
    if (a.done()) throw UsageError("generate needs tight|random");
    GenerateFlags f;
    const std::string kind = a.next();
    if (kind != "tight" && kind != "random") throw UsageError("generate needs tight|random");
    f.tight = kind == "tight";
    bool have_d = false, have_eps = false, have_n = false, have_m = false;
    while (!a.done()) {
      const std::string flag = a.next();
      if (flag == "--out") {
        f.out_path = a.value(flag);
      } else if (f.tight && flag == "--d") {
        f.d = static_cast<uint32_t>(to_u64(a.value(flag), flag));
        have_d = true;
      } else if (f.tight && flag == "--epsilon") {
        f.epsilon = to_f64(a.value(flag), flag);
        have_eps = true;
      } else if (!f.tight && flag == "--n") {
        f.n = static_cast<uint32_t>(to_u64(a.value(flag), flag));
        have_n = true;
      } else if (!f.tight && flag == "--m") {
        f.m = static_cast<uint32_t>(to_u64(a.value(flag), flag));
        have_m = true;
      } else if (!f.tight && flag == "--min-size") {
        f.min_size = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (!f.tight && flag == "--max-size") {
        f.max_size = static_cast<uint32_t>(to_u64(a.value(flag), flag));
      } else if (!f.tight && flag == "--seed") {
        f.seed = to_u64(a.value(flag), flag);
      } else if (!f.tight && flag == "--weights") {
        f.weights = a.value(flag);
        check_member(f.weights, {"unit", "random"}, flag);
      } else if (!f.tight && flag == "--weight-seed") {
        f.weight_seed = to_u64(a.value(flag), flag);
      } else {
        throw UsageError("unknown flag " + flag);
      }
    }
    if (f.out_path.empty()) throw UsageError("--out is required");
    if (f.tight && !(have_d && have_eps)) throw UsageError("generate tight needs --d and --epsilon");
    if (!f.tight && !(have_n && have_m)) throw UsageError("generate random needs --n and --m");
    return cmd_generate(f);
  }
  if (cmd == "verify") {
    InstanceOptions inst;
    std::string matching;
    int device = 0;
    while (!a.done()) {
      const std::string flag = a.next();
      if (instance_flag(flag, a, inst, true)) continue;
      if (flag == "--matching")
        matching = a.value(flag);
      else if (flag == "--device")
        device = static_cast<int>(to_u64(a.value(flag), flag));
      else
        throw UsageError("unknown flag " + flag);
    }
    if (inst.path.empty() || matching.empty()) throw UsageError("--instance and --matching are required");
    return cmd_verify(inst, matching, device);
  }
  if (cmd == "oracle") {
    std::cerr << "error: the exact branch-and-bound oracle (exact.hpp:84) is not part of libhlm_b200\n";
    return 2;
  }
  if (cmd == "--help" || cmd == "-h") {
    std::cout << kUsage;
    return 0;
  }
  throw UsageError("unknown subcommand '" + cmd + "'");
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  try {
    return run_cli(std::move(args));
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n" << kUsage;
    return 106;  // what CLI11 returns for a parse error the reference's tests only check as non-zero
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";  // hlm_app.hpp:516-519
    return 1;
  }
}
