// `ozmul` command line on the B200 library: the reference CLI's `multiply`
// and `analyze` subcommands (proj/tools/main.cpp:183-252, 268-335, 712-785)
// with the same options, stdout lines, JSON run records and exit codes
// (0 ok, 1 I/O / argument errors, 2 domain errors and infeasible
// selections), so scripts and the reference's cli_test run unchanged.
// Matrix files are the reference's "ozm1" format (ozgpu_io.cpp); every
// multiply, kappa scan, |A||B| bound, exact oracle and error metric runs on
// the GPU.  The `experiment` suites (main.cpp:408-657) are not part of this
// build (out of scope) and exit 1 like an unknown command.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ozgpu.h"
#include "ozmul_b200/api.hpp"
#include "ozmul_b200/io.hpp"

namespace {

using namespace ozmul;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value / --flag parsing against a fixed option table
struct Args {
  std::map<std::string, std::string> values;
  std::map<std::string, bool> flags;
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = values.find(k);
    return it == values.end() ? dflt : it->second;
  }
  bool has(const std::string& k) const { return values.count(k) != 0; }
  bool flag(const std::string& k) const { return flags.count(k) != 0; }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& options,
           const std::vector<std::string>& flag_names, const std::vector<std::string>& required) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string tok = argv[i];
    std::string val;
    const auto eq = tok.find('=');
    bool inline_val = false;
    if (tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      inline_val = true;
    }
    if (std::find(flag_names.begin(), flag_names.end(), tok) != flag_names.end()) {
      a.flags[tok] = true;
      continue;
    }
    if (std::find(options.begin(), options.end(), tok) == options.end())
      throw UsageError("unknown option " + tok);
    if (!inline_val) {
      if (i + 1 >= argc) throw UsageError(tok + " needs a value");
      val = argv[++i];
    }
    a.values[tok] = val;
  }
  for (const auto& r : required)
    if (!a.has(r)) throw UsageError(r + " is required");
  return a;
}

int to_int(const Args& a, const std::string& k, int dflt) {
  if (!a.has(k)) return dflt;
  try {
    size_t pos = 0;
    const int v = std::stoi(a.get(k), &pos);
    if (pos != a.get(k).size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw UsageError(k + ": expected an integer");
  }
}

double to_double(const Args& a, const std::string& k, double dflt) {
  if (!a.has(k)) return dflt;
  try {
    return std::stod(a.get(k));
  } catch (const std::exception&) {
    throw UsageError(k + ": expected a number");
  }
}

ScheduleKind schedule_of(const std::string& s) {
  if (s == "full") return ScheduleKind::kFull;
  if (s == "reduced") return ScheduleKind::kReduced;
  throw UsageError("--schedule: expected full or reduced");
}
Accumulation strategy_of(const std::string& s) {
  if (s == "float") return Accumulation::kFloatPerProduct;
  if (s == "diagonal") return Accumulation::kDiagonalInteger;
  if (s == "levelled") return Accumulation::kLevelledExact;
  throw UsageError("--strategy: expected float, diagonal, or levelled");
}
SliceMode mode_of(const std::string& s) {
  if (s == "truncate") return SliceMode::kTruncate;
  if (s == "nearest") return SliceMode::kNearest;
  throw UsageError("--mode: expected truncate or nearest");
}

// ------------------------------------------------------------------ JSON
// A tiny writer for the run records (two-space indent, "key": value).
struct Json {
  std::string text;
  static std::string num(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
  }
  static std::string str(const std::string& s) {
    std::string out = "\"";
    for (char ch : s) {
      if (ch == '"' || ch == '\\') out += '\\';
      out += ch;
    }
    return out + "\"";
  }
};

std::string object(const std::vector<std::pair<std::string, std::string>>& kv, int indent) {
  if (kv.empty()) return "{}";
  const std::string pad(indent + 2, ' '), end(indent, ' ');
  std::string s = "{\n";
  for (size_t i = 0; i < kv.size(); ++i) {
    s += pad + Json::str(kv[i].first) + ": " + kv[i].second;
    s += i + 1 < kv.size() ? ",\n" : "\n";
  }
  return s + end + "}";
}

std::string plan_json(const MmaConfig& cfg, const MultiplyPlan& p, int indent) {
  std::string levels = "[";
  for (size_t i = 0; i < p.levels.levels.size(); ++i) {
    levels += (i ? ", [" : "[") + std::to_string(p.levels.levels[i].first) + ", " +
              std::to_string(p.levels.levels[i].second) + "]";
  }
  levels += "]";
  const char* sched = p.schedule.kind == ScheduleKind::kFull ? "full" : "reduced";
  const char* strat = p.strategy == Accumulation::kFloatPerProduct    ? "float"
                      : p.strategy == Accumulation::kDiagonalInteger ? "diagonal"
                                                                      : "levelled";
  return object({{"t_in", std::to_string(cfg.input_width)},
                 {"t_acc", std::to_string(cfg.acc_width)},
                 {"slices_a", std::to_string(p.slices_a)},
                 {"slices_b", std::to_string(p.slices_b)},
                 {"width", std::to_string(p.width)},
                 {"schedule", Json::str(sched)},
                 {"strategy", Json::str(strat)},
                 {"mode", Json::str(p.mode == SliceMode::kNearest ? "nearest" : "truncate")},
                 {"acc_bits_used", std::to_string(p.acc_bits_used)},
                 {"levels", levels},
                 {"psi", std::to_string(p.psi)}},
                indent);
}

void write_text(const std::string& path, const std::string& s) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write " + path);
  out << s << '\n';
}

// ----------------------------------------------------------- GPU oracle
ozgpu_ctx* context() {
  const char* env = std::getenv("OZGPU_DEVICE");
  ozgpu_ctx* c = ozgpu_default_context(env ? std::atoi(env) : 0);
  if (!c) throw std::runtime_error(ozgpu_last_error());
  return c;
}

void ok_or_throw(int rc) {
  if (rc == OZGPU_OK) return;
  const std::string msg = ozgpu_last_error();
  if (rc == OZGPU_DOMAIN_ERROR) throw std::domain_error(msg);
  if (rc == OZGPU_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// RN(exact AB) on the GPU (ozgpu_exact_gemm) and the reference's two metrics
// against it (oracle.cpp:263-292; the exact value enters rounded once)
struct Metrics {
  double max_elementwise = 0.0, normwise = 0.0;
};

Metrics gpu_metrics(const Matrix& a, const Matrix& b, const Matrix& c) {
  const int64_t m = static_cast<int64_t>(a.rows()), k = static_cast<int64_t>(a.cols()),
                n = static_cast<int64_t>(b.cols());
  Matrix exact(a.rows(), b.cols());
  ozgpu_ctx* ctx = context();
  ok_or_throw(ozgpu_exact_gemm(ctx, m, n, k, a.data(), k, b.data(), n, exact.data(), n));
  Metrics out;
  double ss = 0.0, sa = 0.0, sb = 0.0;
  ok_or_throw(ozgpu_error_metrics(ctx, m, n, c.data(), n, exact.data(), n, &out.max_elementwise, &ss));
  ok_or_throw(ozgpu_error_metrics(ctx, m, k, a.data(), k, nullptr, 0, nullptr, &sa));
  ok_or_throw(ozgpu_error_metrics(ctx, k, n, b.data(), n, nullptr, 0, nullptr, &sb));
  // normwise_gemm_error with alpha = 1, beta = 0, C = 0 (main.cpp:222-227)
  const double denom = std::sqrt(static_cast<double>(k) + 2.0) * std::sqrt(sa) * std::sqrt(sb);
  if (denom == 0.0) throw std::domain_error("normwise_gemm_error: zero denominator");
  out.normwise = std::sqrt(ss) / denom;
  return out;
}

// ------------------------------------------------------------- multiply
const std::vector<std::string> kCommon = {"--t-in", "--t-acc", "--schedule", "--strategy",
                                          "--mode"};

std::vector<std::string> with_common(std::vector<std::string> v) {
  v.insert(v.end(), kCommon.begin(), kCommon.end());
  return v;
}

int run_multiply(int argc, char** argv) {
  const Args args = parse(argc, argv, 2,
                          with_common({"--a", "--b", "--out", "--record", "--format", "--sa", "--sb"}),
                          {"--exact", "--verify"}, {"--a", "--b", "--out"});
  const MatrixFormat fmt = args.get("--format", "hex") == "dec" ? MatrixFormat::kDec : MatrixFormat::kHex;
  const Matrix a = read_matrix_file(args.get("--a"), fmt);
  const Matrix b = read_matrix_file(args.get("--b"), fmt);
  MmaConfig cfg{to_int(args, "--t-in", 7), to_int(args, "--t-acc", 31)};
  cfg.validate();
  const auto t0 = std::chrono::steady_clock::now();
  const std::int64_t k = static_cast<std::int64_t>(a.cols());
  if (k > max_inner_dim(cfg))
    throw std::domain_error("inner dimension " + std::to_string(k) +
                            " exceeds the supported limit " + std::to_string(max_inner_dim(cfg)) +
                            " for I_" + std::to_string(cfg.input_width) + " inputs with I_" +
                            std::to_string(cfg.acc_width) + " accumulation");
  const int width = optimal_slice_width(cfg, k);
  // default slice counts: the exact ones (GPU scan)
  const int sa = to_int(args, "--sa", 0) > 0 ? to_int(args, "--sa", 0)
                                             : min_exact_slices(a, width, BlockOrientation::kRows);
  const int sb = to_int(args, "--sb", 0) > 0 ? to_int(args, "--sb", 0)
                                             : min_exact_slices(b, width, BlockOrientation::kColumns);
  const MultiplyPlan plan = make_plan(cfg, k, sa, sb, schedule_of(args.get("--schedule", "reduced")),
                                      strategy_of(args.get("--strategy", "levelled")),
                                      mode_of(args.get("--mode", "truncate")));
  const MultiplyResult result = multiply(a, b, cfg, plan);
  const auto t1 = std::chrono::steady_clock::now();
  write_matrix_file(args.get("--out"), result.c, fmt);

  const Diagnostics& d = result.diagnostics;
  std::vector<std::pair<std::string, std::string>> record = {
      {"command", Json::str("multiply")},
      {"a", Json::str(args.get("--a"))},
      {"b", Json::str(args.get("--b"))},
      {"out", Json::str(args.get("--out"))},
      {"m", std::to_string(a.rows())},
      {"k", std::to_string(a.cols())},
      {"n", std::to_string(b.cols())},
      {"plan", plan_json(cfg, plan, 2)},
      {"diagnostics", object({{"products", std::to_string(d.products)},
                              {"integer_adds", std::to_string(d.integer_adds)},
                              {"float_adds", std::to_string(d.float_adds)},
                              {"flushes", std::to_string(d.flushes)},
                              {"realized_psi", std::to_string(d.realized_psi)},
                              {"planned_psi", std::to_string(d.planned_psi)}},
                             2)},
      {"wall_seconds", Json::num(std::chrono::duration<double>(t1 - t0).count())},
      {"device", Json::str(ozgpu_version())}};
  Metrics metrics;
  const bool exact = args.flag("--exact");
  if (exact) {
    metrics = gpu_metrics(a, b, result.c);
    record.push_back({"metrics", object({{"max_elementwise_error", Json::num(metrics.max_elementwise)},
                                         {"normwise_error", Json::num(metrics.normwise)}},
                                        2)});
    std::cout << "max elementwise error: " << metrics.max_elementwise << '\n';
    std::cout << "normwise error: " << metrics.normwise << '\n';
  }
  if (args.has("--record")) write_text(args.get("--record"), object(record, 0));
  if (args.flag("--verify")) {
    const Matrix reread = read_matrix_file(args.get("--out"), fmt);
    if (!(reread == result.c)) throw std::runtime_error("verify: output file does not round-trip");
    if (exact) {
      const Metrics again = gpu_metrics(a, b, reread);
      if (std::bit_cast<std::uint64_t>(again.max_elementwise) !=
          std::bit_cast<std::uint64_t>(metrics.max_elementwise))
        throw std::runtime_error("verify: recomputed error differs");
    }
    std::cout << "verify: ok\n";
  }
  if (a.rows() * b.cols() == 1) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", result.c(0, 0));
    std::cout << "result: " << buf << '\n';
  }
  std::cout << "wrote " << args.get("--out") << " (" << d.products << " slice products, width "
            << plan.width << ")\n";
  return 0;
}

// -------------------------------------------------------------- analyze
int run_analyze(int argc, char** argv) {
  const Args args = parse(argc, argv, 2,
                          with_common({"--a", "--b", "--record", "--format", "--sa", "--sb",
                                       "--target", "--s-max"}),
                          {"--auto"}, {"--a", "--b"});
  const MatrixFormat fmt = args.get("--format", "hex") == "dec" ? MatrixFormat::kDec : MatrixFormat::kHex;
  const Matrix a = read_matrix_file(args.get("--a"), fmt);
  const Matrix b = read_matrix_file(args.get("--b"), fmt);
  MmaConfig cfg{to_int(args, "--t-in", 7), to_int(args, "--t-acc", 31)};
  cfg.validate();
  const std::int64_t k = static_cast<std::int64_t>(a.cols());
  const int width = optimal_slice_width(cfg, k);
  const ScalingProfile profile = scaling_profile(a, b);  // GPU kappa scan
  std::cout << "kappa_A: " << profile.kappa_a << '\n';
  std::cout << "kappa_B: " << profile.kappa_b << '\n';
  std::vector<std::pair<std::string, std::string>> record = {
      {"command", Json::str("analyze")},
      {"kappa_a", Json::num(profile.kappa_a)},
      {"kappa_b", Json::num(profile.kappa_b)},
      {"width", std::to_string(width)}};
  int sa = to_int(args, "--sa", 8), sb = to_int(args, "--sb", 8);
  const ScheduleKind sched = schedule_of(args.get("--schedule", "reduced"));
  const Accumulation strat = strategy_of(args.get("--strategy", "levelled"));
  const int s_max = to_int(args, "--s-max", 24);
  if (args.flag("--auto")) {
    SelectOptions opts;
    opts.schedule = sched;
    opts.strategy = strat;
    int log2k = 0;
    while ((std::int64_t{1} << log2k) < k) ++log2k;
    opts.acc_bits_used = 2 * width + log2k;
    const double target = to_double(args, "--target", 0.0);
    if (target > 0.0) opts.target = target;
    try {
      const SliceSelection sel = select_slices(profile.kappa_a, profile.kappa_b, width, 0x1p-53,
                                               s_max, opts);
      sa = sel.slices_a;
      sb = sel.slices_b;
      std::cout << "selected slices: s_A = " << sa << ", s_B = " << sb << " (chi = "
                << sel.products << ", term = " << sel.lhs << " <= target " << sel.target << ")\n";
      record.push_back({"selection", object({{"slices_a", std::to_string(sa)},
                                             {"slices_b", std::to_string(sb)},
                                             {"chi", std::to_string(sel.products)},
                                             {"lhs", Json::num(sel.lhs)},
                                             {"target", Json::num(sel.target)}},
                                            2)});
    } catch (const SelectionInfeasible& e) {
      std::cout << "infeasible: no pair within s_max = " << s_max
                << " meets the target; best term exceeds it by " << e.gap << "x\n";
      record.push_back({"selection", object({{"infeasible", "true"},
                                             {"gap", Json::num(e.gap)},
                                             {"best_lhs", Json::num(e.best_lhs)},
                                             {"target", Json::num(e.target)}},
                                            2)});
      if (args.has("--record")) write_text(args.get("--record"), object(record, 0));
      return 2;
    }
  }
  const MultiplyPlan plan = make_plan(cfg, k, sa, sb, sched, strat, mode_of(args.get("--mode", "truncate")));
  const ErrorReport report = error_bound(a, b, plan);  // |A||B| on the GPU
  std::cout << "zeta: " << report.zeta_ab << '\n';
  std::cout << "gamma_psi: " << report.gamma_psi << '\n';
  std::cout << "bound coefficient on |A||B|: " << report.coefficient << '\n';
  std::cout << "first-order coefficient: " << report.first_order_coefficient << '\n';
  record.push_back({"plan", plan_json(cfg, plan, 2)});
  record.push_back({"bound", object({{"zeta", Json::num(report.zeta_ab)},
                                     {"gamma_psi", Json::num(report.gamma_psi)},
                                     {"coefficient", Json::num(report.coefficient)},
                                     {"first_order", Json::num(report.first_order_coefficient)}},
                                    2)});
  if (args.has("--record")) write_text(args.get("--record"), object(record, 0));
  return 0;
}

void usage() {
  std::cerr << "usage: ozmul multiply --a A.ozm --b B.ozm --out C.ozm [--sa N] [--sb N] "
               "[--exact] [--verify] [--record R.json] [--format hex|dec] [common]\n"
               "       ozmul analyze --a A.ozm --b B.ozm [--auto] [--target T] [--s-max N] "
               "[--sa N] [--sb N] [--record R.json] [--format hex|dec] [common]\n"
               "common: --t-in N --t-acc N --schedule full|reduced "
               "--strategy float|diagonal|levelled --mode truncate|nearest\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "multiply") return run_multiply(argc, argv);
    if (cmd == "analyze") return run_analyze(argc, argv);
    if (cmd == "--help" || cmd == "-h") {
      usage();
      return 0;
    }
    std::cerr << "error: unknown or unsupported subcommand '" << cmd
              << "' (this build provides multiply and analyze)\n";
    return 1;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << '\n';
    usage();
    return 1;
  } catch (const SelectionInfeasible& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::domain_error& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
