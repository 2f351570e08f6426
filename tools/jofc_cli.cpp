// jofc -- command-line front end on the B200 path.
//
// The reference's `jofc embed | oos | simulate | bench` (proj/tools/
// jofc_main.cpp:84-230) with the same options, outputs and exit codes
// (0 ok, 1 invalid input, 2 numerical failure), on a small hand-written
// argument parser (the reference's CLI11 is not vendored).  `embed` streams
// file inputs straight into HBM (jofc_load_problem_files) and builds
// generated problems on the device from their features
// (jofc_set_problem_features); the solve, the initialisers and the OOS
// updates are the GPU kernels.  Not part of this build: `eval` (k-means /
// ARI metrics) and the dense JOFC algorithm (`--algorithm jofc`).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "jofc/bench.hpp"
#include "jofc/io.hpp"
#include "jofc/linalg.hpp"
#include "jofc/oos.hpp"
#include "jofc/simulate.hpp"
#include "jofc/solver.hpp"
#include "jofc/stress.hpp"
#include "jofc_gpu.h"

namespace {

using namespace jofc;

// ------------------------------------------------------------ arguments
struct Spec {
  std::string name;
  bool flag = false;   // takes no value
  bool multi = false;  // takes one or more values
  bool required = false;
};

struct Args {
  std::map<std::string, std::vector<std::string>> values;
  bool has(const std::string& k) const { return values.count(k) != 0; }
  const std::string& one(const std::string& k) const { return values.at(k).front(); }
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

Args parse(int argc, char** argv, int first, const std::vector<Spec>& specs) {
  Args out;
  for (int i = first; i < argc; ++i) {
    std::string tok = argv[i], inline_value;
    bool has_inline = false;
    if (tok.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + tok + "'");
    const size_t eq = tok.find('=');
    if (eq != std::string::npos) {
      inline_value = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      has_inline = true;
    }
    const Spec* sp = nullptr;
    for (const Spec& s : specs)
      if ("--" + s.name == tok) sp = &s;
    if (!sp) throw UsageError("unknown option '" + tok + "'");
    std::vector<std::string>& v = out.values[sp->name];
    if (sp->flag) {
      if (has_inline) throw UsageError(tok + " takes no value");
      v.push_back("1");
      continue;
    }
    if (has_inline) {
      v.push_back(inline_value);
    } else {
      if (i + 1 >= argc) throw UsageError(tok + " needs a value");
      v.push_back(argv[++i]);
    }
    while (sp->multi && i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0) v.push_back(argv[++i]);
  }
  for (const Spec& s : specs)
    if (s.required && !out.has(s.name)) throw UsageError("--" + s.name + " is required");
  return out;
}

double num(const Args& a, const std::string& k, double dflt) {
  if (!a.has(k)) return dflt;
  size_t used = 0;
  const double v = std::stod(a.one(k), &used);
  if (used != a.one(k).size()) throw UsageError("--" + k + ": not a number");
  return v;
}

long long integer(const Args& a, const std::string& k, long long dflt) {
  if (!a.has(k)) return dflt;
  size_t used = 0;
  const long long v = std::stoll(a.one(k), &used);
  if (used != a.one(k).size()) throw UsageError("--" + k + ": not an integer");
  return v;
}

// ------------------------------------------------------------ device plumbing
struct Ctx {
  jofc_ctx* h = nullptr;
  Ctx() {
    if (jofc_ctx_create(0, &h) != 0) fail(JOFC_ECUDA);
  }
  ~Ctx() { jofc_ctx_destroy(h); }
  [[noreturn]] static void fail(int rc) {
    const std::string msg = jofc_last_error();
    if (rc == JOFC_ENUMERIC) throw NumericalError(msg);
    if (rc == JOFC_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  void check(int rc) const {
    if (rc != 0) fail(rc);
  }
};

struct CWeights {
  jofc_weights w{};
  std::vector<double> general, within;
  explicit CWeights(const WeightSpec& s) {
    if (s.kind() == WeightSpec::Kind::uniform) {
      w.kind = 0;
      w.w = s.uniform_w();
    } else if (s.kind() == WeightSpec::Kind::general_symmetric) {
      w.kind = 1;
      general.assign(s.general_matrix().data(), s.general_matrix().data() + s.general_matrix().size());
      w.general = general.data();
    } else {
      w.kind = 2;
      within = s.product_within();
      w.within = within.data();
      w.scale = s.fidelity_scale();
    }
  }
};

void write_trace(const std::string& path, const std::vector<double>& trace, double pairs,
                 const std::vector<double>& step_seconds) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::invalid_argument("cannot open '" + path + "'");
  std::fprintf(f, "iteration,stress,normalized_stress,step_seconds\n");
  for (size_t i = 0; i < trace.size(); ++i)
    std::fprintf(f, "%zu,%.17g,%.17g,%.9e\n", i, trace[i], trace[i] / pairs,
                 i == 0 ? 0.0 : step_seconds[i - 1]);
  std::fclose(f);
}

// ------------------------------------------------------------ commands
int run_embed(const Args& a) {
  RunConfig cfg = parse_run_config(a.one("config"));
  if (a.has("algorithm")) {
    const std::string alg = a.one("algorithm");
    if (alg != "fjofc" && alg != "jofc") throw UsageError("--algorithm: expected fjofc|jofc");
    cfg.algorithm = alg == "jofc" ? Algorithm::jofc_reference : Algorithm::fjofc;
  }
  if (num(a, "w", -1.0) > 0.0) cfg.weights = WeightSpec::uniform(num(a, "w", -1.0));
  if (integer(a, "d", -1) > 0) cfg.d = static_cast<size_t>(integer(a, "d", -1));
  if (num(a, "eps", -1.0) > 0.0) cfg.eps = num(a, "eps", -1.0);
  if (integer(a, "seed", -1) >= 0) cfg.seed = static_cast<uint64_t>(integer(a, "seed", -1));
  if (a.has("parallel")) cfg.parallel = true;
  if (a.has("out")) cfg.out = a.one("out");
  if (cfg.out.empty()) cfg.out = "embedding.csv";
  if (cfg.algorithm == Algorithm::jofc_reference)
    throw std::invalid_argument("algorithm jofc (the dense reference JOFC) is not part of this build");
  if (!cfg.init_explicit) cfg.init = InitKind::averaged_procrustes;

  Ctx c;
  if (!cfg.inputs.empty()) {
    std::vector<const char*> ps;
    for (const std::string& p : cfg.inputs) ps.push_back(p.c_str());
    c.check(jofc_load_problem_files(c.h, ps.size(), ps.data(), cfg.normalize ? 1 : 0));
  } else {
    const size_t anom = *cfg.generator == "matched" ? 0 : cfg.n_anom;
    const std::vector<DenseMatrix> f = simulate_features(cfg.n, cfg.m, anom, cfg.dim, cfg.seed);
    std::vector<double> flat;
    for (const DenseMatrix& b : f) flat.insert(flat.end(), b.data(), b.data() + b.size());
    c.check(jofc_set_problem_features(c.h, cfg.m, cfg.n, cfg.dim, flat.data()));
    if (cfg.normalize)
      throw std::invalid_argument("normalize with a generator: write the problem with "
                                  "`jofc simulate` and load it");
  }
  size_t m = 0, n = 0;
  c.check(jofc_problem_shape(c.h, &m, &n));
  const size_t d = cfg.d;
  cfg.weights.validate(m);
  if (!(cfg.eps > 0.0)) throw std::invalid_argument("SolveOptions: eps must be positive");
  const CWeights cw(cfg.weights);

  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double> x0(m * n * d), x(m * n * d), trace(cfg.max_iterations + 1),
      steps(cfg.max_iterations);
  if (cfg.init == InitKind::imputed_cmds)
    c.check(jofc_init_imputed_cmds(c.h, d, 4096, x0.data()));
  else
    c.check(jofc_init_averaged_procrustes(c.h, d, x0.data()));
  size_t its = 0;
  int conv = 0;
  c.check(jofc_fjofc_embed(c.h, &cw.w, d, x0.data(), cfg.eps, cfg.max_iterations, x.data(),
                           trace.data(), &its, &conv, steps.data()));
  const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  trace.resize(its + 1);
  steps.resize(its);

  Configuration out;
  for (size_t l = 0; l < m; ++l) {
    DenseMatrix b(n, d);
    std::copy(x.begin() + l * n * d, x.begin() + (l + 1) * n * d, b.data());
    out.blocks.push_back(std::move(b));
  }
  save_embedding(cfg.out, out);
  const double pairs = stress_pair_count(m, n);
  if (a.has("trace")) write_trace(a.one("trace"), trace, pairs, steps);
  const double mean_step =
      steps.empty() ? 0.0 : std::accumulate(steps.begin(), steps.end(), 0.0) / steps.size();
  std::printf("embedding: %s\n", cfg.out.c_str());
  std::printf("iterations: %zu (%s)\n", its, conv ? "converged" : "max_iterations");
  std::printf("final_stress: %.10g\n", trace.back());
  std::printf("final_normalized_stress: %.10g\n", trace.back() / pairs);
  std::printf("mean_step_seconds: %.6e\n", mean_step);
  std::printf("total_seconds: %.3f\n", total);
  return 0;
}

int run_oos(const Args& a) {
  const Configuration x = load_embedding(a.one("embedding"));
  OosDissimilarity deltas{load_delta_vectors(a.values.at("deltas"))};
  OosOptions opt;
  opt.eps = num(a, "eps", 1e-6);
  opt.max_iterations = static_cast<size_t>(integer(a, "max-iterations", 1000));
  const OosResult r = oos_embed(x, deltas, num(a, "w", 1.0), opt,
                                static_cast<uint64_t>(integer(a, "seed", 0)));
  const std::string out = a.has("out") ? a.one("out") : "";
  std::FILE* sink = out.empty() ? stdout : std::fopen(out.c_str(), "w");
  if (!sink) throw std::invalid_argument("cannot open '" + out + "'");
  for (size_t i = 0; i < r.y.rows(); ++i) {
    for (size_t j = 0; j < r.y.cols(); ++j) std::fprintf(sink, j ? ",%.17g" : "%.17g", r.y(i, j));
    std::fputc('\n', sink);
  }
  if (!out.empty()) std::fclose(sink);
  std::fprintf(stderr, "oos iterations: %zu (%s), final stress %.10g\n", r.iterations,
               r.terminated == Termination::converged ? "converged" : "max_iterations",
               r.stress_trace.back());
  return 0;
}

int run_simulate(const Args& a) {
  const std::string setting = a.one("setting");
  if (setting != "matched" && setting != "anomaly")
    throw UsageError("--setting: expected matched|anomaly");
  const size_t n = static_cast<size_t>(integer(a, "n", 400)), m = static_cast<size_t>(integer(a, "m", 3));
  const size_t dim = static_cast<size_t>(integer(a, "dim", 2));
  const size_t n_anom = static_cast<size_t>(integer(a, "n-anom", 10));
  const uint64_t seed = static_cast<uint64_t>(integer(a, "seed", 0));
  const std::string out = a.has("out") ? a.one("out") : "problem";
  const SimulatedProblem sim =
      setting == "matched" ? generate_matched(n, m, dim, seed) : generate_anomaly(n, m, n_anom, dim, seed);
  std::vector<std::string> written;
  const bool binary = out.size() > 5 && out.compare(out.size() - 5, 5, ".jofc") == 0;
  if (binary) {
    save_problem_binary(out, sim.problem());
    written.push_back(out);
  } else {
    for (size_t i = 0; i < sim.modalities.size(); ++i) {
      written.push_back(out + "_" + std::to_string(i + 1) + ".csv");
      save_csv_matrix(written.back(), sim.modalities[i]);
    }
  }
  const std::string lab = binary ? out + ".labels.csv" : out + "_labels.csv";
  save_labels(lab, sim.labels);
  written.push_back(lab);
  if (!sim.anomalies.empty()) {
    const std::string an = binary ? out + ".anomalies.csv" : out + "_anomalies.csv";
    save_indices(an, sim.anomalies);
    written.push_back(an);
  }
  for (const std::string& p : written) std::printf("wrote %s\n", p.c_str());
  return 0;
}

int run_bench_cmd(const Args& a) {
  const BenchOptions opt = parse_bench_config(a.one("grid"));
  const std::string out = a.has("out") ? a.one("out") : "bench.csv";
  const std::vector<BenchRow> rows = run_bench(opt);
  write_bench_csv(out, rows);
  std::printf("%6s %3s %-6s %14s %14s %14s\n", "n", "m", "algo", "mean_s", "stderr_s", "median_s");
  for (const BenchRow& r : rows)
    std::printf("%6zu %3zu %-6s %14.6e %14.6e %14.6e\n", r.n, r.m, r.algorithm.c_str(),
                r.mean_step_seconds, r.stderr_step_seconds, r.median_step_seconds);
  std::printf("wrote %s\n", out.c_str());
  return 0;
}

const char* kUsage =
    "usage: jofc <command> [options]\n"
    "  embed    --config FILE [--algorithm fjofc] [--w W] [--d D] [--eps E] [--seed S]\n"
    "           [--parallel] [--out PATH] [--trace PATH]\n"
    "  oos      --embedding PATH --deltas FILE... [--w W] [--eps E] [--max-iterations K]\n"
    "           [--seed S] [--out PATH]\n"
    "  simulate --setting matched|anomaly [--n N] [--m M] [--dim D] [--n-anom K] [--seed S]\n"
    "           [--out PREFIX|FILE.jofc]\n"
    "  bench    --grid FILE [--out PATH]\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
    std::fputs(kUsage, argc < 2 ? stderr : stdout);
    return argc < 2 ? 1 : 0;
  }
  const std::string cmd = argv[1];
  for (int i = 2; i < argc; ++i)
    if (!std::strcmp(argv[i], "--help")) {
      std::fputs(kUsage, stdout);
      return 0;
    }
  try {
    if (cmd == "embed")
      return run_embed(parse(argc, argv, 2,
                             {{"config", false, false, true}, {"algorithm"}, {"w"}, {"d"}, {"eps"},
                              {"seed"}, {"parallel", true}, {"out"}, {"trace"}}));
    if (cmd == "oos")
      return run_oos(parse(argc, argv, 2,
                           {{"embedding", false, false, true}, {"deltas", false, true, true}, {"w"},
                            {"eps"}, {"max-iterations"}, {"seed"}, {"out"}}));
    if (cmd == "simulate")
      return run_simulate(parse(argc, argv, 2,
                                {{"setting", false, false, true}, {"n"}, {"m"}, {"dim"}, {"n-anom"},
                                 {"seed"}, {"out"}}));
    if (cmd == "bench")
      return run_bench_cmd(parse(argc, argv, 2, {{"grid", false, false, true}, {"out"}}));
    if (cmd == "eval") {
      std::cerr << "error: eval (k-means / ARI metrics) is not part of this build\n";
      return 1;
    }
    throw UsageError("unknown command '" + cmd + "'");
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n" << kUsage;
    return 1;
  } catch (const NumericalError& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
