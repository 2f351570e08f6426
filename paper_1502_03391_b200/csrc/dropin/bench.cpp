// The `bench` grid of the drop-in API (include/jofc/bench.hpp) after
// proj/src/bench.cpp: same grid file, seeds, shared start per cell and CSV;
// the fJOFC rows time the GPU transform (EmbeddingResult::step_seconds).  The
// dense JOFC comparison rows need jofc_embed_reference, which is not part of
// this build: they are skipped with a note on stderr.
#include "jofc/bench.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>

#include "jofc/init.hpp"
#include "jofc/simulate.hpp"
#include "jofc/solver.hpp"

namespace jofc {

namespace {

std::string strip(const std::string& s) {
  const size_t a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return {};
  return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

std::vector<std::size_t> sizes(const std::string& v) {
  std::vector<std::size_t> out;
  std::stringstream ss(v);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(static_cast<std::size_t>(std::stoull(strip(tok))));
  return out;
}

bool yes(const std::string& v) { return v == "true" || v == "1" || v == "yes"; }

BenchRow summary(std::size_t n, std::size_t m, const BenchOptions& o, std::vector<double> t) {
  BenchRow r{n, m, "fjofc", o.replicates, o.iterations};
  const std::size_t k = t.size();
  if (k == 0) return r;
  double mean = 0.0;
  for (double v : t) mean += v;
  mean /= static_cast<double>(k);
  double ss = 0.0;
  for (double v : t) ss += (v - mean) * (v - mean);
  std::sort(t.begin(), t.end());
  r.mean_step_seconds = mean;
  r.stderr_step_seconds =
      k > 1 ? std::sqrt(ss / static_cast<double>(k - 1)) / std::sqrt(static_cast<double>(k)) : 0.0;
  r.median_step_seconds = (k % 2) ? t[k / 2] : 0.5 * (t[k / 2 - 1] + t[k / 2]);
  r.min_step_seconds = t.front();
  return r;
}

}  // namespace

std::vector<BenchRow> run_bench(const BenchOptions& o) {
  if (o.run_reference)
    std::cerr << "note: dense JOFC rows (jofc_embed_reference) are not part of this build; "
                 "timing fJOFC only\n";
  std::vector<BenchRow> rows;
  const WeightSpec spec = WeightSpec::uniform(o.w);
  for (std::size_t n : o.n_list)
    for (std::size_t m : o.m_list) {
      std::vector<double> times;
      for (std::size_t rep = 0; rep < o.replicates; ++rep) {
        const OmnibusProblem problem = generate_matched(n, m, o.dim, o.seed + 977u * rep).problem();
        SolveOptions s;
        s.dim = o.d;
        s.eps = 1e-300;  // fixed budget
        s.max_iterations = o.iterations;
        s.parallel = o.parallel;
        s.dense_cap = o.dense_cap;
        s.init = InitKind::provided;
        s.init_config = (o.init == InitKind::imputed_cmds)
                            ? imputed_omnibus_init(problem, o.d, o.dense_cap)
                            : averaged_procrustes_init(problem, o.d, o.parallel);
        const EmbeddingResult r = fjofc_embed(problem, spec, s);
        times.insert(times.end(), r.step_seconds.begin(), r.step_seconds.end());
      }
      rows.push_back(summary(n, m, o, std::move(times)));
    }
  return rows;
}

void write_bench_csv(const std::string& path, const std::vector<BenchRow>& rows) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::invalid_argument("cannot open '" + path + "'");
  std::fprintf(f, "n,m,algorithm,replicates,iterations,mean_step_seconds,stderr_step_seconds,"
                  "median_step_seconds,min_step_seconds\n");
  for (const BenchRow& r : rows)
    std::fprintf(f, "%zu,%zu,%s,%zu,%zu,%.9e,%.9e,%.9e,%.9e\n", r.n, r.m, r.algorithm.c_str(),
                 r.replicates, r.iterations, r.mean_step_seconds, r.stderr_step_seconds,
                 r.median_step_seconds, r.min_step_seconds);
  std::fclose(f);
}

BenchOptions parse_bench_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::invalid_argument("cannot open '" + path + "'");
  BenchOptions o;
  std::string line;
  for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
    const std::string t = strip(line.substr(0, line.find('#')));
    if (t.empty()) continue;
    const size_t eq = t.find('=');
    const std::string at = "'" + path + "' line " + std::to_string(lineno);
    if (eq == std::string::npos) throw std::invalid_argument(at + ": expected key = value");
    const std::string key = strip(t.substr(0, eq)), v = strip(t.substr(eq + 1));
    if (key == "n_list") o.n_list = sizes(v);
    else if (key == "m_list") o.m_list = sizes(v);
    else if (key == "d") o.d = std::stoull(v);
    else if (key == "dim") o.dim = std::stoull(v);
    else if (key == "w") o.w = std::stod(v);
    else if (key == "replicates") o.replicates = std::stoull(v);
    else if (key == "iterations") o.iterations = std::stoull(v);
    else if (key == "seed") o.seed = std::stoull(v);
    else if (key == "init") o.init = (v == "averaged") ? InitKind::averaged_procrustes : InitKind::imputed_cmds;
    else if (key == "reference") o.run_reference = yes(v);
    else if (key == "parallel") o.parallel = yes(v);
    else if (key == "dense_cap") o.dense_cap = std::stoull(v);
    else throw std::invalid_argument(at + ": unknown key '" + key + "'");
  }
  return o;
}

}  // namespace jofc
