// The `bench` grid of the drop-in API (include/jofc/bench.hpp): the grid file,
// matched-setting problems, one shared start per cell and the CSV of the
// reference's `jofc bench` (proj/src/bench.cpp:18-174 is the contract), timing
// the GPU fJOFC loop (EmbeddingResult::step_seconds, the device's mean time
// per iteration).  The dense Algorithm-1 rows need jofc_embed_reference,
// which is not part of this build: they are skipped with a note on stderr.
#include "jofc/bench.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <numeric>
#include <sstream>
#include <stdexcept>

#include "jofc/init.hpp"
#include "jofc/simulate.hpp"
#include "jofc/solver.hpp"

namespace jofc {

namespace {

std::string trimmed(const std::string& s) {
  const auto first = s.find_first_not_of(" \t\r\n");
  const auto last = s.find_last_not_of(" \t\r\n");
  return first == std::string::npos ? std::string() : s.substr(first, last - first + 1);
}

std::vector<std::size_t> size_list(const std::string& text) {
  std::vector<std::size_t> out;
  std::istringstream in(text);
  for (std::string item; std::getline(in, item, ',');)
    out.push_back(static_cast<std::size_t>(std::stoull(trimmed(item))));
  return out;
}

bool truthy(const std::string& v) { return v == "true" || v == "1" || v == "yes"; }

// Sample statistics of one grid cell's per-iteration times.
struct CellStats {
  double mean = 0.0, std_error = 0.0, median = 0.0, minimum = 0.0;
  explicit CellStats(std::vector<double> t) {
    const std::size_t k = t.size();
    if (k == 0) return;
    mean = std::accumulate(t.begin(), t.end(), 0.0) / static_cast<double>(k);
    double dev2 = 0.0;
    for (double x : t) dev2 += (x - mean) * (x - mean);
    if (k > 1) std_error = std::sqrt(dev2 / static_cast<double>(k - 1) / static_cast<double>(k));
    std::sort(t.begin(), t.end());
    minimum = t.front();
    median = (k & 1) ? t[k / 2] : 0.5 * (t[k / 2 - 1] + t[k / 2]);
  }
};

using Setter = std::function<void(BenchOptions&, const std::string&)>;

const std::map<std::string, Setter>& grid_keys() {
  static const std::map<std::string, Setter> keys = {
      {"n_list", [](BenchOptions& o, const std::string& v) { o.n_list = size_list(v); }},
      {"m_list", [](BenchOptions& o, const std::string& v) { o.m_list = size_list(v); }},
      {"d", [](BenchOptions& o, const std::string& v) { o.d = std::stoull(v); }},
      {"dim", [](BenchOptions& o, const std::string& v) { o.dim = std::stoull(v); }},
      {"w", [](BenchOptions& o, const std::string& v) { o.w = std::stod(v); }},
      {"replicates", [](BenchOptions& o, const std::string& v) { o.replicates = std::stoull(v); }},
      {"iterations", [](BenchOptions& o, const std::string& v) { o.iterations = std::stoull(v); }},
      {"seed", [](BenchOptions& o, const std::string& v) { o.seed = std::stoull(v); }},
      {"init",
       [](BenchOptions& o, const std::string& v) {
         o.init = v == "averaged" ? InitKind::averaged_procrustes : InitKind::imputed_cmds;
       }},
      {"reference", [](BenchOptions& o, const std::string& v) { o.run_reference = truthy(v); }},
      {"parallel", [](BenchOptions& o, const std::string& v) { o.parallel = truthy(v); }},
      {"dense_cap", [](BenchOptions& o, const std::string& v) { o.dense_cap = std::stoull(v); }},
  };
  return keys;
}

}  // namespace

std::vector<BenchRow> run_bench(const BenchOptions& o) {
  if (o.run_reference)
    std::cerr << "note: dense JOFC rows (jofc_embed_reference) are not part of this build; "
                 "timing fJOFC only\n";
  const WeightSpec spec = WeightSpec::uniform(o.w);
  std::vector<BenchRow> rows;
  for (std::size_t n : o.n_list)
    for (std::size_t m : o.m_list) {
      std::vector<double> per_iteration;
      for (std::size_t rep = 0; rep < o.replicates; ++rep) {
        const OmnibusProblem problem = generate_matched(n, m, o.dim, o.seed + 977u * rep).problem();
        SolveOptions solve;
        solve.dim = o.d;
        solve.eps = 1e-300;  // a fixed iteration budget
        solve.max_iterations = o.iterations;
        solve.parallel = o.parallel;
        solve.dense_cap = o.dense_cap;
        solve.init = InitKind::provided;  // the cell's shared start, outside the clock
        solve.init_config = o.init == InitKind::imputed_cmds
                                ? imputed_omnibus_init(problem, o.d, o.dense_cap)
                                : averaged_procrustes_init(problem, o.d, o.parallel);
        const EmbeddingResult r = fjofc_embed(problem, spec, solve);
        per_iteration.insert(per_iteration.end(), r.step_seconds.begin(), r.step_seconds.end());
      }
      const CellStats st(std::move(per_iteration));
      BenchRow row{n, m, "fjofc", o.replicates, o.iterations};
      row.mean_step_seconds = st.mean;
      row.stderr_step_seconds = st.std_error;
      row.median_step_seconds = st.median;
      row.min_step_seconds = st.minimum;
      rows.push_back(row);
    }
  return rows;
}

void write_bench_csv(const std::string& path, const std::vector<BenchRow>& rows) {
  std::ofstream out(path);
  if (!out) throw std::invalid_argument("cannot open '" + path + "'");
  out << "n,m,algorithm,replicates,iterations,mean_step_seconds,stderr_step_seconds,"
         "median_step_seconds,min_step_seconds\n";
  char num[4][32];
  for (const BenchRow& r : rows) {
    const double v[4] = {r.mean_step_seconds, r.stderr_step_seconds, r.median_step_seconds,
                         r.min_step_seconds};
    for (int i = 0; i < 4; ++i) std::snprintf(num[i], sizeof num[i], "%.9e", v[i]);
    out << r.n << ',' << r.m << ',' << r.algorithm << ',' << r.replicates << ',' << r.iterations
        << ',' << num[0] << ',' << num[1] << ',' << num[2] << ',' << num[3] << '\n';
  }
}

BenchOptions parse_bench_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::invalid_argument("cannot open '" + path + "'");
  BenchOptions o;
  std::size_t lineno = 0;
  for (std::string raw; std::getline(in, raw);) {
    ++lineno;
    const std::string line = trimmed(raw.substr(0, raw.find('#')));
    if (line.empty()) continue;
    const std::string where = "'" + path + "' line " + std::to_string(lineno);
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw std::invalid_argument(where + ": expected key = value");
    const std::string key = trimmed(line.substr(0, eq));
    const auto setter = grid_keys().find(key);
    if (setter == grid_keys().end())
      throw std::invalid_argument(where + ": unknown key '" + key + "'");
    setter->second(o, trimmed(line.substr(eq + 1)));
  }
  return o;
}

}  // namespace jofc
