// C++ parity suite for the drop-in jofc:: API (libjofc.so over the CUDA path),
// written the way the reference's own suites are (proj/tests/test_embed_core.cpp,
// proj/tests/test_oos.cpp): seeded random problems, checks against an oracle.
// The oracle is the C restatement (oracle/jofc_oracle.c), itself pinned
// bit-for-bit to the reference by tests/test_oracle.py.  Exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "jofc/init.hpp"
#include "jofc/io.hpp"
#include "jofc/linalg.hpp"
#include "jofc/oos.hpp"
#include "jofc/rng.hpp"
#include "jofc/solver.hpp"
#include "jofc/stress.hpp"
#include "jofc/weights.hpp"
#include "jofc_oracle.h"

using namespace jofc;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                            \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// ---------------------------------------------------------------- helpers
static DenseMatrix random_matrix(Rng& rng, std::size_t r, std::size_t c, double scale = 1.0) {
  DenseMatrix m(r, c);
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = scale * rng.normal();
  return m;
}

static DenseMatrix edm(const DenseMatrix& x) {
  DenseMatrix out(x.rows(), x.rows());
  jo_euclidean_distance_matrix(x.rows(), x.cols(), x.data(), out.data());
  return out;
}

static OmnibusProblem random_problem(Rng& rng, std::size_t n, std::size_t m, std::size_t dim) {
  std::vector<DenseMatrix> mods;
  for (std::size_t l = 0; l < m; ++l) mods.push_back(edm(random_matrix(rng, n, dim, 2.0)));
  return OmnibusProblem(std::move(mods));
}

static Configuration random_config(Rng& rng, std::size_t n, std::size_t m, std::size_t d,
                                   double scale = 1.0) {
  Configuration c;
  for (std::size_t l = 0; l < m; ++l) c.blocks.push_back(random_matrix(rng, n, d, scale));
  return c;
}

static std::vector<WeightSpec> families(std::size_t m, double w) {
  std::vector<WeightSpec> out{WeightSpec::uniform(w)};
  DenseMatrix g(m, m);
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < m; ++j)
      g(i, j) = (i == j) ? w * (1.0 + 0.1 * i) : w * (1.0 + 0.25 * std::abs(double(i) - double(j)));
  out.push_back(WeightSpec::general(g));
  std::vector<double> within(m);
  for (std::size_t i = 0; i < m; ++i) within[i] = w * (1.0 + 0.5 * i);
  out.push_back(WeightSpec::product(within, 1.5));
  return out;
}

struct OracleSpec {
  jo_weights w{};
  std::vector<double> g, p;
  explicit OracleSpec(const WeightSpec& s) {
    if (s.kind() == WeightSpec::Kind::uniform) {
      w.kind = 0;
      w.w = s.uniform_w();
    } else if (s.kind() == WeightSpec::Kind::general_symmetric) {
      w.kind = 1;
      g.assign(s.general_matrix().data(), s.general_matrix().data() + s.general_matrix().size());
      w.general = g.data();
    } else {
      w.kind = 2;
      p = s.product_within();
      w.within = p.data();
      w.scale = s.fidelity_scale();
    }
  }
};

static std::vector<double> flat(const Configuration& c) {
  std::vector<double> v;
  for (const auto& b : c.blocks) v.insert(v.end(), b.data(), b.data() + b.size());
  return v;
}

static std::vector<double> flat(const OmnibusProblem& p) {
  std::vector<double> v;
  for (std::size_t l = 0; l < p.modality_count(); ++l)
    v.insert(v.end(), p.modality(l).data(), p.modality(l).data() + p.modality(l).size());
  return v;
}

static double rel_fro(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num) / (den > 0 ? std::sqrt(den) : 1.0);
}

static double rel(double a, double b) { return std::abs(a - b) / std::max(std::abs(b), 1e-300); }

// ---------------------------------------------------------------- tests
static void fast_step_grid() {
  // proj/tests/test_embed_core.cpp:170-183 grid, against the oracle
  Rng rng(38);
  for (std::size_t m : {1, 2, 3})
    for (std::size_t n : {3, 5, 8, 70})
      for (std::size_t d : {1, 2, 3})
        for (double w : {0.5, 1.0, 10.0})
          for (const WeightSpec& spec : families(m, w)) {
            const OmnibusProblem problem = random_problem(rng, n, m, d);
            const Configuration x = random_config(rng, n, m, d);
            const Configuration step = guttman_step_fast(x, problem, spec);
            const OracleSpec os(spec);
            const auto delta = flat(problem);
            const auto xf = flat(x);
            std::vector<double> ref(xf.size());
            jo_guttman_step_fast(m, n, d, delta.data(), &os.w, xf.data(), ref.data());
            CHECK(rel_fro(flat(step), ref) < 1e-12);
            double s_ref = 0.0;
            jo_raw_stress(m, n, d, delta.data(), &os.w, xf.data(), &s_ref);
            CHECK(rel(raw_stress(x, problem, spec), s_ref) < 1e-12);
          }
}

static void solve_trajectory() {
  // proj/tests/test_embed_core.cpp:310-329 style: same iterates as the oracle
  Rng rng(47);
  for (std::size_t m : {1, 2, 3}) {
    const std::size_t n = 90, d = 2;
    const OmnibusProblem problem = random_problem(rng, n, m, d);
    const Configuration start = random_config(rng, n, m, d);
    for (const WeightSpec& spec : families(m, 0.8)) {
      SolveOptions opt;
      opt.dim = d;
      opt.max_iterations = 30;
      opt.eps = 1e-300;
      opt.init = InitKind::provided;
      opt.init_config = start;
      const EmbeddingResult r = fjofc_embed(problem, spec, opt);
      const OracleSpec os(spec);
      const auto delta = flat(problem);
      const auto x0 = flat(start);
      std::vector<double> xr(x0.size()), tr(31);
      std::size_t its = 0;
      int conv = 0;
      jo_fjofc_embed(m, n, d, delta.data(), &os.w, x0.data(), 1e-300, 30, 0, xr.data(), tr.data(),
                     &its, &conv);
      CHECK(r.iterations == its);
      CHECK(rel_fro(flat(r.config), xr) < 1e-8);
      for (std::size_t t = 0; t <= std::min(its, r.iterations); ++t)
        CHECK(rel(r.stress_trace[t], tr[t]) < 1e-10);
      CHECK(r.step_seconds.size() == r.iterations);
      for (std::size_t t = 1; t < r.stress_trace.size(); ++t)
        CHECK(r.stress_trace[t] <= r.stress_trace[t - 1] + 1e-9);
      // keep_config_trace walks the same iterates through the host loop
      opt.keep_config_trace = true;
      opt.max_iterations = 6;
      const EmbeddingResult k = fjofc_embed(problem, spec, opt);
      CHECK(k.config_trace.size() == k.iterations + 1);
      CHECK(rel(k.stress_trace.back(), tr[k.iterations]) < 1e-10);
    }
  }
}

static void default_init_runs() {
  // fjofc_embed with default SolveOptions (InitKind::averaged_procrustes) now
  // works end to end; the trace decreases from the cMDS start.
  Rng rng(77);
  const OmnibusProblem problem = random_problem(rng, 120, 2, 3);
  SolveOptions opt;
  opt.dim = 2;
  opt.max_iterations = 50;
  const EmbeddingResult r = fjofc_embed(problem, WeightSpec::uniform(1.0), opt);
  CHECK(r.iterations >= 1);
  for (std::size_t t = 1; t < r.stress_trace.size(); ++t)
    CHECK(r.stress_trace[t] <= r.stress_trace[t - 1] + 1e-9);
  SolveOptions imp = opt;
  imp.init = InitKind::imputed_cmds;
  const EmbeddingResult ri = fjofc_embed(problem, WeightSpec::uniform(1.0), imp);
  CHECK(ri.iterations >= 1);
  const Configuration start = imputed_omnibus_init(problem, 2);
  CHECK(std::abs(raw_stress(start, problem, WeightSpec::uniform(1.0)) - ri.stress_trace[0]) <=
        1e-10 * ri.stress_trace[0]);
  imp.dense_cap = 100;
  CHECK(throws<std::invalid_argument>([&] { fjofc_embed(problem, WeightSpec::uniform(1.0), imp); }));
  const Configuration init = averaged_procrustes_init(problem, 2);
  CHECK(init.modality_count() == 2 && init.object_count() == 120 && init.dim() == 2);
  CHECK(std::abs(raw_stress(init, problem, WeightSpec::uniform(1.0)) - r.stress_trace[0]) <=
        1e-10 * r.stress_trace[0]);
}

static void realizable_converges() {
  // proj/tests/test_embed_core.cpp:277-292
  Rng rng(45);
  DenseMatrix x = random_matrix(rng, 10, 2);
  center_columns(x);
  const DenseMatrix delta = edm(x);
  OmnibusProblem problem({delta, delta, delta});
  SolveOptions opt;
  opt.dim = 2;
  opt.init = InitKind::provided;
  opt.init_config = Configuration{{x, x, x}};
  const EmbeddingResult r = fjofc_embed(problem, WeightSpec::uniform(1.0), opt);
  CHECK(r.iterations <= 2);
  CHECK(r.final_stress() < 1e-16);
  CHECK(r.terminated == Termination::converged);
}

static void errors() {
  Rng rng(48);
  const OmnibusProblem problem = random_problem(rng, 5, 2, 2);
  Configuration bad = random_config(rng, 5, 2, 2);
  bad.blocks[0](0, 0) = std::numeric_limits<double>::quiet_NaN();
  SolveOptions opt;
  opt.dim = 2;
  opt.init = InitKind::provided;
  opt.init_config = bad;
  CHECK(throws<NumericalError>([&] { fjofc_embed(problem, WeightSpec::uniform(1.0), opt); }));
  const Configuration wrong = random_config(rng, 6, 2, 2);
  CHECK(throws<std::invalid_argument>([&] { raw_stress(wrong, problem, WeightSpec::uniform(1.0)); }));
  CHECK(throws<std::invalid_argument>(
      [&] { guttman_step_fast(wrong, problem, WeightSpec::uniform(1.0)); }));
  opt.init = InitKind::imputed_cmds;
  opt.dense_cap = 1;  // m n above the cap: the reference's invalid_argument
  CHECK(throws<std::invalid_argument>([&] { fjofc_embed(problem, WeightSpec::uniform(1.0), opt); }));
  DenseMatrix asym = problem.modality(0);
  asym(0, 1) += 1.0;
  CHECK(throws<std::invalid_argument>([&] { OmnibusProblem({asym}); }));
  CHECK(throws<std::invalid_argument>([&] { WeightSpec::uniform(0.0); }));
}

static void out_of_sample() {
  // proj/tests/test_oos.cpp:136-148 grid + embed + seed determinism
  Rng rng(85);
  for (std::size_t m : {1, 2, 4})
    for (std::size_t n : {5, 9, 300})
      for (std::size_t d : {1, 2, 3})
        for (double w : {1.0, 10.0}) {
          const Configuration x = random_config(rng, n, m, d);
          OosDissimilarity deltas;
          deltas.deltas.assign(m, std::vector<double>(n));
          for (auto& v : deltas.deltas)
            for (double& e : v) e = std::abs(rng.normal()) + 0.1;
          const DenseMatrix y = random_matrix(rng, m, d, 1.5);
          const auto xf = flat(x);
          std::vector<double> df;
          for (const auto& v : deltas.deltas) df.insert(df.end(), v.begin(), v.end());
          std::vector<double> ref(m * d);
          jo_oos_step_fast(m, n, d, y.data(), xf.data(), df.data(), w, ref.data());
          const DenseMatrix got = oos_step_fast(y, x, deltas, w);
          CHECK(rel_fro(std::vector<double>(got.data(), got.data() + got.size()), ref) < 1e-12);
          double sref = 0.0;
          jo_oos_stress(m, n, d, y.data(), xf.data(), df.data(), w, &sref);
          CHECK(rel(oos_stress(y, x, deltas, w), sref) < 1e-12);
          const OosResult e = oos_embed(x, deltas, w, OosOptions{1e-300, 60}, 11);
          std::vector<double> ye(m * d), tr(61);
          std::size_t its = 0;
          int conv = 0;
          jo_oos_embed(m, n, d, xf.data(), df.data(), w, 1e-300, 60, 11, ye.data(), tr.data(), &its,
                       &conv);
          CHECK(rel(e.stress_trace[0], tr[0]) < 1e-12);
          if (e.iterations == its)
            CHECK(rel_fro(std::vector<double>(e.y.data(), e.y.data() + e.y.size()), ye) < 1e-8);
          const OosResult e2 = oos_embed(x, deltas, w, OosOptions{1e-300, 60}, 11);
          CHECK(max_abs_diff(e.y, e2.y) == 0.0);
        }
}

static void sharded_nccl() {
  // set_shard with an NCCL id: a one-rank group on this one-GPU box (the
  // exchange's real NCCL calls inside the solve's graph) ends on the
  // unsharded iterate; set_shard(0, 1, {}) returns to the plain context
  Rng rng(93);
  const std::size_t m = 2, n = 700, d = 3;
  std::vector<DenseMatrix> mods;
  const DenseMatrix z = random_matrix(rng, n, 3);
  for (std::size_t l = 0; l < m; ++l) {
    DenseMatrix f = z;
    for (std::size_t i = 0; i < f.size(); ++i) f.data()[i] += 0.1 * rng.normal();
    mods.push_back(edm(f));
  }
  const OmnibusProblem problem(mods);
  const Configuration x0 = random_config(rng, n, m, d);
  SolveOptions o;
  o.dim = d;
  o.eps = 1e-300;
  o.max_iterations = 30;
  o.init = InitKind::provided;
  o.init_config = x0;
  const EmbeddingResult plain = fjofc_embed(problem, WeightSpec::uniform(0.5), o);
  set_shard(0, 1, nccl_unique_id());
  const EmbeddingResult sh = fjofc_embed(problem, WeightSpec::uniform(0.5), o);
  CHECK(sh.iterations == plain.iterations);
  CHECK(rel_fro(flat(sh.config), flat(plain.config)) < 1e-12);
  CHECK(rel(sh.stress_trace.back(), plain.stress_trace.back()) < 1e-12);
  CHECK(throws<std::invalid_argument>([] { set_shard(1, 2, {}); }));
  set_shard(0, 1, {});
  const EmbeddingResult again = fjofc_embed(problem, WeightSpec::uniform(0.5), o);
  CHECK(rel_fro(flat(again.config), flat(plain.config)) < 1e-12);
}

static double max_abs_mat(const DenseMatrix& a, const DenseMatrix& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.data()[i] - b.data()[i]));
  return m;
}

static void linear_algebra() {
  // proj/include/jofc/linalg.hpp contracts, checked through their defining
  // identities (the subspace solver additionally against the Jacobi route)
  Rng rng(91);
  for (std::size_t n : {1, 2, 3, 5, 8}) {
    const DenseMatrix a = random_matrix(rng, n, n);
    const Svd svd = svd_small(a);
    DenseMatrix sig(n, n);
    for (std::size_t i = 0; i < n; ++i) sig(i, i) = svd.sigma[i];
    CHECK(max_abs_mat(svd.u * sig * transpose(svd.v), a) < 1e-12 * std::max(1.0, max_abs(a)));
    CHECK(max_abs_mat(transpose(svd.u) * svd.u, DenseMatrix::identity(n)) < 1e-12);
    CHECK(max_abs_mat(transpose(svd.v) * svd.v, DenseMatrix::identity(n)) < 1e-12);
    for (std::size_t i = 1; i < n; ++i) CHECK(svd.sigma[i - 1] >= svd.sigma[i]);
    const DenseMatrix inv = invert_small(a);
    CHECK(max_abs_mat(a * inv, DenseMatrix::identity(n)) < 1e-9);
  }
  DenseMatrix rank1(3, 3);  // rank-deficient: U still orthogonal
  for (std::size_t i = 0; i < 3; ++i)
    for (std::size_t j = 0; j < 3; ++j) rank1(i, j) = double(i + 1) * double(j + 2);
  const Svd r1 = svd_small(rank1);
  CHECK(max_abs_mat(transpose(r1.u) * r1.u, DenseMatrix::identity(3)) < 1e-12);
  CHECK(throws<NumericalError>([&] { invert_small(rank1); }));
  CHECK(throws<std::invalid_argument>([&] { invert_small(DenseMatrix(2, 3)); }));

  const std::size_t n = 200;
  const DenseMatrix g = random_matrix(rng, n, 9);
  const DenseMatrix s = g * transpose(g);  // rank 9, symmetric PSD
  const auto all = symmetric_eigen_all(s);
  CHECK(all.size() == n);
  for (std::size_t i = 1; i < n; ++i) CHECK(all[i - 1].value >= all[i].value);
  const auto top = symmetric_top_eigenpairs(s, 4);
  const auto sub = symmetric_top_eigenpairs_subspace(s, 4);  // GPU route (n > 64)
  for (std::size_t c = 0; c < 4; ++c) {
    CHECK(std::abs(top[c].value - all[c].value) <= 1e-12 * std::abs(all[0].value));
    CHECK(std::abs(sub[c].value - top[c].value) <= 1e-9 * std::abs(all[0].value));
    double dev = 0.0;
    for (std::size_t r = 0; r < n; ++r)
      dev = std::max(dev, std::abs(sub[c].vector[r] - top[c].vector[r]));
    CHECK(dev < 1e-6);
  }
  DenseMatrix asym = s;
  asym(0, 1) += 1.0;
  CHECK(throws<std::invalid_argument>([&] { symmetric_top_eigenpairs_subspace(asym, 2); }));
  CHECK(throws<std::invalid_argument>([&] { symmetric_top_eigenpairs(s, n + 1); }));

  // Procrustes recovers a rotation (up to the centring it applies)
  const DenseMatrix src = random_matrix(rng, 50, 2);
  DenseMatrix rot(2, 2);
  rot(0, 0) = std::cos(0.7);
  rot(0, 1) = -std::sin(0.7);
  rot(1, 0) = std::sin(0.7);
  rot(1, 1) = std::cos(0.7);
  DenseMatrix centred = src;
  center_columns(centred);
  const DenseMatrix tgt = centred * rot;
  CHECK(max_abs_mat(orthogonal_procrustes(src, tgt), tgt) < 1e-12);
}

// load_dissimilarities over CSV (proj/src/io.cpp:127-215): values round-trip
// exactly through %.17g text with blank lines, padding and CRLF; errors carry
// the reference's wording and the line of the first bad row (the GPU ingest
// suite, tests/test_gpu_ingest.py, compares the same strings with the reference).
static std::string write_text(const std::string& name, const std::string& body) {
  const std::string path = "/tmp/jofc_dropin_" + name;
  std::ofstream(path, std::ios::binary) << body;
  return path;
}

static std::string message_of(const std::vector<std::string>& paths) {
  try {
    load_dissimilarities(paths);
  } catch (const std::invalid_argument& e) {
    return e.what();
  }
  return "";
}

static void io_csv() {
  Rng rng(91);
  const std::size_t n = 700;  // ~13 MB of text per file: several parser threads
  DenseMatrix z = random_matrix(rng, n, 3);
  DenseMatrix d = edm(z);
  std::string body;
  char buf[64];
  for (std::size_t i = 0; i < n; ++i) {
    if (i % 97 == 5) body += "   \r\n";
    for (std::size_t j = 0; j < n; ++j) {
      std::snprintf(buf, sizeof buf, "%s %.17g", j ? "," : "", d(i, j));
      body += buf;
    }
    body += (i % 2) ? "\r\n" : "\n";
  }
  const std::string a = write_text("a.csv", body), b = write_text("b.csv", body);
  OmnibusProblem p = load_dissimilarities({a, b});
  CHECK(p.modality_count() == 2 && p.object_count() == n);
  bool same = true;
  for (std::size_t l = 0; l < 2; ++l)
    for (std::size_t i = 0; i < n * n; ++i) same &= p.modality(l).data()[i] == d.data()[i];
  CHECK(same);
  // the first bad line wins, in file order
  std::string bad_body = body;
  const std::size_t at = bad_body.find('\n', bad_body.size() / 2) + 1;  // a line start
  bad_body.insert(at, "0,x");  // a bad number joined to the next row
  const std::string bp = write_text("bad.csv", bad_body);
  const std::string msg = message_of({bp});
  CHECK(msg.find("'" + bp + "' line ") == 0);
  CHECK(msg.find(": cannot parse number '") != std::string::npos);
  std::size_t line = 1;
  for (std::size_t i = 0; i < at; ++i) line += bad_body[i] == '\n';
  CHECK(msg.find(" line " + std::to_string(line) + ":") != std::string::npos);
  const std::string rg = write_text("ragged.csv", "0,1,2\n1,0\n2,1,0\n");
  CHECK(message_of({rg}) == "'" + rg + "' line 2: ragged row");
  const std::string em = write_text("empty.csv", "\n  \n");
  CHECK(message_of({em}) == "'" + em + "': empty matrix");
  CHECK(message_of({"/tmp/jofc_dropin_missing.csv"}) ==
        "cannot open '/tmp/jofc_dropin_missing.csv'");
}

// `dropin_parity oos IN OUT`: jofc::oos_embed (the drop-in entry point) for
// k points of one problem read from IN -- u64 m, n, d, k; X (m x n x d);
// deltas (k x m x n); u64 seeds[k]; f64 w, eps; u64 max_it -- writing per
// point y (m x d), iterations (f64) and the stress trace (max_it + 1, NaN
// padded) to OUT.  tests/test_gpu_oos_c5.py compares it with the reference.
static int oos_file(const char* in_path, const char* out_path) {
  std::ifstream in(in_path, std::ios::binary);
  std::uint64_t hdr[4];
  in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  const std::size_t m = hdr[0], n = hdr[1], d = hdr[2], k = hdr[3];
  std::vector<double> xf(m * n * d), df(k * m * n);
  std::vector<std::uint64_t> seeds(k);
  double w = 0.0, eps = 0.0;
  std::uint64_t max_it = 0;
  in.read(reinterpret_cast<char*>(xf.data()), xf.size() * sizeof(double));
  in.read(reinterpret_cast<char*>(df.data()), df.size() * sizeof(double));
  in.read(reinterpret_cast<char*>(seeds.data()), k * sizeof(std::uint64_t));
  in.read(reinterpret_cast<char*>(&w), sizeof w);
  in.read(reinterpret_cast<char*>(&eps), sizeof eps);
  in.read(reinterpret_cast<char*>(&max_it), sizeof max_it);
  if (!in) return 2;
  Configuration x;
  for (std::size_t l = 0; l < m; ++l) {
    DenseMatrix b(n, d);
    std::copy(xf.begin() + l * n * d, xf.begin() + (l + 1) * n * d, b.data());
    x.blocks.push_back(std::move(b));
  }
  std::ofstream out(out_path, std::ios::binary);
  for (std::size_t q = 0; q < k; ++q) {
    OosDissimilarity dl;
    for (std::size_t l = 0; l < m; ++l)
      dl.deltas.emplace_back(df.begin() + (q * m + l) * n, df.begin() + (q * m + l + 1) * n);
    const OosResult r = oos_embed(x, dl, w, OosOptions{eps, static_cast<std::size_t>(max_it)},
                                  seeds[q]);
    std::vector<double> rec(m * d + 1 + max_it + 1, std::numeric_limits<double>::quiet_NaN());
    std::copy(r.y.data(), r.y.data() + m * d, rec.begin());
    rec[m * d] = static_cast<double>(r.iterations);
    std::copy(r.stress_trace.begin(), r.stress_trace.end(), rec.begin() + m * d + 1);
    out.write(reinterpret_cast<const char*>(rec.data()), rec.size() * sizeof(double));
  }
  return out ? 0 : 3;
}

int main(int argc, char** argv) {
  if (argc == 4 && std::string(argv[1]) == "oos") return oos_file(argv[2], argv[3]);
  fast_step_grid();
  solve_trajectory();
  realizable_converges();
  default_init_runs();
  errors();
  out_of_sample();
  sharded_nccl();
  linear_algebra();
  io_csv();
  std::printf("dropin_parity: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
