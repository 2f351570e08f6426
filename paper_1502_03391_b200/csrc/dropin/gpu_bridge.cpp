// Drop-in jofc:: entry points (raw_stress, guttman_step_fast, fjofc_embed,
// oos_*) implemented over the C ABI of libjofc_gpu.so.  Error codes become
// the reference's exceptions: JOFC_EINVAL -> std::invalid_argument,
// JOFC_ENUMERIC -> jofc::NumericalError, CUDA / comm -> std::runtime_error.
// One context per (thread, device); each keeps the packed Delta of the last
// OmnibusProblem it saw resident in HBM (OmnibusProblem is immutable, keyed
// by cache_id()).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "jofc/init.hpp"
#include "jofc/linalg.hpp"
#include "jofc/oos.hpp"
#include "jofc/rng.hpp"
#include "jofc/solver.hpp"
#include "jofc/stress.hpp"
#include "jofc/weights.hpp"
#include "jofc_gpu.h"

namespace jofc {

namespace {

void check(int rc) {
  if (rc == JOFC_OK) return;
  const std::string msg = jofc_last_error();
  if (rc == JOFC_EINVAL) throw std::invalid_argument(msg);
  if (rc == JOFC_ENUMERIC) throw NumericalError(msg);
  throw std::runtime_error("jofc_gpu: " + msg);
}

struct Ctx {
  jofc_ctx* h = nullptr;
  std::uint64_t problem = 0;  // cache_id of the resident problem (0: none)
  bool normalized = false;
  explicit Ctx(int device) { check(jofc_ctx_create(device, &h)); }
  ~Ctx() { jofc_ctx_destroy(h); }
};

thread_local int t_device = 0;
thread_local std::map<int, std::unique_ptr<Ctx>> t_ctx;

Ctx& ctx() {
  auto& slot = t_ctx[t_device];
  if (!slot) slot = std::make_unique<Ctx>(t_device);
  return *slot;
}

Ctx& with_problem(const OmnibusProblem& p, bool normalize) {
  Ctx& c = ctx();
  if (c.problem != p.cache_id() || c.normalized != normalize) {
    std::vector<const double*> ptrs;
    for (std::size_t l = 0; l < p.modality_count(); ++l) ptrs.push_back(p.modality(l).data());
    c.problem = 0;
    check(jofc_set_problem(c.h, p.modality_count(), p.object_count(), ptrs.data(),
                           normalize ? 1 : 0));
    c.problem = p.cache_id();
    c.normalized = normalize;
  }
  return c;
}

// WeightSpec -> the C ABI's plain struct (pointers borrowed for the call).
struct CSpec {
  jofc_weights w{};
  std::vector<double> general;
  explicit CSpec(const WeightSpec& s) {
    switch (s.kind()) {
      case WeightSpec::Kind::uniform:
        w.kind = 0;
        w.w = s.uniform_w();
        break;
      case WeightSpec::Kind::general_symmetric:
        w.kind = 1;
        general.assign(s.general_matrix().data(),
                       s.general_matrix().data() + s.general_matrix().size());
        w.general = general.data();
        break;
      case WeightSpec::Kind::product:
        w.kind = 2;
        w.within = s.product_within().data();
        w.scale = s.fidelity_scale();
        break;
    }
  }
};

std::vector<double> flatten(const Configuration& c) {
  std::vector<double> out;
  out.reserve(c.modality_count() * c.object_count() * c.dim());
  for (const DenseMatrix& b : c.blocks) out.insert(out.end(), b.data(), b.data() + b.size());
  return out;
}

Configuration unflatten(const std::vector<double>& x, std::size_t m, std::size_t n,
                        std::size_t d) {
  Configuration c;
  for (std::size_t l = 0; l < m; ++l) {
    DenseMatrix b(n, d);
    std::memcpy(b.data(), x.data() + l * n * d, n * d * sizeof(double));
    c.blocks.push_back(std::move(b));
  }
  return c;
}

}  // namespace

void set_device(int device) { t_device = device; }

std::vector<unsigned char> nccl_unique_id() {
  std::vector<unsigned char> id(JOFC_NCCL_ID_BYTES);
  check(jofc_nccl_unique_id(id.data()));
  return id;
}

void set_shard(int rank, int world, const std::vector<unsigned char>& nccl_id) {
  if (world > 1 && nccl_id.empty())
    throw std::invalid_argument("set_shard: a sharded context needs the group's NCCL id");
  if (!nccl_id.empty() && nccl_id.size() != JOFC_NCCL_ID_BYTES)
    throw std::invalid_argument("set_shard: the NCCL id is 128 bytes");
  Ctx& c = ctx();
  check(jofc_set_shard(c.h, rank, world));  // (drops the resident problem)
  c.problem = 0;
  if (!nccl_id.empty()) check(jofc_nccl_init(c.h, nccl_id.data(), rank, world));
}

Configuration averaged_procrustes_init(const OmnibusProblem& problem, std::size_t d, bool) {
  Ctx& c = with_problem(problem, false);
  std::vector<double> x(problem.modality_count() * problem.object_count() * d);
  check(jofc_init_averaged_procrustes(c.h, d, x.data()));
  return unflatten(x, problem.modality_count(), problem.object_count(), d);
}

Configuration imputed_omnibus_init(const OmnibusProblem& problem, std::size_t d,
                                   std::size_t dense_cap) {
  Ctx& c = with_problem(problem, false);
  std::vector<double> x(problem.modality_count() * problem.object_count() * d);
  check(jofc_init_imputed_cmds(c.h, d, dense_cap, x.data()));
  return unflatten(x, problem.modality_count(), problem.object_count(), d);
}

std::vector<EigenPair> symmetric_top_eigenpairs_subspace(const DenseMatrix& s, std::size_t k) {
  if (!is_square(s))
    throw std::invalid_argument("symmetric_top_eigenpairs_subspace: matrix not square");
  if (symmetry_gap(s) > 1e-9 * std::max(1.0, max_abs(s)))
    throw std::invalid_argument("symmetric_top_eigenpairs_subspace: matrix not symmetric");
  const std::size_t n = s.rows();
  std::vector<double> values(k), vectors(k * n);
  check(jofc_symmetric_top_eigenpairs_subspace(ctx().h, n, s.data(), k, values.data(),
                                               vectors.data()));
  std::vector<EigenPair> out(k);
  for (std::size_t c = 0; c < k; ++c) {
    out[c].value = values[c];
    out[c].vector.assign(vectors.begin() + c * n, vectors.begin() + (c + 1) * n);
  }
  return out;
}

DenseMatrix cmds(const DenseMatrix& delta, std::size_t d) {
  if (!is_square(delta)) throw std::invalid_argument("cmds: matrix not square");
  // one-modality problem (its upper triangle), its own short-lived residency
  OmnibusProblem single({delta});
  Ctx& c = with_problem(single, false);
  DenseMatrix out(delta.rows(), d);
  check(jofc_cmds(c.h, 0, d, out.data()));
  return out;
}

double stress_pair_count(std::size_t m, std::size_t n) {
  const double mn = static_cast<double>(m) * static_cast<double>(n);
  return mn * (mn - 1.0) / 2.0;
}

void require_consistent_shapes(const Configuration& config, const OmnibusProblem& problem,
                               const WeightSpec& spec) {
  spec.validate(problem.modality_count());
  if (config.modality_count() != problem.modality_count())
    throw std::invalid_argument("configuration/problem modality count mismatch");
  if (config.object_count() != problem.object_count())
    throw std::invalid_argument("configuration/problem object count mismatch");
  for (const DenseMatrix& b : config.blocks)
    if (b.rows() != config.object_count() || b.cols() != config.dim())
      throw std::invalid_argument("configuration blocks have inconsistent shapes");
}

double raw_stress(const Configuration& config, const OmnibusProblem& problem,
                  const WeightSpec& spec, bool) {
  require_consistent_shapes(config, problem, spec);
  Ctx& c = with_problem(problem, false);
  const CSpec cs(spec);
  const std::vector<double> x = flatten(config);
  double out = 0.0;
  check(jofc_raw_stress(c.h, &cs.w, config.dim(), x.data(), &out));
  return out;
}

Configuration guttman_step_fast(const Configuration& config, const OmnibusProblem& problem,
                                const WeightSpec& spec, bool) {
  require_consistent_shapes(config, problem, spec);
  Ctx& c = with_problem(problem, false);
  const CSpec cs(spec);
  const std::vector<double> x = flatten(config);
  std::vector<double> next(x.size());
  check(jofc_guttman_step(c.h, &cs.w, config.dim(), x.data(), next.data()));
  return unflatten(next, config.modality_count(), config.object_count(), config.dim());
}

EmbeddingResult fjofc_embed(const OmnibusProblem& problem, const WeightSpec& spec,
                            const SolveOptions& options) {
  // make_init semantics (proj/src/solver.cpp:82-104) for the provided start
  spec.validate(problem.modality_count());
  if (options.dim < 1) throw std::invalid_argument("SolveOptions: dim must be positive");
  if (!(options.eps > 0.0)) throw std::invalid_argument("SolveOptions: eps must be positive");
  const std::size_t m = problem.modality_count(), n = problem.object_count(), d = options.dim;
  Configuration start;
  if (options.init == InitKind::averaged_procrustes) {
    // the reference default, computed on the GPU from the resident Delta
    Ctx& c = with_problem(problem, options.normalize);
    std::vector<double> x(m * n * d);
    check(jofc_init_averaged_procrustes(c.h, d, x.data()));
    start = unflatten(x, m, n, d);
  } else if (options.init == InitKind::imputed_cmds) {
    Ctx& c = with_problem(problem, options.normalize);
    std::vector<double> x(m * n * d);
    check(jofc_init_imputed_cmds(c.h, d, options.dense_cap, x.data()));
    start = unflatten(x, m, n, d);
  } else {
    if (!options.init_config)
      throw std::invalid_argument("SolveOptions: provided init missing a configuration");
    start = *options.init_config;
  }
  const Configuration& x0 = start;
  if (x0.modality_count() != m || x0.object_count() != n || x0.dim() != d)
    throw std::invalid_argument("SolveOptions: provided init has the wrong shape");
  for (const DenseMatrix& b : x0.blocks)
    if (b.rows() != n || b.cols() != d)
      throw std::invalid_argument("configuration blocks have inconsistent shapes");

  const double pairs = stress_pair_count(m, n);
  EmbeddingResult result;
  if (options.keep_config_trace) {
    // Every iterate is wanted: drive the reference loop (solver.cpp:106-150)
    // from the host, one GPU transform + one GPU stress per iteration.
    const OmnibusProblem& p = problem;
    const OmnibusProblem normalized = options.normalize ? problem.normalized() : problem;
    const OmnibusProblem& use = options.normalize ? normalized : p;
    result.config = x0;
    double stress = raw_stress(result.config, use, spec);
    if (!std::isfinite(stress))
      throw NumericalError("embed: non-finite stress at the initial configuration");
    result.stress_trace.push_back(stress);
    result.config_trace.push_back(result.config);
    result.terminated = Termination::max_iterations;
    for (std::size_t it = 0; it < options.max_iterations; ++it) {
      Configuration next = guttman_step_fast(result.config, use, spec);
      const double ns = raw_stress(next, use, spec);
      if (!std::isfinite(ns))
        throw NumericalError("embed: non-finite stress at iteration " + std::to_string(it + 1));
      result.config = std::move(next);
      result.stress_trace.push_back(ns);
      result.config_trace.push_back(result.config);
      ++result.iterations;
      const double decrease = (stress - ns) / pairs;
      stress = ns;
      if (decrease < options.eps) {
        result.terminated = Termination::converged;
        break;
      }
    }
  } else {
    Ctx& c = with_problem(problem, options.normalize);
    const CSpec cs(spec);
    const std::vector<double> x = flatten(x0);
    std::vector<double> out(x.size());
    std::vector<double> trace(options.max_iterations + 1);
    std::vector<double> steps(std::max<std::size_t>(options.max_iterations, 1));
    std::size_t its = 0;
    int converged = 0;
    check(jofc_fjofc_embed(c.h, &cs.w, d, x.data(), options.eps, options.max_iterations,
                           out.data(), trace.data(), &its, &converged, steps.data()));
    result.config = unflatten(out, m, n, d);
    result.stress_trace.assign(trace.begin(), trace.begin() + its + 1);
    result.iterations = its;
    result.terminated = converged ? Termination::converged : Termination::max_iterations;
    result.step_seconds.assign(steps.begin(), steps.begin() + its);
  }
  result.normalized_stress_trace.resize(result.stress_trace.size());
  for (std::size_t i = 0; i < result.stress_trace.size(); ++i)
    result.normalized_stress_trace[i] = result.stress_trace[i] / pairs;
  return result;
}

// ---------------------------------------------------------------- out-of-sample
namespace {

void oos_check(const Configuration& x, const OosDissimilarity& deltas, double w) {
  if (!(w > 0.0)) throw std::invalid_argument("oos: w must be strictly positive");
  if (deltas.modality_count() != x.modality_count())
    throw std::invalid_argument("oos: delta count does not match the configuration");
  for (const auto& v : deltas.deltas) {
    if (v.size() != x.object_count())
      throw std::invalid_argument("oos: delta length does not match the configuration");
    for (double e : v)
      if (!(e >= 0.0) || !std::isfinite(e))
        throw std::invalid_argument("oos: deltas must be finite and nonnegative");
  }
}

std::vector<double> flatten(const OosDissimilarity& d) {
  std::vector<double> out;
  for (const auto& v : d.deltas) out.insert(out.end(), v.begin(), v.end());
  return out;
}

DenseMatrix oos_start(const Configuration& x, std::uint64_t seed) {
  const std::size_t m = x.modality_count(), n = x.object_count(), d = x.dim();
  double rms = 0.0;
  for (const DenseMatrix& b : x.blocks) {
    const double f = frobenius_norm(b);
    rms += f * f;
  }
  rms = std::sqrt(rms / static_cast<double>(m * n));
  Rng rng(seed);
  DenseMatrix y(m, d);
  const double scale = rms / std::sqrt(static_cast<double>(d));
  for (std::size_t i = 0; i < y.size(); ++i) y.data()[i] = scale * rng.normal();
  return y;
}

}  // namespace

double oos_stress(const DenseMatrix& y, const Configuration& x, const OosDissimilarity& deltas,
                  double w) {
  oos_check(x, deltas, w);
  if (y.rows() != x.modality_count() || y.cols() != x.dim())
    throw std::invalid_argument("oos: y must be m x d");
  const std::vector<double> xf = flatten(x), df = flatten(deltas);
  double out = 0.0;
  check(jofc_oos_stress(ctx().h, x.modality_count(), x.object_count(), x.dim(), y.data(),
                        xf.data(), df.data(), w, &out));
  return out;
}

DenseMatrix oos_step_fast(const DenseMatrix& y, const Configuration& x,
                          const OosDissimilarity& deltas, double w) {
  oos_check(x, deltas, w);
  if (y.rows() != x.modality_count() || y.cols() != x.dim())
    throw std::invalid_argument("oos: y must be m x d");
  const std::vector<double> xf = flatten(x), df = flatten(deltas);
  DenseMatrix out(y.rows(), y.cols());
  check(jofc_oos_step(ctx().h, x.modality_count(), x.object_count(), x.dim(), y.data(),
                      xf.data(), df.data(), w, out.data()));
  return out;
}

std::vector<OosResult> oos_embed_batch(const Configuration& x,
                                       const std::vector<OosDissimilarity>& points, double w,
                                       const OosOptions& options,
                                       const std::vector<std::uint64_t>& seeds) {
  if (!(options.eps > 0.0)) throw std::invalid_argument("OosOptions: eps must be positive");
  if (seeds.size() != points.size())
    throw std::invalid_argument("oos_embed_batch: one seed per point required");
  const std::size_t k = points.size(), m = x.modality_count(), n = x.object_count(),
                    d = x.dim();
  std::vector<OosResult> results(k);
  if (k == 0) return results;
  std::vector<double> deltas, y0;
  deltas.reserve(k * m * n);
  y0.reserve(k * m * d);
  for (std::size_t p = 0; p < k; ++p) {
    oos_check(x, points[p], w);
    const std::vector<double> df = flatten(points[p]);
    deltas.insert(deltas.end(), df.begin(), df.end());
    const DenseMatrix s = oos_start(x, seeds[p]);
    y0.insert(y0.end(), s.data(), s.data() + s.size());
  }
  const std::vector<double> xf = flatten(x);
  const std::size_t T = options.max_iterations;
  std::vector<double> y(k * m * d), traces(k * (T + 1));
  std::vector<std::size_t> its(k);
  check(jofc_oos_batch(ctx().h, k, m, n, d, xf.data(), deltas.data(), w, y0.data(), options.eps,
                       T, 0, y.data(), traces.data(), its.data()));
  const double terms = static_cast<double>(m * n) + 0.5 * static_cast<double>(m * (m - 1));
  for (std::size_t p = 0; p < k; ++p) {
    OosResult& r = results[p];
    r.y = DenseMatrix(m, d);
    std::memcpy(r.y.data(), y.data() + p * m * d, m * d * sizeof(double));
    r.iterations = its[p];
    r.stress_trace.assign(traces.begin() + p * (T + 1), traces.begin() + p * (T + 1) + its[p] + 1);
    const bool fired = its[p] >= 1 && (r.stress_trace[its[p] - 1] - r.stress_trace[its[p]]) /
                                              terms < options.eps;
    r.terminated = (its[p] < T || fired) ? Termination::converged : Termination::max_iterations;
  }
  return results;
}

OosResult oos_embed(const Configuration& x, const OosDissimilarity& deltas, double w,
                    const OosOptions& options, std::uint64_t seed) {
  return oos_embed_batch(x, {deltas}, w, options, {seed}).front();
}

}  // namespace jofc
