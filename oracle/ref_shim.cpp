// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj/src by oracle/Makefile
// (namespace renamed to jofc_ref with -Djofc=jofc_ref so it can share a
// process with this repo's drop-in jofc:: library).  Output: oracle/_ref/
// libjofc_ref.so (git-ignored; travels to the GPU box with the snapshot).
// It is the pin for the C restatement (oracle/jofc_oracle.c) and the
// "reference" CPU baseline in bench.py.  Same argument conventions as
// jofc_oracle.h; status 0 ok / 1 std::invalid_argument / 2 NumericalError.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "jofc/distance.hpp"
#include "jofc/init.hpp"
#include "jofc/io.hpp"
#include "jofc/simulate.hpp"
#include "jofc/linalg.hpp"
#include "jofc/oos.hpp"
#include "jofc/problem.hpp"
#include "jofc/rng.hpp"
#include "jofc/solver.hpp"
#include "jofc/stress.hpp"
#include "jofc/weights.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace jofc;

extern "C" {
typedef struct {
  int kind;
  double w;
  const double* general;
  const double* within;
  double scale;
} jo_weights;
}

namespace {
thread_local std::string g_err;

WeightSpec make_spec(const jo_weights* s, std::size_t m) {
  switch (s->kind) {
    case 0: return WeightSpec::uniform(s->w);
    case 1: {
      DenseMatrix g(m, m);
      std::memcpy(g.data(), s->general, m * m * sizeof(double));
      return WeightSpec::general(std::move(g));
    }
    case 2: return WeightSpec::product(std::vector<double>(s->within, s->within + m), s->scale);
  }
  throw std::invalid_argument("unknown weight kind");
}

Configuration to_config(const double* x, std::size_t m, std::size_t n, std::size_t d) {
  Configuration c;
  for (std::size_t l = 0; l < m; ++l) {
    DenseMatrix b(n, d);
    std::memcpy(b.data(), x + l * n * d, n * d * sizeof(double));
    c.blocks.push_back(std::move(b));
  }
  return c;
}

void from_config(const Configuration& c, double* out) {
  std::size_t off = 0;
  for (const auto& b : c.blocks) {
    std::memcpy(out + off, b.data(), b.size() * sizeof(double));
    off += b.size();
  }
}

OosDissimilarity to_deltas(const double* deltas, std::size_t m, std::size_t n) {
  OosDissimilarity o;
  for (std::size_t l = 0; l < m; ++l) o.deltas.emplace_back(deltas + l * n, deltas + (l + 1) * n);
  return o;
}

DenseMatrix to_y(const double* y, std::size_t m, std::size_t d) {
  DenseMatrix out(m, d);
  std::memcpy(out.data(), y, m * d * sizeof(double));
  return out;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ref_rng_normals(uint64_t seed, size_t count, double scale, double* out) {
  Rng r(seed);
  for (size_t i = 0; i < count; ++i) out[i] = scale * r.normal();
}

// A stateful Rng stream (the reference's class): the bench's reference arm
// draws the synthetic workloads through it (oracle/workloads_ref.py).
void* ref_rng_create(uint64_t seed) { return new Rng(seed); }
void ref_rng_destroy(void* h) { delete static_cast<Rng*>(h); }
// kind 0: uniform() [0,1), 1: normal()
void ref_rng_draw(void* h, int kind, size_t count, double* out) {
  Rng& r = *static_cast<Rng*>(h);
  for (size_t i = 0; i < count; ++i) out[i] = kind ? r.normal() : r.uniform();
}

void ref_rng_u64(uint64_t seed, size_t count, uint64_t* out) {
  Rng r(seed);
  for (size_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

int ref_euclidean_distance_matrix(size_t n, size_t p, const double* feats, double* out,
                                  int parallel) {
  return guarded([&] {
    DenseMatrix x(n, p);
    std::memcpy(x.data(), feats, n * p * sizeof(double));
    DenseMatrix dm = euclidean_distance_matrix(x, parallel != 0);
    std::memcpy(out, dm.data(), n * n * sizeof(double));
  });
}

int ref_script_w_inverse(const jo_weights* spec, size_t m, size_t n, double* out) {
  return guarded([&] {
    DenseMatrix inv = ScriptW::make(make_spec(spec, m), m, n).w_inverse;
    std::memcpy(out, inv.data(), m * m * sizeof(double));
  });
}

int ref_script_w(const jo_weights* spec, size_t m, size_t n, double* out) {
  return guarded([&] {
    DenseMatrix w = script_w(make_spec(spec, m), m, n);
    std::memcpy(out, w.data(), m * m * sizeof(double));
  });
}

// Owns the validated OmnibusProblem so that construction (O(m n^2)) stays
// outside any timed region.
void* ref_problem_create(size_t m, size_t n, const double* delta) {
  OmnibusProblem* out = nullptr;
  int rc = guarded([&] {
    std::vector<DenseMatrix> mods;
    for (size_t l = 0; l < m; ++l) {
      DenseMatrix d(n, n);
      std::memcpy(d.data(), delta + l * n * n, n * n * sizeof(double));
      mods.push_back(std::move(d));
    }
    out = new OmnibusProblem(std::move(mods));
  });
  return rc ? nullptr : out;
}

void ref_problem_destroy(void* p) { delete static_cast<OmnibusProblem*>(p); }

// load_dissimilarities (proj/src/io.cpp:152-215): a problem handle, or null
// with ref_last_error() set.
void* ref_load_dissimilarities(const char* const* paths, size_t count) {
  OmnibusProblem* out = nullptr;
  int rc = guarded([&] {
    std::vector<std::string> ps(paths, paths + count);
    out = new OmnibusProblem(load_dissimilarities(ps));
  });
  return rc ? nullptr : out;
}

// The reference library calls behind `jofc simulate` (the CLI's own file
// naming, proj/tools/jofc_main.cpp:108-139, restated here for the test).
int ref_simulate_save(const char* setting, size_t n, size_t m, size_t dim, size_t n_anom,
                      uint64_t seed, const char* out_c) {
  return guarded([&] {
    const std::string out = out_c;
    const SimulatedProblem sim = std::string(setting) == "matched"
                                     ? generate_matched(n, m, dim, seed)
                                     : generate_anomaly(n, m, n_anom, dim, seed);
    const bool binary = out.size() > 5 && out.substr(out.size() - 5) == ".jofc";
    if (binary) {
      save_problem_binary(out, sim.problem());
    } else {
      for (size_t i = 0; i < sim.modalities.size(); ++i)
        save_csv_matrix(out + "_" + std::to_string(i + 1) + ".csv", sim.modalities[i]);
    }
    save_labels(binary ? out + ".labels.csv" : out + "_labels.csv", sim.labels);
    if (!sim.anomalies.empty())
      save_indices(binary ? out + ".anomalies.csv" : out + "_anomalies.csv", sim.anomalies);
  });
}

// parse_run_config (proj/src/io.cpp:354-460): 0, or 1 with the message.
int ref_parse_run_config(const char* path) {
  return guarded([&] { (void)parse_run_config(path); });
}

// symmetric_top_eigenpairs_subspace (proj/src/linalg.cpp:198-271): values k,
// vectors k x n.
int ref_symmetric_top_eigenpairs_subspace(size_t n, const double* s, size_t k, double* values,
                                          double* vectors) {
  return guarded([&] {
    DenseMatrix m(n, n);
    std::memcpy(m.data(), s, n * n * sizeof(double));
    const auto pairs = symmetric_top_eigenpairs_subspace(m, k);
    for (size_t c = 0; c < k; ++c) {
      values[c] = pairs[c].value;
      std::memcpy(vectors + c * n, pairs[c].vector.data(), n * sizeof(double));
    }
  });
}

// oos_step_reference (proj/src/oos.cpp:129-178, the dense OOS transform).
int ref_oos_step_reference(size_t m, size_t n, size_t d, const double* y, const double* x,
                           const double* deltas, double w, double* y_out) {
  return guarded([&] {
    DenseMatrix ym(m, d);
    std::memcpy(ym.data(), y, m * d * sizeof(double));
    Configuration xc;
    for (size_t l = 0; l < m; ++l) {
      DenseMatrix b(n, d);
      std::memcpy(b.data(), x + l * n * d, n * d * sizeof(double));
      xc.blocks.push_back(std::move(b));
    }
    OosDissimilarity od;
    for (size_t l = 0; l < m; ++l) od.deltas.emplace_back(deltas + l * n, deltas + (l + 1) * n);
    const DenseMatrix out = oos_step_reference(ym, xc, od, w);
    std::memcpy(y_out, out.data(), m * d * sizeof(double));
  });
}

// generate_matched (proj/src/simulate.cpp): the m dense n x n dissimilarities.
int ref_generate_matched(size_t n, size_t m, size_t dim, uint64_t seed, double* delta_out) {
  return guarded([&] {
    const SimulatedProblem sim = generate_matched(n, m, dim, seed);
    for (size_t l = 0; l < m; ++l)
      std::memcpy(delta_out + l * n * n, sim.modalities[l].data(), n * n * sizeof(double));
  });
}

int ref_problem_shape(void* prob, size_t* m, size_t* n) {
  const auto& p = *static_cast<OmnibusProblem*>(prob);
  *m = p.modality_count();
  *n = p.object_count();
  return 0;
}

int ref_problem_modality(void* prob, size_t l, double* out) {
  return guarded([&] {
    const auto& d = static_cast<OmnibusProblem*>(prob)->modality(l);
    std::memcpy(out, d.data(), d.size() * sizeof(double));
  });
}

int ref_save_problem_binary(void* prob, const char* path) {
  return guarded([&] { save_problem_binary(path, *static_cast<OmnibusProblem*>(prob)); });
}

int ref_raw_stress(void* prob, const jo_weights* spec, size_t d, const double* x, int parallel,
                   double* out) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    const size_t m = p.modality_count(), n = p.object_count();
    *out = raw_stress(to_config(x, m, n, d), p, make_spec(spec, m), parallel != 0);
  });
}

int ref_guttman_step_fast(void* prob, const jo_weights* spec, size_t d, const double* x,
                          int parallel, double* x_next) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    const size_t m = p.modality_count(), n = p.object_count();
    from_config(guttman_step_fast(to_config(x, m, n, d), p, make_spec(spec, m), parallel != 0),
                x_next);
  });
}

int ref_guttman_step_reference(void* prob, const jo_weights* spec, size_t d, const double* x,
                               double* x_next) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    const size_t m = p.modality_count(), n = p.object_count();
    from_config(guttman_step_reference(to_config(x, m, n, d), p, make_spec(spec, m)), x_next);
  });
}

// fjofc_embed with InitKind::provided; wall_seconds covers the call only.
int ref_fjofc_embed(void* prob, const jo_weights* spec, size_t d, const double* x0, double eps,
                    size_t max_it, int parallel, int normalize, double* x_out, double* trace_out,
                    size_t* iterations, int* converged, double* step_seconds_sum,
                    double* wall_seconds) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    const size_t m = p.modality_count(), n = p.object_count();
    SolveOptions opt;
    opt.dim = d;
    opt.eps = eps;
    opt.max_iterations = max_it;
    opt.parallel = parallel != 0;
    opt.normalize = normalize != 0;
    opt.init = InitKind::provided;
    opt.init_config = to_config(x0, m, n, d);
    const WeightSpec ws = make_spec(spec, m);
    const auto t0 = std::chrono::steady_clock::now();
    EmbeddingResult r = fjofc_embed(p, ws, opt);
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_seconds) *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
    from_config(r.config, x_out);
    for (size_t i = 0; i < r.stress_trace.size(); ++i) trace_out[i] = r.stress_trace[i];
    *iterations = r.iterations;
    *converged = r.terminated == Termination::converged ? 1 : 0;
    double s = 0.0;
    for (double v : r.step_seconds) s += v;
    if (step_seconds_sum) *step_seconds_sum = s;
  });
}

int ref_cmds(void* prob, int modality, size_t d, double* x_out) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    if (modality >= static_cast<int>(p.modality_count()))
      throw std::invalid_argument("cmds: modality out of range");
    DenseMatrix x;
    if (modality < 0) {  // the average, built as averaged_procrustes_init does
      const size_t n = p.object_count();
      DenseMatrix average(n, n);
      for (size_t l = 0; l < p.modality_count(); ++l)
        for (size_t i = 0; i < average.size(); ++i) average.data()[i] += p.modality(l).data()[i];
      for (size_t i = 0; i < average.size(); ++i)
        average.data()[i] /= static_cast<double>(p.modality_count());
      x = cmds(average, d);
    } else {
      x = cmds(p.modality(static_cast<size_t>(modality)), d);
    }
    std::memcpy(x_out, x.data(), x.size() * sizeof(double));
  });
}

int ref_imputed_omnibus_init(void* prob, size_t d, size_t dense_cap, double* x_out) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    from_config(imputed_omnibus_init(p, d, dense_cap), x_out);
  });
}

int ref_averaged_procrustes_init(void* prob, size_t d, int parallel, double* x_out) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    from_config(averaged_procrustes_init(p, d, parallel != 0), x_out);
  });
}

// fjofc_embed with the default InitKind::averaged_procrustes
int ref_fjofc_embed_default_init(void* prob, const jo_weights* spec, size_t d, double eps,
                                 size_t max_it, double* x_out, double* trace_out,
                                 size_t* iterations, int* converged) {
  return guarded([&] {
    const auto& p = *static_cast<OmnibusProblem*>(prob);
    SolveOptions opt;
    opt.dim = d;
    opt.eps = eps;
    opt.max_iterations = max_it;
    opt.parallel = true;
    EmbeddingResult r = fjofc_embed(p, make_spec(spec, p.modality_count()), opt);
    from_config(r.config, x_out);
    for (size_t i = 0; i < r.stress_trace.size(); ++i) trace_out[i] = r.stress_trace[i];
    *iterations = r.iterations;
    *converged = r.terminated == Termination::converged ? 1 : 0;
  });
}

int ref_oos_stress(size_t m, size_t n, size_t d, const double* y, const double* x,
                   const double* deltas, double w, double* out) {
  return guarded([&] {
    *out = oos_stress(to_y(y, m, d), to_config(x, m, n, d), to_deltas(deltas, m, n), w);
  });
}

int ref_oos_step_fast(size_t m, size_t n, size_t d, const double* y, const double* x,
                      const double* deltas, double w, double* y_next) {
  return guarded([&] {
    DenseMatrix r = oos_step_fast(to_y(y, m, d), to_config(x, m, n, d), to_deltas(deltas, m, n), w);
    std::memcpy(y_next, r.data(), m * d * sizeof(double));
  });
}

int ref_oos_embed(size_t m, size_t n, size_t d, const double* x, const double* deltas, double w,
                  double eps, size_t max_it, uint64_t seed, double* y_out, double* trace_out,
                  size_t* iterations, int* converged) {
  return guarded([&] {
    OosOptions opt;
    opt.eps = eps;
    opt.max_iterations = max_it;
    OosResult r = oos_embed(to_config(x, m, n, d), to_deltas(deltas, m, n), w, opt, seed);
    std::memcpy(y_out, r.y.data(), m * d * sizeof(double));
    for (size_t i = 0; i < r.stress_trace.size(); ++i) trace_out[i] = r.stress_trace[i];
    *iterations = r.iterations;
    *converged = r.terminated == Termination::converged ? 1 : 0;
  });
}

// k independent points from caller-given starts.  Per point the loop is the
// control flow of oos_embed (proj/src/oos.cpp:203-227) around the reference's
// own oos_step_fast / oos_stress; fixed != 0 drives max_it steps regardless
// of the stop rule (proj/tests/acceptance/acceptance_main.cpp:457-460 style).
// The OpenMP loop over points is the harness's, not the reference's.
int ref_oos_batch(size_t k, size_t m, size_t n, size_t d, const double* x, const double* deltas,
                  double w, const double* y0, double eps, size_t max_it, int fixed,
                  double* y_out, double* traces, size_t* iterations) {
  const Configuration cx = to_config(x, m, n, d);
  const double term_count = static_cast<double>(m * n) + 0.5 * static_cast<double>(m * (m - 1));
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (size_t p = 0; p < k; ++p) {
    try {
      const OosDissimilarity dl = to_deltas(deltas + p * m * n, m, n);
      DenseMatrix y = to_y(y0 + p * m * d, m, d);
      double* tr = traces + p * (max_it + 1);
      double stress = oos_stress(y, cx, dl, w);
      tr[0] = stress;
      size_t its = 0;
      for (size_t it = 0; it < max_it; ++it) {
        DenseMatrix next = oos_step_fast(y, cx, dl, w);
        const double ns = oos_stress(next, cx, dl, w);
        y = std::move(next);
        tr[it + 1] = ns;
        ++its;
        const double dec = (stress - ns) / term_count;
        stress = ns;
        if (!fixed && dec < eps) break;
      }
      std::memcpy(y_out + p * m * d, y.data(), m * d * sizeof(double));
      iterations[p] = its;
    } catch (...) {
      bad = 1;
    }
  }
  return bad ? 2 : 0;
}

}  // extern "C"
