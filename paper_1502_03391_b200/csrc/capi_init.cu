// capi_init.cu -- the initialisers of the C ABI (include/jofc_gpu.h):
// cmds, averaged_procrustes_init, imputed_omnibus_init and the subspace
// eigen-solver behind them (kernels in jofc_init.cuh).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "jofc_init.cuh"
#include "capi_internal.h"

using namespace jofc_gpu;
using namespace jofc_gpu::capi;

// ---------------------------------------------------------------- initialisation
namespace {

// The panel kernels, instantiated per subspace width p = d + 4.
struct PanelOps {
  void (*matvec)(const double*, long long, const double*, double*, int, cudaStream_t);
  void (*gram_shift)(const double*, const double*, double*, double*, long long, int, double,
                     double*, int, cudaStream_t);
  void (*ritz_orth)(double*, const double*, const double*, long long, int,
                    const init::RitzParams&, double*, double*, int, cudaStream_t);
  void (*apply_rinv)(double*, long long, const init::RitzParams&, cudaStream_t);
};

template <int P>
PanelOps panel_ops() {
  PanelOps o;
  o.matvec = [](const double* S, long long n, const double* q, double* z, int splits,
                 cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((n + init::kMvRows - 1) / init::kMvRows),
                    static_cast<unsigned>(splits));
    init::matvec_sym_kernel<P><<<grid, 256, 0, st>>>(S, n, q, z);
  };
  o.gram_shift = [](const double* q, const double* zp, double* z, double* w, long long n,
                    int splits, double shift, double* part, int grid, cudaStream_t st) {
    init::gram_shift_kernel<P><<<grid, 256, 0, st>>>(q, zp, z, w, n, splits, shift, part);
  };
  o.ritz_orth = [](double* q, const double* z, const double* w, long long n, int k,
                   const init::RitzParams& prm, double* ritz, double* part, int grid,
                   cudaStream_t st) {
    init::ritz_orth_kernel<P><<<grid, 256, 0, st>>>(q, z, w, n, k, prm, ritz, part);
  };
  o.apply_rinv = [](double* q, long long n, const init::RitzParams& prm, cudaStream_t st) {
    init::apply_rinv_kernel<P><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(q, n, prm);
  };
  return o;
}

bool panel_ops_for(int p, PanelOps& o) {
  switch (p) {
    case 5: o = panel_ops<5>(); return true;
    case 6: o = panel_ops<6>(); return true;
    case 7: o = panel_ops<7>(); return true;
    case 8: o = panel_ops<8>(); return true;
    case 9: o = panel_ops<9>(); return true;
    case 10: o = panel_ops<10>(); return true;
    case 11: o = panel_ops<11>(); return true;
    case 12: o = panel_ops<12>(); return true;
    case 13: o = panel_ops<13>(); return true;
    case 14: o = panel_ops<14>(); return true;
    default: return false;
  }
}

// Top-k eigenpairs of the symmetric n x n matrix S (device, row-major) with
// ||S||_F = snorm: the reference's dense cyclic Jacobi (host) when
// n <= jacobi_limit or k + 4 >= n, else its shifted orthogonal iteration with
// Rayleigh-Ritz (proj/src/linalg.cpp:167-271) with the n x p panels on the
// device.  values (k, descending) and vecs (n x k, unit columns, largest
// component positive).
int eigen_top_device(jofc_ctx* c, const double* S_dev, long long n, size_t k, double snorm,
                     long long jacobi_limit, std::vector<double>& values, init::Mat& vecs,
                     int& sweeps, double& t_sync) {
  using clk = std::chrono::steady_clock;
  struct {
    const double* p;
  } S{S_dev};
  values.assign(k, 0.0);
  vecs = init::Mat(n, k);
  if (n <= jacobi_limit || k + 4 >= static_cast<size_t>(n)) {
    // the reference's dense route (cyclic Jacobi on the whole S)
    init::Mat h(n, n);
    JOFC_TRY(copy_sync(c, h.a.data(), S.p, h.a.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> ev;
    init::Mat v;
    if (!init::jacobi_eigen(h, ev, v))
      return set_error(JOFC_ENUMERIC, "jacobi eigensolver did not converge within the sweep cap");
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ev[a] > ev[b]; });
    for (size_t cc = 0; cc < k; ++cc) {
      std::vector<double> col(n);
      for (long long r = 0; r < n; ++r) col[r] = v(r, order[cc]);
      init::fix_sign(col);
      values[cc] = ev[order[cc]];
      for (long long r = 0; r < n; ++r) vecs(r, cc) = col[r];
    }
  } else if (snorm == 0.0) {
    for (size_t cc = 0; cc < k; ++cc) {
      values[cc] = 0.0;
      vecs(cc, cc) = 1.0;
    }
  } else {
    // shifted orthogonal iteration with Rayleigh-Ritz (proj/src/linalg.cpp:167-271)
    const size_t p = k + 4;
    const double shift = snorm, tol = 1e-9 * snorm;
    PanelOps ops;
    if (!panel_ops_for(static_cast<int>(p), ops))
      return set_error(JOFC_EINVAL, "cmds: subspace width %zu unsupported", p);
    init::Mat q(n, p);
    init::Normals rng(0x9e3779b97f4a7c15ull);
    for (double& v : q.a) v = rng.next();
    init::orthonormalize(q);
    const int grid1 = std::min<int>(c->num_sms * 8, static_cast<int>((n + 63) / 64));
    const int grid2 = std::min<int>(c->num_sms * 2, static_cast<int>((n + 255) / 256));
    const int grid = std::max(grid1, grid2);
    const size_t part1 = 2 * p * p, part2 = p + p * p;
    // column splits: enough CTAs for ~16 per SM, each split one n x p partial
    const long long row_blocks = (n + init::kMvRows - 1) / init::kMvRows;
    const int splits = static_cast<int>(std::min<long long>(
        init::kMvMaxSplits, std::max<long long>(1, (16LL * c->num_sms + row_blocks - 1) / row_blocks)));
    DevBuf<double> dq, dzp, dz, dw, dritz, dpart;
    JOFC_CUDA(dzp.ensure(splits * n * p));
    JOFC_CUDA(dq.ensure(n * p));
    JOFC_CUDA(dz.ensure(n * p));
    JOFC_CUDA(dw.ensure(n * p));
    JOFC_CUDA(dritz.ensure(n * k));
    JOFC_CUDA(dpart.ensure(grid * std::max(part1, part2)));
    DevBuf<double> dsum;  // the per-CTA partials summed on the device (CTA order)
    JOFC_CUDA(dsum.ensure(std::max(part1, part2)));
    // pinned staging for the per-CTA partials (two small D2H reads per sweep)
    struct Pinned {
      double* p = nullptr;
      ~Pinned() {
        if (p) cudaFreeHost(p);
      }
    } hpart;
    JOFC_CUDA(cudaMallocHost(&hpart.p, grid * std::max(part1, part2) * sizeof(double)));
    JOFC_CUDA(cudaMemcpyAsync(dq.p, q.a.data(), q.a.size() * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    // per-CTA partials -> one vector on the device (summed in CTA order, as the
    // host did) -> the host: `per` doubles per fetch instead of blocks x per
    auto fetch = [&](int blocks, size_t per) -> int {
      JOFC_CUDA(cudaGetLastError());
      init::sum_partials_kernel<<<static_cast<unsigned>((per + 255) / 256), 256, 0, c->stream>>>(
          dpart.p, blocks, static_cast<int>(per), dsum.p);
      JOFC_CUDA(cudaGetLastError());
      ++c->launches;
      const auto t0 = clk::now();
      JOFC_CUDA(cudaMemcpyAsync(hpart.p, dsum.p, per * sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream));
      JOFC_CUDA(cudaStreamSynchronize(c->stream));
      t_sync += std::chrono::duration<double>(clk::now() - t0).count();
      return JOFC_OK;
    };
    auto sum_part = [&](int, size_t, size_t off, size_t cnt, std::vector<double>& out) {
      out.assign(hpart.p + off, hpart.p + off + cnt);
    };
    bool done = false;
    std::vector<double> acc;
    for (int iter = 0; iter < 5000 && !done; ++iter) {
      ++sweeps;
      cudaEvent_t pe1 = nullptr;
      int rc = prof_begin(c, &pe1);
      if (rc) return rc;
      ops.matvec(S.p, n, dq.p, dzp.p, splits, c->stream);
      if (pe1) JOFC_CUDA(cudaEventRecord(pe1, c->stream));
      ops.gram_shift(dq.p, dzp.p, dz.p, dw.p, n, splits, shift, dpart.p, grid1, c->stream);
      c->launches += 2;
      rc = fetch(grid1, part1);
      if (rc) return rc;
      init::Mat t(p, p), g(p, p);
      sum_part(grid1, part1, 0, p * p, acc);
      std::copy(acc.begin(), acc.end(), t.a.begin());
      sum_part(grid1, part1, p * p, p * p, acc);
      std::copy(acc.begin(), acc.end(), g.a.begin());
      for (size_t i = 0; i < p; ++i)
        for (size_t j = i + 1; j < p; ++j) t(i, j) = t(j, i) = 0.5 * (t(i, j) + t(j, i));
      std::vector<double> theta;
      init::Mat u;
      if (!init::jacobi_eigen(t, theta, u))
        return set_error(JOFC_ENUMERIC, "jacobi eigensolver did not converge within the sweep cap");
      std::vector<size_t> order(p);
      std::iota(order.begin(), order.end(), size_t{0});
      std::stable_sort(order.begin(), order.end(),
                       [&](size_t a, size_t b) { return theta[a] > theta[b]; });
      init::RitzParams prm{};
      for (size_t cc = 0; cc < k; ++cc) {
        for (size_t j = 0; j < p; ++j) prm.u[j * init::kMaxP + cc] = u(j, order[cc]);
        prm.theta[cc] = theta[order[cc]];
        values[cc] = theta[order[cc]];
      }
      init::Mat rinv;
      const bool chol = init::cholesky_rinv(g, rinv);
      for (size_t i = 0; i < p; ++i)
        for (size_t j = 0; j < p; ++j)
          prm.rinv[i * init::kMaxP + j] = chol ? rinv(i, j) : (i == j ? 1.0 : 0.0);
      ops.ritz_orth(dq.p, dz.p, dw.p, n, static_cast<int>(k), prm, dritz.p, dpart.p, grid2,
                    c->stream);
      ++c->launches;
      rc = fetch(grid2, part2);
      if (rc) return rc;
      sum_part(grid2, part2, 0, k, acc);
      bool conv = true;
      for (size_t cc = 0; cc < k; ++cc)
        if (std::sqrt(acc[cc]) > tol) conv = false;
      if (conv) {
        init::Mat ritz(n, k);
        JOFC_TRY(copy_sync(c, ritz.a.data(), dritz.p, ritz.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        for (size_t cc = 0; cc < k; ++cc) {
          std::vector<double> col(n);
          double nr = 0.0;
          for (long long r = 0; r < n; ++r) {
            col[r] = ritz(r, cc);
            nr += col[r] * col[r];
          }
          nr = std::sqrt(nr);
          for (double& v : col) v /= nr;
          init::fix_sign(col);
          for (long long r = 0; r < n; ++r) vecs(r, cc) = col[r];
        }
        done = true;
        break;
      }
      if (!chol) {  // ill-conditioned panel: the reference's Gram-Schmidt on the host
        JOFC_TRY(copy_sync(c, q.a.data(), dw.p, q.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        init::orthonormalize(q);
        JOFC_TRY(copy_sync(c, dq.p, q.a.data(), q.a.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
        continue;
      }
      sum_part(grid2, part2, p, p * p, acc);
      std::copy(acc.begin(), acc.end(), g.a.begin());
      if (init::cholesky_rinv(g, rinv)) {
        for (size_t i = 0; i < p; ++i)
          for (size_t j = 0; j < p; ++j) prm.rinv[i * init::kMaxP + j] = rinv(i, j);
        ops.apply_rinv(dq.p, n, prm, c->stream);
        ++c->launches;
        JOFC_CUDA(cudaGetLastError());
      } else {
        JOFC_TRY(copy_sync(c, q.a.data(), dq.p, q.a.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
        init::orthonormalize(q);
        JOFC_TRY(copy_sync(c, dq.p, q.a.data(), q.a.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
      }
    }
    if (!done)
      return set_error(JOFC_ENUMERIC,
                       "subspace eigensolver did not converge within the iteration cap");
  }
  return JOFC_OK;
}

constexpr int kOmnibus = -2;

// cmds (proj/src/init.cpp:21-42) of modality `which` (-1: the modality
// average, kOmnibus: the imputed omnibus matrix) of the resident problem; x is
// n x d (m n x d for the omnibus) row-major.
int cmds_gpu(jofc_ctx* c, int which, size_t d, init::Mat& x) {
  using clk = std::chrono::steady_clock;
  const bool trace = std::getenv("JOFC_INIT_TRACE") != nullptr;
  const auto t_start = clk::now();
  double t_sync = 0.0;  // seconds spent waiting on the device inside the sweep loop
  int sweeps = 0;
  const Layout& L = c->lay;
  // which >= 0: modality, -1: modality average, kOmnibus: the m n x m n
  // imputed omnibus matrix
  const long long n = (which == kOmnibus) ? static_cast<long long>(L.m) * L.n : L.n;
  if (d < 1 || static_cast<long long>(d) > n)
    return set_error(JOFC_EINVAL, "cmds: dimension out of range");
  DevBuf<double> S, aux;
  JOFC_CUDA(S.ensure(static_cast<size_t>(n) * n));
  JOFC_CUDA(aux.ensure(static_cast<size_t>(n) + 1));
  JOFC_CUDA(cudaMemsetAsync(S.p, 0, static_cast<size_t>(n) * n * sizeof(double), c->stream));
  if (which == kOmnibus)
    init::omnibus_d2_kernel<<<static_cast<unsigned>(L.bpm), 256, 0, c->stream>>>(
        c->delta.p, L.n, L.nT, L.bpm, L.m, S.p);
  else
    init::dense_d2_kernel<<<static_cast<unsigned>(L.bpm), 256, 0, c->stream>>>(
        c->delta.p, n, L.nT, L.bpm, L.m, which, S.p);
  JOFC_CUDA(cudaGetLastError());
  init::row_sums_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, c->stream>>>(S.p, n,
                                                                                          aux.p);
  JOFC_CUDA(cudaGetLastError());
  std::vector<double> rs(n);
  JOFC_CUDA(cudaMemcpyAsync(rs.data(), aux.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  const double inv_n = 1.0 / static_cast<double>(n);
  double total = 0.0;
  for (long long i = 0; i < n; ++i) {
    total += rs[i];
    rs[i] *= inv_n;
  }
  total *= inv_n * inv_n;
  JOFC_CUDA(cudaMemcpyAsync(aux.p, rs.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
  DevBuf<double> fro2;
  JOFC_CUDA(fro2.ensure(1));
  JOFC_CUDA(cudaMemsetAsync(fro2.p, 0, sizeof(double), c->stream));
  init::double_center_kernel<<<static_cast<unsigned>(c->num_sms * 8), 256, 0, c->stream>>>(
      S.p, n, aux.p, total, fro2.p);
  JOFC_CUDA(cudaGetLastError());
  c->launches += 3;
  double f2 = 0.0;
  JOFC_CUDA(cudaMemcpyAsync(&f2, fro2.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  const double snorm = std::sqrt(f2);

  const size_t k = d;
  std::vector<double> values;
  init::Mat vecs;
  {
    const int rc = eigen_top_device(c, S.p, n, k, snorm, 320, values, vecs, sweeps, t_sync);
    if (rc) return rc;
  }
  if (trace)
    std::fprintf(stderr, "[init] cmds(%d) total %.3f s, %d sweeps, device wait %.3f s\n", which,
                 std::chrono::duration<double>(clk::now() - t_start).count(), sweeps, t_sync);
  x = init::Mat(n, d);
  for (size_t cc = 0; cc < d; ++cc) {
    const double sc = std::sqrt(std::max(values[cc], 0.0));  // Torgerson clamp
    for (long long r = 0; r < n; ++r) x(r, cc) = sc * vecs(r, cc);
  }
  init::center_columns(x);
  return JOFC_OK;
}

int require_full_problem(jofc_ctx* c) {
  int rc = require_problem(c);
  if (rc) return rc;
  if (c->world != 1)
    return set_error(JOFC_EINVAL, "initialisation needs an unsharded context (whole Delta)");
  return JOFC_OK;
}

}  // namespace

extern "C" {

int jofc_cmds(jofc_ctx* c, int modality, size_t d, double* x_out) {
  const NvtxScope nvtx_scope("jofc_cmds");
  int rc = require_full_problem(c);
  if (rc) return rc;
  if (modality >= c->lay.m) return set_error(JOFC_EINVAL, "cmds: modality out of range");
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat x;
  rc = cmds_gpu(c, modality, d, x);
  if (rc) return rc;
  JOFC_TRY(copy_sync(c, x_out, x.a.data(), x.a.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_symmetric_top_eigenpairs_subspace(jofc_ctx* c, size_t n, const double* s, size_t k,
                                           double* values, double* vectors) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (!s || !values || !vectors) return set_error(JOFC_EINVAL, "null argument");
  if (k < 1 || k > n)
    return set_error(JOFC_EINVAL, "symmetric_top_eigenpairs_subspace: k out of range");
  if (k + 4 > static_cast<size_t>(init::kMaxP) && n > 64 && k + 4 < n)
    return set_error(JOFC_EINVAL, "symmetric_top_eigenpairs_subspace: k %zu above %d", k,
                     init::kMaxP - 4);
  JOFC_CUDA(cudaSetDevice(c->device));
  const long long nn = static_cast<long long>(n);
  DevBuf<double> S, rows;
  JOFC_CUDA(S.ensure(n * n));
  JOFC_CUDA(rows.ensure(n));
  JOFC_CUDA(cudaMemcpyAsync(S.p, s, n * n * sizeof(double), cudaMemcpyDefault, c->stream));
  init::row_sumsq_kernel<<<static_cast<unsigned>((nn * 32 + 255) / 256), 256, 0, c->stream>>>(
      S.p, nn, rows.p);
  JOFC_CUDA(cudaGetLastError());
  ++c->launches;
  std::vector<double> rs(n);
  JOFC_TRY(copy_sync(c, rs.data(), rows.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  double f2 = 0.0;
  for (double v : rs) f2 += v;
  std::vector<double> vals;
  init::Mat vecs;
  int sweeps = 0;
  double t_sync = 0.0;
  JOFC_TRY(eigen_top_device(c, S.p, nn, k, std::sqrt(f2), 64, vals, vecs, sweeps, t_sync));
  std::vector<double> out(k * n);
  for (size_t cc = 0; cc < k; ++cc)
    for (size_t r = 0; r < n; ++r) out[cc * n + r] = vecs(r, cc);
  JOFC_TRY(copy_sync(c, values, vals.data(), k * sizeof(double), cudaMemcpyDefault));
  JOFC_TRY(copy_sync(c, vectors, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_init_imputed_cmds(jofc_ctx* c, size_t d, size_t dense_cap, double* x_out) {
  const NvtxScope nvtx_scope("jofc_init_imputed_cmds");
  int rc = require_full_problem(c);
  if (rc) return rc;
  const size_t m = static_cast<size_t>(c->lay.m), n = static_cast<size_t>(c->lay.n);
  if (m * n > dense_cap)
    return set_error(JOFC_EINVAL, "imputed_omnibus_init: mn exceeds the dense cap");
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat x;
  rc = cmds_gpu(c, kOmnibus, d, x);
  if (rc) return rc;
  // Configuration::from_stacked, then each block re-centred (init.cpp:111-114)
  std::vector<double> out(m * n * d);
  for (size_t l = 0; l < m; ++l) {
    init::Mat blk(n, d);
    std::copy(x.a.begin() + l * n * d, x.a.begin() + (l + 1) * n * d, blk.a.begin());
    init::center_columns(blk);
    std::copy(blk.a.begin(), blk.a.end(), out.begin() + l * n * d);
  }
  JOFC_TRY(copy_sync(c, x_out, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

int jofc_init_averaged_procrustes(jofc_ctx* c, size_t d, double* x_out) {
  const NvtxScope nvtx_scope("jofc_init_averaged_procrustes");
  int rc = require_full_problem(c);
  if (rc) return rc;
  JOFC_CUDA(cudaSetDevice(c->device));
  init::Mat anchor;
  rc = cmds_gpu(c, -1, d, anchor);
  if (rc) return rc;
  init::center_columns(anchor);
  const size_t block = static_cast<size_t>(c->lay.n) * d;
  std::vector<double> out(static_cast<size_t>(c->lay.m) * block);
  for (int l = 0; l < c->lay.m; ++l) {
    init::Mat xl;
    rc = cmds_gpu(c, l, d, xl);
    if (rc) return rc;
    init::center_columns(xl);
    const init::Mat rot = init::procrustes(xl, anchor);
    std::copy(rot.a.begin(), rot.a.end(), out.begin() + l * block);
  }
  JOFC_TRY(copy_sync(c, x_out, out.data(), out.size() * sizeof(double), cudaMemcpyDefault));
  return JOFC_OK;
}

}  // extern "C"

