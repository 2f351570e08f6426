// capi_ingest.cu -- load_dissimilarities straight into the packed device
// layout: jofc_load_problem_files, jofc_problem_shape.
#include <omp.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "ingest_io.h"
#include "capi_internal.h"

using namespace jofc_gpu;
using namespace jofc_gpu::capi;

// ---------------------------------------------------------------- streaming ingest
// load_dissimilarities (proj/src/io.cpp:152-215) straight into the packed
// device layout: files are read in 128-row panels into two pinned host
// buffers, copied asynchronously, and packed by jofc_pack_kernel (upper
// part, raw) and jofc_ingest_combine_kernel (lower part: symmetry check and
// averaging against the mirror).  Entry checks (non-finite, negative) and the
// diagonal run on the host rows while the previous panel is on the device.
// Errors are reported in the reference's order and wording: parse errors of
// any file first (files are read in order), then per file: shape, size,
// entries, symmetry; then the diagonal warnings; then OmnibusProblem's own
// checks (proj/src/problem.cpp:8-32).
namespace {

struct InputCheck {
  std::string name;
  long long rows = 0, cols = 0;
  bool bad = false, nonfinite = false;
  long long bi = 0, bj = 0;
  double bv = 0.0;
  std::vector<std::pair<long long, double>> diag;  // nonzero diagonal entries
};

// True if some entry of v[0, cols) is negative, NaN or infinite: one
// branch-free (vectorisable) pass; the exact position is searched only then.
bool row_has_bad(const double* v, long long cols) {
  int bad = 0;
  for (long long j = 0; j < cols; ++j) bad |= !(v[j] >= 0.0 && v[j] <= 1.7976931348623157e308);
  return bad != 0;
}

void check_row(InputCheck& ck, long long r, const double* v, long long cols) {
  if (!ck.bad && row_has_bad(v, cols))
    for (long long j = 0; j < cols; ++j) {
      const double x = v[j];
      if (!std::isfinite(x) || x < 0.0) {
        ck.bad = true;
        ck.nonfinite = !std::isfinite(x);
        ck.bi = r;
        ck.bj = j;
        ck.bv = x;
        break;
      }
    }
  if (r < cols && v[r] != 0.0) ck.diag.emplace_back(r, v[r]);
}

int load_files(jofc_ctx* c, const std::vector<std::string>& paths, int normalize) {
  using namespace ingest;
  using clk = std::chrono::steady_clock;
  const auto t_call = clk::now();
  if (paths.empty()) return set_error(JOFC_EINVAL, "load_dissimilarities: no input files");
  const std::string& p0 = paths.front();
  const bool binary = paths.size() == 1 && p0.size() >= 5 && p0.compare(p0.size() - 5, 5, ".jofc") == 0;
  c->has_problem = false;
  std::string err;
  std::FILE* bf = nullptr;
  struct Closer {
    std::FILE*& f;
    ~Closer() {
      if (f) std::fclose(f);
    }
  } closer{bf};
  JofcHeader hdr;
  std::unique_ptr<CsvRows> csv(new CsvRows);
  std::vector<double> row;
  long long m = 0, n = 0;
  if (binary) {
    if (!open_jofc(p0, bf, hdr, err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
    if (hdr.d != 0)
      return set_error(JOFC_EINVAL, "'%s': file holds an embedding, not a problem", p0.c_str());
    m = hdr.m;
    n = hdr.n;
  } else {
    m = static_cast<long long>(paths.size());
    if (!csv->open(p0, err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
    const int rc = csv->next(row, err);
    if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
    if (rc == 0) return set_error(JOFC_EINVAL, "'%s': empty matrix", p0.c_str());
    n = static_cast<long long>(row.size());
  }
  const bool device = m >= 1 && n >= 2;
  if (normalize && c->world > 1)
    return set_error(JOFC_EINVAL, "load with normalize needs an unsharded context");
  // panels of whole row blocks, ~64 MB each
  const long long panel_rows =
      std::max<long long>(1, (64LL << 20) / (8LL * std::max<long long>(n, 1)) / kRows) * kRows;
  DevBuf<unsigned long long>& keys = c->ingest_keys;  // first asymmetric pair per modality
  IngestPanels& pin = c->ingest;
  if (device) {
    make_layout(c, static_cast<size_t>(m), static_cast<size_t>(n));
    JOFC_CUDA(c->delta.ensure(static_cast<size_t>(std::max<long long>(c->lay.local(), 1)) *
                              kBlockElems));
    JOFC_CUDA(pin.ensure(static_cast<size_t>(panel_rows) * n));
    JOFC_CUDA(keys.ensure(static_cast<size_t>(m)));
    JOFC_CUDA(cudaMemsetAsync(keys.p, 0xff, m * sizeof(unsigned long long), c->stream));
  }
  const Layout& L = c->lay;
  long long panels = 0;
  // ships host panel k (rows [r0, r0 + rows) of modality l; r0 a multiple of
  // 128) to the device and packs it row block by row block
  auto flush = [&](int k, int l, long long r0, long long rows) -> int {
    JOFC_CUDA(cudaMemcpyAsync(pin.stage[k].p, pin.host[k], static_cast<size_t>(rows) * n * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    JOFC_CUDA(cudaEventRecord(pin.copied[k], c->stream));
    for (long long rb = r0; rb < r0 + rows; rb += kRows) {
      const int B = static_cast<int>(rb / kRows);
      const double* st = pin.stage[k].p + (rb - r0) * n;
      PackParams pk{};
      pk.stage = st;
      pk.pitch = n;
      pk.r0 = rb;
      pk.c0 = 0;
      pk.n = n;
      pk.nT = L.nT;
      pk.bpm = L.bpm;
      pk.g_first = static_cast<long long>(l) * L.bpm + row_first(L.nT, B);
      pk.begin = L.begin;
      pk.end = L.end;
      pk.dst = c->delta.p;
      pk.norm = 0.0;
      pk.bad = nullptr;
      jofc_pack_kernel<<<static_cast<unsigned>(L.nT - 2 * B), 256, 0, c->stream>>>(pk);
      JOFC_CUDA(cudaGetLastError());
      CombineParams cb{};
      cb.stage = st;
      cb.n = n;
      cb.nT = L.nT;
      cb.bpm = L.bpm;
      cb.l = l;
      cb.Bp = B;
      cb.rows = static_cast<int>(std::min<long long>(kRows, r0 + rows - rb));
      cb.begin = L.begin;
      cb.end = L.end;
      cb.dst = c->delta.p;
      cb.asym_key = keys.p + l;
      jofc_ingest_combine_kernel<<<static_cast<unsigned>(2 * (B + 1)), 256, 0, c->stream>>>(cb);
      JOFC_CUDA(cudaGetLastError());
      c->launches += 2;
    }
    return JOFC_OK;
  };
  // JOFC_INGEST_TRACE=1: seconds spent reading + checking, waiting for a free
  // panel, enqueuing copies/kernels, and in the final synchronisation (stderr)
  static const bool trace = std::getenv("JOFC_INGEST_TRACE") != nullptr;
  double t_read = 0.0, t_wait = 0.0, t_flush = 0.0;
  const auto t_begin = clk::now();
  auto since = [](clk::time_point a) {
    return std::chrono::duration<double>(clk::now() - a).count();
  };
  auto acquire = [&](int k) -> int {  // host panel k free again (its last copy landed)
    const auto a = clk::now();
    if (panels >= 2) JOFC_CUDA(cudaEventSynchronize(pin.copied[k]));
    t_wait += since(a);
    return JOFC_OK;
  };

  std::vector<InputCheck> checks(static_cast<size_t>(m));
  for (long long l = 0; l < m; ++l) {
    InputCheck& ck = checks[l];
    ck.name = binary ? p0 : paths[l];
    if (binary) {
      ck.rows = ck.cols = n;
      const int fd = fileno(bf);
      std::vector<double> scratch;
      for (long long r0 = 0; r0 < n; r0 += panel_rows) {
        const long long rows = std::min<long long>(panel_rows, n - r0);
        const int k = static_cast<int>(panels & 1);
        int rc = acquire(k);
        if (rc) return rc;
        double* dst = pin.host[k];
        if (!device) {
          scratch.resize(static_cast<size_t>(rows) * n);
          dst = scratch.data();
        }
        // parallel positioned reads + entry checks, one slab of rows per thread
        const int nt = std::max(1, std::min(16, omp_get_max_threads()));
        const auto t_r0 = clk::now();
        std::vector<InputCheck> part(nt);
        int io_err = 0;
#pragma omp parallel num_threads(nt)
        {
          const int t = omp_get_thread_num();
          const long long a = rows * t / nt, b = rows * (t + 1) / nt;
          const size_t bytes = static_cast<size_t>(b - a) * n * sizeof(double);
          const off_t off = 20 + static_cast<off_t>((l * n + r0 + a) * n) * 8;
          size_t done = 0;
          while (done < bytes) {
            const ssize_t got = pread(fd, reinterpret_cast<char*>(dst + (a * n)) + done,
                                      bytes - done, off + static_cast<off_t>(done));
            if (got <= 0) {
#pragma omp atomic write
              io_err = 1;
              break;
            }
            done += static_cast<size_t>(got);
          }
          if (done == bytes)
            for (long long i = a; i < b; ++i) check_row(part[t], r0 + i, dst + i * n, n);
        }
        t_read += since(t_r0);
        if (io_err) return set_error(JOFC_EINVAL, "'%s': truncated payload", p0.c_str());
        for (const InputCheck& pc : part) {  // merge in row order
          if (pc.bad && !ck.bad) {
            ck.bad = true;
            ck.nonfinite = pc.nonfinite;
            ck.bi = pc.bi;
            ck.bj = pc.bj;
            ck.bv = pc.bv;
          }
          ck.diag.insert(ck.diag.end(), pc.diag.begin(), pc.diag.end());
        }
        if (device && !ck.bad) {
          const auto t_f0 = clk::now();
          rc = flush(k, static_cast<int>(l), r0, rows);
          if (rc) return rc;
          t_flush += since(t_f0);
          ++panels;
        }
      }
      continue;
    }
    // CSV: file l (file 0 is open with its first row parsed)
    if (l > 0) {
      csv.reset(new CsvRows);
      if (!csv->open(paths[l], err)) return set_error(JOFC_EINVAL, "%s", err.c_str());
      const int rc = csv->next(row, err);
      if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
      if (rc == 0) return set_error(JOFC_EINVAL, "'%s': empty matrix", paths[l].c_str());
    }
    ck.cols = static_cast<long long>(row.size());
    const bool packable = device && ck.cols == n;
    long long filled = 0;
    int k = static_cast<int>(panels & 1);
    bool have = true;
    for (long long r = 0;; ++r) {
      if (!have) {
        const int rc = csv->next(row, err);
        if (rc < 0) return set_error(JOFC_EINVAL, "%s", err.c_str());
        if (rc == 0) break;
        if (static_cast<long long>(row.size()) != ck.cols)
          return set_error(JOFC_EINVAL, "'%s' line %zu: ragged row", paths[l].c_str(),
                           csv->line());
      }
      have = false;
      ck.rows = r + 1;
      check_row(ck, r, row.data(), ck.cols);
      if (packable && r < n && !ck.bad) {
        if (filled == 0) {
          k = static_cast<int>(panels & 1);
          const int rc = acquire(k);
          if (rc) return rc;
        }
        std::memcpy(pin.host[k] + static_cast<size_t>(filled) * n, row.data(), n * sizeof(double));
        if (++filled == panel_rows || r == n - 1) {
          const int rc = flush(k, static_cast<int>(l), r + 1 - filled, filled);
          if (rc) return rc;
          ++panels;
          filled = 0;
        }
      }
    }
  }
  // the reference's per-file validation, in file order
  std::vector<unsigned long long> hkeys(static_cast<size_t>(m), ~0ull);
  if (device) {
    JOFC_CUDA(cudaMemcpyAsync(hkeys.data(), keys.p, m * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->stream));
    JOFC_CUDA(cudaStreamSynchronize(c->stream));
  }
  for (long long l = 0; l < m; ++l) {
    const InputCheck& ck = checks[l];
    const char* nm = ck.name.c_str();
    if (ck.rows != ck.cols)
      return set_error(JOFC_EINVAL, "'%s': matrix is %lldx%lld, expected square", nm, ck.rows,
                       ck.cols);
    if (l > 0 && ck.rows != n)
      return set_error(JOFC_EINVAL, "'%s': size %lld differs from earlier modalities (%lld)", nm,
                       ck.rows, n);
    if (ck.bad && ck.nonfinite)
      return set_error(JOFC_EINVAL, "'%s': non-finite entry at (%lld,%lld)", nm, ck.bi, ck.bj);
    if (ck.bad)
      return set_error(JOFC_EINVAL, "'%s': negative entry %s at (%lld,%lld)", nm,
                       std::to_string(ck.bv).c_str(), ck.bi, ck.bj);
    if (hkeys[l] != ~0ull)
      return set_error(JOFC_EINVAL, "'%s': asymmetry beyond tolerance at (%llu,%llu)", nm,
                       hkeys[l] / static_cast<unsigned long long>(n),
                       hkeys[l] % static_cast<unsigned long long>(n));
    for (const auto& dg : ck.diag)
      std::fprintf(stderr, "warning: '%s' diagonal entry (%lld,%lld) = %g forced to 0\n", nm,
                   dg.first, dg.first, dg.second);
  }
  if (m == 0) return set_error(JOFC_EINVAL, "OmnibusProblem: at least one modality required");
  if (n < 2) return set_error(JOFC_EINVAL, "OmnibusProblem: need at least two objects");
  if (normalize) {  // Frobenius norm of each (averaged, zero-diagonal) modality
    const int grid = c->num_sms * 4;
    DevBuf<double> part;
    JOFC_CUDA(part.ensure(grid));
    std::vector<double> hp(grid);
    for (long long l = 0; l < m; ++l) {
      jofc_sumsq_kernel<<<grid, 256, 0, c->stream>>>(c->delta.p, l * L.bpm, L.bpm, part.p);
      JOFC_CUDA(cudaGetLastError());
      JOFC_TRY(copy_sync(c, hp.data(), part.p, grid * sizeof(double), cudaMemcpyDeviceToHost));
      double s = 0.0;
      for (double v : hp) s += v;
      const double norm = std::sqrt(2.0 * s);
      if (norm != 0.0) {
        jofc_scale_kernel<<<grid, 256, 0, c->stream>>>(c->delta.p, l * L.bpm, L.bpm, norm);
        JOFC_CUDA(cudaGetLastError());
      }
      c->launches += 2;
    }
  }
  JOFC_TRY(delta_sumsq(c));
  const auto t_s0 = clk::now();
  JOFC_CUDA(cudaStreamSynchronize(c->stream));
  if (trace)
    std::fprintf(stderr, "ingest: %lld panels, read+check %.2f ms, wait %.2f ms, enqueue %.2f ms, "
                 "final sync %.2f ms, pipeline %.2f ms, call %.2f ms\n", panels, t_read * 1e3,
                 t_wait * 1e3, t_flush * 1e3, since(t_s0) * 1e3, since(t_begin) * 1e3,
                 since(t_call) * 1e3);
  c->has_problem = true;
  return JOFC_OK;
}

}  // namespace

extern "C" int jofc_problem_shape(jofc_ctx* c, size_t* m, size_t* n) {
  const int rc = require_problem(c);
  if (rc) return rc;
  if (m) *m = static_cast<size_t>(c->lay.m);
  if (n) *n = static_cast<size_t>(c->lay.n);
  return JOFC_OK;
}

extern "C" int jofc_load_problem_files(jofc_ctx* c, size_t count, const char* const* paths,
                                       int normalize) {
  if (!c) return set_error(JOFC_EINVAL, "null context");
  if (count && !paths) return set_error(JOFC_EINVAL, "null path list");
  std::vector<std::string> ps;
  for (size_t i = 0; i < count; ++i) {
    if (!paths[i]) return set_error(JOFC_EINVAL, "null path %zu", i);
    ps.emplace_back(paths[i]);
  }
  JOFC_CUDA(cudaSetDevice(c->device));
  return load_files(c, ps, normalize);
}
