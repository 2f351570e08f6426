"""The BASELINE.json synthetic workloads drawn through the REFERENCE's own Rng
and euclidean_distance_matrix -- TEST INFRASTRUCTURE ONLY.

bench.py's ``--impl reference`` arm must not load this repo's product library
(``paper_1502_03391_b200``), so it cannot use ``workloads.make``.  This module
restates the same recipes (seeds data 1000 + cfg, X0
2000 + cfg) on a stateful ``jofc::Rng`` stream of ``oracle/_ref`` (the real
reference, ``proj/include/jofc/rng.hpp:17-55``) or, when that was not built,
of the C restatement (``oracle/jofc_oracle.c``).  Every arithmetic step is the
one the product generator performs, in the same order and without fused
multiply-adds, so the arrays are bit-identical to ``workloads.make`` --
``tests/test_workloads_ref.py`` checks that.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from .oracle import PORT_SO, REF_SO, Port, Reference, Spec

DATA_SEED = 1000
X0_SEED = 2000

# cfg -> (m, n, d, p, iterations, w, general weights, oos points)
SHAPES = {
    1: (2, 500, 2, 2, 100, 0.5, True, 0),
    2: (3, 2000, 3, 4, 200, 0.9, False, 0),
    3: (2, 20000, 5, 10, 100, 0.5, False, 0),
    4: (10, 10000, 3, 3, 100, 0.99, False, 0),
    5: (2, 5000, 3, 3, 100, 0.5, False, 1000),
}


class _Stream:
    """One Rng stream of the chosen CPU implementation (uniform / normal draws)."""

    def __init__(self, impl, seed):
        self.impl = impl
        lib = impl.lib
        if isinstance(impl, Reference):
            lib.ref_rng_create.restype = C.c_void_p
            lib.ref_rng_create.argtypes = [C.c_uint64]
            self._h = C.c_void_p(lib.ref_rng_create(C.c_uint64(seed)))
            self._draw, self._free = lib.ref_rng_draw, lib.ref_rng_destroy
        else:
            lib.jo_rng_create.restype = C.c_void_p
            lib.jo_rng_create.argtypes = [C.c_uint64]
            self._h = C.c_void_p(lib.jo_rng_create(C.c_uint64(seed)))
            self._draw, self._free = lib.jo_rng_draw, lib.jo_rng_destroy

    def _take(self, kind, count):
        out = np.empty(int(count))
        self._draw(self._h, C.c_int(kind), C.c_size_t(out.size),
                   out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def uniform(self, count):
        return self._take(0, count)

    def normal(self, count):
        return self._take(1, count)

    def close(self):
        if self._h:
            self._free(self._h)
            self._h = None


def _matmul_in_order(z, q):
    """acc_c = sum_k z[:, k] * q[k, c], k ascending, separate roundings (no FMA)."""
    n, p = z.shape
    out = np.empty((n, q.shape[1]))
    for c in range(q.shape[1]):
        acc = np.zeros(n)
        for k in range(p):
            acc = acc + z[:, k] * q[k, c]
        out[:, c] = acc
    return out


def _orthogonal(rs, q):
    """Gram-Schmidt of a q x q Gaussian draw, column by column."""
    a = rs.normal(q * q).reshape(q, q)
    for j in range(q):
        for i in range(j):
            dot = 0.0
            for r in range(q):
                dot += a[r, i] * a[r, j]
            for r in range(q):
                a[r, j] -= dot * a[r, i]
        nrm = 0.0
        for r in range(q):
            nrm += a[r, j] * a[r, j]
        nrm = float(np.sqrt(nrm))
        for r in range(q):
            a[r, j] /= nrm
    return a


def features(impl, cfg, seed, n_total):
    """(m, n_total, p) per-modality features of config cfg."""
    m, _, _, p, _, _, _, _ = SHAPES[cfg]
    N = n_total
    rs = _Stream(impl, seed)
    try:
        out = np.empty((m, N, p))
        if cfg in (1, 5):  # Z ~ N(0, I); X_l = Z + 0.1 N
            z = rs.normal(N * p)
            for l in range(m):
                out[l] = (z + 0.1 * rs.normal(N * p)).reshape(N, p)
        elif cfg == 2:  # Dirichlet(1,1,1,1) latent; X_l = Z Q_l + 0.05 N
            u = rs.uniform(N * p).reshape(N, p)
            # libm's log (math.log), as std::log: numpy's vectorised log may differ by an ulp
            e = -np.array([math.log(1.0 - v) for v in u.reshape(-1)]).reshape(N, p)
            s = np.zeros(N)
            for k in range(p):
                s = s + e[:, k]
            z = e / s[:, None]
            for l in range(m):
                q = _orthogonal(rs, p)
                x = _matmul_in_order(z, q).reshape(-1)
                out[l] = (x + 0.05 * rs.normal(N * p)).reshape(N, p)
        elif cfg == 3:  # X_1 = Z; X_2 = Z A + 0.2 N, A_ij ~ N(0, 1/p)
            z = rs.normal(N * p).reshape(N, p)
            out[0] = z
            a = (1.0 / np.sqrt(float(p))) * rs.normal(p * p).reshape(p, p)
            x = _matmul_in_order(z, a).reshape(-1)
            out[1] = (x + 0.2 * rs.normal(N * p)).reshape(N, p)
        elif cfg == 4:  # X_l = s_l Z + 0.05 N, Z ~ U[0,1)^3, s_l ~ U[0.5, 2]
            z = rs.uniform(N * p)
            for l in range(m):
                sl = 0.5 + (2.0 - 0.5) * rs.uniform(1)[0]
                out[l] = (sl * z + 0.05 * rs.normal(N * p)).reshape(N, p)
        else:
            raise ValueError(f"unknown workload config {cfg}")
        return out
    finally:
        rs.close()


@dataclass
class RefWorkload:
    cfg: int
    m: int
    n: int
    d: int
    p: int
    iterations: int
    w: float
    general_weights: bool
    features: np.ndarray
    impl: object

    @property
    def spec(self) -> Spec:
        if self.general_weights:
            g = np.full((self.m, self.m), self.w)
            np.fill_diagonal(g, 1.0 - self.w)
            return Spec.general_(g)
        return Spec.uniform(self.w)

    def describe_spec(self):
        if self.general_weights:
            return f"general(diag {1.0 - self.w:g}, off {self.w:g})"
        return f"uniform({self.w:g})"

    def x0(self):
        rs = _Stream(self.impl, X0_SEED + self.cfg)
        try:
            return rs.normal(self.m * self.n * self.d).reshape(self.m, self.n, self.d)
        finally:
            rs.close()

    def dense_delta(self):
        """(m, n, n): the reference's euclidean_distance_matrix of each modality."""
        out = np.empty((self.m, self.n, self.n))
        for l in range(self.m):
            f = np.ascontiguousarray(self.features[l, : self.n])
            if isinstance(self.impl, Reference):
                out[l] = self.impl.distance_matrix(f, parallel=True)
            else:
                out[l] = self.impl.distance_matrix(f)
        return out


def make(cfg, n=None, impl=None) -> RefWorkload:
    """Config cfg with the reference's generators (the Port when _ref is absent)."""
    if impl is None:
        try:
            impl = Reference(REF_SO)
        except (FileNotFoundError, OSError):
            impl = Port(PORT_SO)
    m, n0, d, p, its, w, gen, k = SHAPES[cfg]
    n = int(n or n0)
    feats = features(impl, cfg, DATA_SEED + cfg, n + k)
    return RefWorkload(cfg, m, n, d, p, its, w, gen, feats, impl)
