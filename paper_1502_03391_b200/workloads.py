"""Seeded synthetic inputs for the five BASELINE.json configs.

The generators live in libjofc_gpu.so (paper_1502_03391_b200/csrc/workloads.cpp)
and use the reference's Rng arithmetic, so a host holding the reference can
rebuild identical bits.  Seeds: data = 1000 + cfg, X0 = 2000 + cfg, OOS start
of point q = 3000 + q.  See DESIGN.md "Synthetic workloads".
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import dptr
from .api import WeightSpec

DATA_SEED = 1000
X0_SEED = 2000
OOS_SEED = 3000


@dataclass
class Workload:
    cfg: int
    m: int
    n: int
    d: int
    p: int
    iterations: int
    w: float
    general_weights: bool
    oos_points: int
    features: np.ndarray  # (m, n_total, p)

    @property
    def spec(self) -> WeightSpec:
        if self.general_weights:
            g = np.full((self.m, self.m), self.w)
            np.fill_diagonal(g, 1.0 - self.w)
            return WeightSpec.general(g)
        return WeightSpec.uniform(self.w)

    @property
    def in_features(self):
        return np.ascontiguousarray(self.features[:, : self.n, :])

    def x0(self):
        return normals(X0_SEED + self.cfg, (self.m, self.n, self.d))

    def dense_delta(self):
        """(m, n, n) host dissimilarities, reference euclidean_distance_matrix bits."""
        lib = _capi.load()
        out = np.empty((self.m, self.n, self.n))
        f = self.in_features
        for l in range(self.m):
            fl = np.ascontiguousarray(f[l])
            lib.jofc_wl_distance_matrix(self.n, self.p, dptr(fl), dptr(out[l]))
        return out

    def oos_deltas(self):
        lib = _capi.load()
        k = self.oos_points
        out = np.empty((k, self.m, self.n))
        f = np.ascontiguousarray(self.features)
        lib.jofc_wl_oos_deltas(self.m, self.n, k, self.p, dptr(f), dptr(out))
        return out

    def describe(self):
        return (f"cfg{self.cfg}: m={self.m} n={self.n} d={self.d} w={self.w} "
                f"{self.spec.describe()} it={self.iterations}")


def shape(cfg):
    s = _capi.WorkloadShape()
    if _capi.load().jofc_wl_shape(int(cfg), C.byref(s)):
        raise ValueError(f"unknown workload config {cfg}")
    return s


def make(cfg, n=None, seed=None) -> Workload:
    """Config `cfg` (1..5) of BASELINE.json; n overrides the object count."""
    s = shape(cfg)
    n = int(n or s.n)
    k = int(s.oos_points)
    n_total = n + k
    feats = np.empty((s.m, n_total, s.p))
    rc = _capi.load().jofc_wl_features(int(cfg), int(DATA_SEED + cfg if seed is None else seed),
                                       n_total, dptr(feats))
    if rc:
        raise ValueError("workload generation failed")
    return Workload(cfg, int(s.m), n, int(s.d), int(s.p), int(s.iterations), float(s.w),
                    bool(s.general_weights), k, feats)


def normals(seed, shape_, scale=1.0):
    out = np.empty(int(np.prod(shape_)))
    _capi.load().jofc_wl_normals(int(seed), out.size, float(scale), dptr(out))
    return out.reshape(shape_)
