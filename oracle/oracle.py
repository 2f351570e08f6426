"""ctypes front end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Two implementations with one calling convention:

* ``Port``      -- ``oracle/libjofc_oracle.so``, the plain-C restatement
                   (``oracle/jofc_oracle.c``); always available once built.
* ``Reference`` -- ``oracle/_ref/libjofc_ref.so``, the unmodified reference
                   sources (``/root/reference/proj/src``) behind
                   ``oracle/ref_shim.cpp``; built here, shipped to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module.  The product package never
does: it fails loudly without its CUDA library instead of falling back here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libjofc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libjofc_ref.so")

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t


class Weights(C.Structure):
    """jo_weights (oracle/jofc_oracle.h); mirrors jofc::WeightSpec."""

    _fields_ = [
        ("kind", C.c_int),
        ("w", C.c_double),
        ("general", _dp),
        ("within", _dp),
        ("scale", C.c_double),
    ]


@dataclass
class Spec:
    """Python-side WeightSpec: kind in {"uniform", "general", "product"}."""

    kind: str
    w: float = 1.0
    general: np.ndarray | None = None
    within: np.ndarray | None = None
    scale: float = 1.0

    @staticmethod
    def uniform(w):
        return Spec("uniform", w=float(w))

    @staticmethod
    def general_(mat):
        return Spec("general", general=np.ascontiguousarray(mat, dtype=np.float64))

    @staticmethod
    def product(within, scale=1.0):
        return Spec("product", within=np.ascontiguousarray(within, dtype=np.float64),
                    scale=float(scale))

    def c(self) -> Weights:
        kinds = {"uniform": 0, "general": 1, "product": 2}
        s = Weights()
        s.kind = kinds[self.kind]
        s.w = self.w
        s.scale = self.scale
        s.general = _ptr(self.general) if self.general is not None else _dp()
        s.within = _ptr(self.within) if self.within is not None else _dp()
        return s


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else _dp()


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(OracleError, ValueError):
    pass


class NumericalError(OracleError, RuntimeError):
    pass


def _raise(code, msg):
    if code == 1:
        raise InvalidArgument(code, msg)
    if code == 2:
        raise NumericalError(code, msg)
    raise OracleError(code, msg)


@dataclass
class EmbedResult:
    x: np.ndarray
    trace: np.ndarray
    iterations: int
    converged: bool
    step_seconds: float = 0.0
    wall_seconds: float = 0.0


class Port:
    """The C restatement; delta is (m, n, n) dense fp64, x is (m, n, d)."""

    kind = "port"

    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        L.jo_last_error.restype = C.c_char_p
        L.jo_stress_pair_count.restype = C.c_double
        L.jo_rng_next_u64.restype = C.c_uint64
        L.jo_rng_normal.restype = C.c_double

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.jo_last_error().decode())

    # -- rng / inputs -------------------------------------------------
    def normals(self, seed, count, scale=1.0):
        out = np.empty(count)
        self.lib.jo_rng_normals(C.c_uint64(seed), _sz(count), C.c_double(scale), _ptr(out))
        return out

    def u64(self, seed, count):
        state = C.create_string_buffer(8 * 312 + 64)
        self.lib.jo_rng_seed(state, C.c_uint64(seed))
        return np.array([self.lib.jo_rng_next_u64(state) for _ in range(count)], dtype=np.uint64)

    def distance_matrix(self, feats):
        feats = _f64(feats)
        n, p = feats.shape
        out = np.empty((n, n))
        self._check(self.lib.jo_euclidean_distance_matrix(_sz(n), _sz(p), _ptr(feats), _ptr(out)))
        return out

    # -- weights ------------------------------------------------------
    def script_w(self, spec, m, n):
        out = np.empty((m, m))
        self._check(self.lib.jo_script_w(C.byref(spec.c()), _sz(m), _sz(n), _ptr(out)))
        return out

    def script_w_inverse(self, spec, m, n):
        out = np.empty((m, m))
        self._check(self.lib.jo_script_w_inverse(C.byref(spec.c()), _sz(m), _sz(n), _ptr(out)))
        return out

    def weights_expand(self, spec, m):
        a, wc = np.empty(m), np.empty((m, m))
        self._check(self.lib.jo_weights_expand(C.byref(spec.c()), _sz(m), _ptr(a), _ptr(wc)))
        return a, wc

    def pair_count(self, m, n):
        return self.lib.jo_stress_pair_count(_sz(m), _sz(n))

    # -- in-sample ----------------------------------------------------
    def raw_stress(self, delta, spec, x, parallel=False):
        delta, x = _f64(delta), _f64(x)
        m, n, d = x.shape
        out = C.c_double()
        self._check(self.lib.jo_raw_stress(_sz(m), _sz(n), _sz(d), _ptr(delta), C.byref(spec.c()),
                                           _ptr(x), C.byref(out)))
        return out.value

    def products(self, delta, spec, x):
        delta, x = _f64(delta), _f64(x)
        m, n, d = x.shape
        out = np.empty_like(x)
        self._check(self.lib.jo_block_guttman_products(_sz(m), _sz(n), _sz(d), _ptr(delta),
                                                       C.byref(spec.c()), _ptr(x), _ptr(out)))
        return out

    def guttman_step_fast(self, delta, spec, x, parallel=False):
        delta, x = _f64(delta), _f64(x)
        m, n, d = x.shape
        out = np.empty_like(x)
        self._check(self.lib.jo_guttman_step_fast(_sz(m), _sz(n), _sz(d), _ptr(delta),
                                                  C.byref(spec.c()), _ptr(x), _ptr(out)))
        return out

    def fjofc_embed(self, delta, spec, x0, eps, max_it, parallel=False, normalize=False):
        delta, x0 = _f64(delta), _f64(x0)
        m, n, d = x0.shape
        x = np.empty_like(x0)
        trace = np.full(max_it + 1, np.nan)
        its, conv = _sz(), C.c_int()
        self._check(self.lib.jo_fjofc_embed(_sz(m), _sz(n), _sz(d), _ptr(delta), C.byref(spec.c()),
                                            _ptr(x0), C.c_double(eps), _sz(max_it), int(normalize),
                                            _ptr(x), _ptr(trace), C.byref(its), C.byref(conv)))
        return EmbedResult(x, trace[: its.value + 1], its.value, bool(conv.value))

    # -- out-of-sample ------------------------------------------------
    def oos_stress(self, y, x, deltas, w):
        y, x, deltas = _f64(y), _f64(x), _f64(deltas)
        m, n, d = x.shape
        out = C.c_double()
        self._check(self.lib.jo_oos_stress(_sz(m), _sz(n), _sz(d), _ptr(y), _ptr(x), _ptr(deltas),
                                           C.c_double(w), C.byref(out)))
        return out.value

    def oos_step_fast(self, y, x, deltas, w):
        y, x, deltas = _f64(y), _f64(x), _f64(deltas)
        m, n, d = x.shape
        out = np.empty((m, d))
        self._check(self.lib.jo_oos_step_fast(_sz(m), _sz(n), _sz(d), _ptr(y), _ptr(x),
                                              _ptr(deltas), C.c_double(w), _ptr(out)))
        return out

    def oos_start(self, x, seed):
        x = _f64(x)
        m, n, d = x.shape
        out = np.empty((m, d))
        self.lib.jo_oos_start(_sz(m), _sz(n), _sz(d), _ptr(x), C.c_uint64(seed), _ptr(out))
        return out

    def oos_embed(self, x, deltas, w, eps, max_it, seed):
        x, deltas = _f64(x), _f64(deltas)
        m, n, d = x.shape
        y = np.empty((m, d))
        trace = np.full(max_it + 1, np.nan)
        its, conv = _sz(), C.c_int()
        self._check(self.lib.jo_oos_embed(_sz(m), _sz(n), _sz(d), _ptr(x), _ptr(deltas),
                                          C.c_double(w), C.c_double(eps), _sz(max_it),
                                          C.c_uint64(seed), _ptr(y), _ptr(trace), C.byref(its),
                                          C.byref(conv)))
        return EmbedResult(y, trace[: its.value + 1], its.value, bool(conv.value))

    def oos_batch(self, x, deltas, w, y0, eps, max_it, fixed=False):
        x, deltas, y0 = _f64(x), _f64(deltas), _f64(y0)
        m, n, d = x.shape
        k = y0.shape[0]
        y = np.empty_like(y0)
        traces = np.full((k, max_it + 1), np.nan)
        its = np.zeros(k, dtype=np.uint64)
        self._check(self.lib.jo_oos_batch(_sz(k), _sz(m), _sz(n), _sz(d), _ptr(x), _ptr(deltas),
                                          C.c_double(w), _ptr(y0), C.c_double(eps), _sz(max_it),
                                          int(fixed), _ptr(y), _ptr(traces),
                                          its.ctypes.data_as(C.POINTER(C.c_size_t))))
        return y, traces, its.astype(np.int64)


class Reference:
    """The real reference (oracle/_ref/libjofc_ref.so) with Port's interface."""

    kind = "reference"

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_create.restype = C.c_void_p
        L.ref_problem_destroy.argtypes = [C.c_void_p]
        for name in ("ref_raw_stress", "ref_guttman_step_fast", "ref_guttman_step_reference",
                     "ref_fjofc_embed"):
            getattr(L, name).argtypes = None
        self._cache = {}

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ref_last_error().decode())

    def max_threads(self):
        return self.lib.ref_max_threads()

    def problem(self, delta):
        """Validated OmnibusProblem handle (cached by array identity)."""
        delta = _f64(delta)
        key = (delta.ctypes.data, delta.shape)
        if key in self._cache:
            return self._cache[key][0]
        m, n, _ = delta.shape
        h = self.lib.ref_problem_create(_sz(m), _sz(n), _ptr(delta))
        if not h:
            _raise(1, self.lib.ref_last_error().decode())
        h = C.c_void_p(h)
        self._cache[key] = (h, delta)
        return h

    def load_dissimilarities(self, paths):
        """proj/src/io.cpp:152-215 -> dense (m, n, n) array (raises on error)."""
        L = self.lib
        L.ref_load_dissimilarities.restype = C.c_void_p
        L.ref_load_dissimilarities.argtypes = [C.POINTER(C.c_char_p), _sz]
        enc = [os.fsencode(p) for p in paths]
        h = L.ref_load_dissimilarities((C.c_char_p * len(enc))(*enc), _sz(len(enc)))
        if not h:
            _raise(1, L.ref_last_error().decode())
        h = C.c_void_p(h)
        try:
            m, n = _sz(), _sz()
            L.ref_problem_shape(h, C.byref(m), C.byref(n))
            out = np.empty((m.value, n.value, n.value))
            for l in range(m.value):
                self._check(L.ref_problem_modality(h, _sz(l), _ptr(out[l])))
            return out
        finally:
            L.ref_problem_destroy(h)

    def oos_step_reference(self, y, x, deltas, w):
        y, x, deltas = _f64(y), _f64(x), _f64(deltas)
        m, n, d = x.shape
        out = np.empty((m, d))
        self.lib.ref_oos_step_reference.argtypes = None
        self._check(self.lib.ref_oos_step_reference(_sz(m), _sz(n), _sz(d), _ptr(y), _ptr(x),
                                                    _ptr(deltas), C.c_double(w), _ptr(out)))
        return out

    def generate_matched(self, n, m, dim, seed):
        out = np.empty((m, n, n))
        self._check(self.lib.ref_generate_matched(_sz(n), _sz(m), _sz(dim), C.c_uint64(seed),
                                                  _ptr(out)))
        return out

    def symmetric_top_eigenpairs_subspace(self, s, k):
        s = _f64(s)
        n = s.shape[0]
        vals, vecs = np.empty(k), np.empty((k, n))
        self._check(self.lib.ref_symmetric_top_eigenpairs_subspace(_sz(n), _ptr(s), _sz(k),
                                                                   _ptr(vals), _ptr(vecs)))
        return vals, vecs

    def simulate_save(self, setting, n, m, dim, n_anom, seed, out):
        self.lib.ref_simulate_save.argtypes = [C.c_char_p, _sz, _sz, _sz, _sz, C.c_uint64,
                                               C.c_char_p]
        self._check(self.lib.ref_simulate_save(setting.encode(), n, m, dim, n_anom, seed,
                                               os.fsencode(out)))

    def parse_run_config(self, path):
        """None when the reference accepts the file, else its message."""
        self.lib.ref_parse_run_config.argtypes = [C.c_char_p]
        rc = self.lib.ref_parse_run_config(os.fsencode(path))
        return None if rc == 0 else self.lib.ref_last_error().decode()

    def save_problem_binary(self, delta, path):
        """proj/src/io.cpp:217-223 (the reference's own .jofc writer)."""
        self._check(self.lib.ref_save_problem_binary(self.problem(delta), os.fsencode(path)))

    def release(self):
        for h, _ in self._cache.values():
            self.lib.ref_problem_destroy(h)
        self._cache.clear()

    def normals(self, seed, count, scale=1.0):
        out = np.empty(count)
        self.lib.ref_rng_normals(C.c_uint64(seed), _sz(count), C.c_double(scale), _ptr(out))
        return out

    def u64(self, seed, count):
        out = np.empty(count, dtype=np.uint64)
        self.lib.ref_rng_u64(C.c_uint64(seed), _sz(count), out.ctypes.data_as(C.c_void_p))
        return out

    def distance_matrix(self, feats, parallel=False):
        feats = _f64(feats)
        n, p = feats.shape
        out = np.empty((n, n))
        self._check(self.lib.ref_euclidean_distance_matrix(_sz(n), _sz(p), _ptr(feats), _ptr(out),
                                                           int(parallel)))
        return out

    def script_w(self, spec, m, n):
        out = np.empty((m, m))
        self._check(self.lib.ref_script_w(C.byref(spec.c()), _sz(m), _sz(n), _ptr(out)))
        return out

    def script_w_inverse(self, spec, m, n):
        out = np.empty((m, m))
        self._check(self.lib.ref_script_w_inverse(C.byref(spec.c()), _sz(m), _sz(n), _ptr(out)))
        return out

    def raw_stress(self, delta, spec, x, parallel=False):
        x = _f64(x)
        m, n, d = x.shape
        out = C.c_double()
        self._check(self.lib.ref_raw_stress(self.problem(delta), C.byref(spec.c()), _sz(d),
                                            _ptr(x), int(parallel), C.byref(out)))
        return out.value

    def guttman_step_fast(self, delta, spec, x, parallel=False):
        x = _f64(x)
        m, n, d = x.shape
        out = np.empty_like(x)
        self._check(self.lib.ref_guttman_step_fast(self.problem(delta), C.byref(spec.c()), _sz(d),
                                                   _ptr(x), int(parallel), _ptr(out)))
        return out

    def guttman_step_reference(self, delta, spec, x):
        x = _f64(x)
        m, n, d = x.shape
        out = np.empty_like(x)
        self._check(self.lib.ref_guttman_step_reference(self.problem(delta), C.byref(spec.c()),
                                                        _sz(d), _ptr(x), _ptr(out)))
        return out

    def fjofc_embed(self, delta, spec, x0, eps, max_it, parallel=False, normalize=False):
        x0 = _f64(x0)
        m, n, d = x0.shape
        x = np.empty_like(x0)
        trace = np.full(max_it + 1, np.nan)
        its, conv = _sz(), C.c_int()
        step_s, wall_s = C.c_double(), C.c_double()
        self._check(self.lib.ref_fjofc_embed(self.problem(delta), C.byref(spec.c()), _sz(d),
                                             _ptr(x0), C.c_double(eps), _sz(max_it), int(parallel),
                                             int(normalize), _ptr(x), _ptr(trace), C.byref(its),
                                             C.byref(conv), C.byref(step_s), C.byref(wall_s)))
        return EmbedResult(x, trace[: its.value + 1], its.value, bool(conv.value),
                           step_s.value, wall_s.value)

    def cmds(self, delta, modality, d):
        n = delta.shape[1]
        out = np.empty((n, d))
        self._check(self.lib.ref_cmds(self.problem(delta), int(modality), _sz(d), _ptr(out)))
        return out

    def imputed_omnibus_init(self, delta, d, dense_cap=4096):
        m, n, _ = delta.shape
        out = np.empty((m, n, d))
        self._check(self.lib.ref_imputed_omnibus_init(self.problem(delta), _sz(d), _sz(dense_cap),
                                                      _ptr(out)))
        return out

    def averaged_procrustes_init(self, delta, d):
        m, n, _ = delta.shape
        out = np.empty((m, n, d))
        self._check(self.lib.ref_averaged_procrustes_init(self.problem(delta), _sz(d), 1,
                                                          _ptr(out)))
        return out

    def fjofc_embed_default_init(self, delta, spec, d, eps, max_it):
        m, n, _ = delta.shape
        x = np.empty((m, n, d))
        trace = np.full(max_it + 1, np.nan)
        its, conv = _sz(), C.c_int()
        self._check(self.lib.ref_fjofc_embed_default_init(
            self.problem(delta), C.byref(spec.c()), _sz(d), C.c_double(eps), _sz(max_it),
            _ptr(x), _ptr(trace), C.byref(its), C.byref(conv)))
        return EmbedResult(x, trace[: its.value + 1], its.value, bool(conv.value))

    def oos_stress(self, y, x, deltas, w):
        y, x, deltas = _f64(y), _f64(x), _f64(deltas)
        m, n, d = x.shape
        out = C.c_double()
        self._check(self.lib.ref_oos_stress(_sz(m), _sz(n), _sz(d), _ptr(y), _ptr(x),
                                            _ptr(deltas), C.c_double(w), C.byref(out)))
        return out.value

    def oos_step_fast(self, y, x, deltas, w):
        y, x, deltas = _f64(y), _f64(x), _f64(deltas)
        m, n, d = x.shape
        out = np.empty((m, d))
        self._check(self.lib.ref_oos_step_fast(_sz(m), _sz(n), _sz(d), _ptr(y), _ptr(x),
                                               _ptr(deltas), C.c_double(w), _ptr(out)))
        return out

    def oos_embed(self, x, deltas, w, eps, max_it, seed):
        x, deltas = _f64(x), _f64(deltas)
        m, n, d = x.shape
        y = np.empty((m, d))
        trace = np.full(max_it + 1, np.nan)
        its, conv = _sz(), C.c_int()
        self._check(self.lib.ref_oos_embed(_sz(m), _sz(n), _sz(d), _ptr(x), _ptr(deltas),
                                           C.c_double(w), C.c_double(eps), _sz(max_it),
                                           C.c_uint64(seed), _ptr(y), _ptr(trace), C.byref(its),
                                           C.byref(conv)))
        return EmbedResult(y, trace[: its.value + 1], its.value, bool(conv.value))

    def oos_batch(self, x, deltas, w, y0, eps, max_it, fixed=False):
        x, deltas, y0 = _f64(x), _f64(deltas), _f64(y0)
        m, n, d = x.shape
        k = y0.shape[0]
        y = np.empty_like(y0)
        traces = np.full((k, max_it + 1), np.nan)
        its = np.zeros(k, dtype=np.uint64)
        self._check(self.lib.ref_oos_batch(_sz(k), _sz(m), _sz(n), _sz(d), _ptr(x), _ptr(deltas),
                                           C.c_double(w), _ptr(y0), C.c_double(eps), _sz(max_it),
                                           int(fixed), _ptr(y), _ptr(traces),
                                           its.ctypes.data_as(C.POINTER(C.c_size_t))))
        return y, traces, its.astype(np.int64)


def best_available():
    """The real reference when it was built here, else the restatement."""
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return Port()
