"""Host-side mirror of the reference's hot-path API over the C ABI.

Names, argument meaning and error behaviour follow proj/include/jofc:

=========================  ==============================================
reference (C++)            here
=========================  ==============================================
WeightSpec::uniform/...    WeightSpec.uniform / .general / .product
OmnibusProblem             OmnibusProblem (same validation, problem.cpp:8-32)
SolveOptions               SolveOptions (InitKind.provided only, see below)
EmbeddingResult            EmbeddingResult
raw_stress                 raw_stress                (stress.hpp:13-14)
stress_pair_count          stress_pair_count         (stress.hpp:17)
guttman_step_fast          guttman_step_fast         (solver.hpp:12-14)
fjofc_embed                fjofc_embed               (solver.hpp:26-27)
OosDissimilarity           an (m, n) array
oos_stress / oos_step_fast oos_stress / oos_step_fast (oos.hpp:33-39)
oos_embed                  oos_embed                 (oos.hpp:50-51)
(batched OOS, new)         oos_embed_batch
=========================  ==============================================

Configurations are numpy arrays of shape (m, n, d) (Configuration::blocks
stacked).  Every call runs on the GPU through libjofc_gpu.so; the problem is
packed into HBM once per OmnibusProblem and stays resident in the Device.
InitKind::averaged_procrustes (the reference default) runs on the GPU
(cmds over the resident Delta); InitKind::imputed_cmds raises
NotImplementedError.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from ._capi import InvalidArgument, NumericalError, check, dptr


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ----------------------------------------------------------------- weights
class WeightSpec:
    """proj/include/jofc/weights.hpp:20-66 (validation in the C ABI)."""

    def __init__(self, kind, w=1.0, general=None, within=None, scale=1.0):
        self.kind, self.w, self.scale = kind, float(w), float(scale)
        self.general = None if general is None else _f64(general)
        self.within = None if within is None else _f64(within)
        if kind == 0 and not (self.w > 0 and math.isfinite(self.w)):
            raise InvalidArgument("WeightSpec: w must be strictly positive")

    @staticmethod
    def uniform(w):
        return WeightSpec(0, w=w)

    @staticmethod
    def general(mat):
        mat = _f64(mat)
        if mat.ndim != 2 or mat.shape[0] != mat.shape[1] or mat.shape[0] == 0:
            raise InvalidArgument("WeightSpec: general weight matrix must be square")
        if np.any(mat != mat.T):
            raise InvalidArgument("WeightSpec: general weight matrix must be symmetric")
        if np.any(~(mat > 0)) or not np.all(np.isfinite(mat)):
            raise InvalidArgument("WeightSpec: w_ij must be strictly positive")
        return WeightSpec(1, general=mat)

    @staticmethod
    def product(within, fidelity_scale=1.0):
        within = _f64(within)
        if within.size == 0:
            raise InvalidArgument("WeightSpec: product weights must be nonempty")
        if np.any(~(within > 0)):
            raise InvalidArgument("WeightSpec: w_ii must be strictly positive")
        if not fidelity_scale > 0:
            raise InvalidArgument("WeightSpec: c must be strictly positive")
        return WeightSpec(2, within=within, scale=fidelity_scale)

    def within_weight(self, i):
        if self.kind == 1:
            return float(self.general[i, i])
        if self.kind == 2:
            return self.scale * float(self.within[i])
        return 1.0

    def cross_weight(self, i, j):
        if self.kind == 1:
            return float(self.general[i, j])
        if self.kind == 2:
            return float(self.within[i] * self.within[j])
        return self.w

    def c(self):
        s = _capi.Weights()
        s.kind, s.w, s.scale = self.kind, self.w, self.scale
        s.general = dptr(self.general) if self.general is not None else None
        s.within = dptr(self.within) if self.within is not None else None
        return s

    def describe(self):
        if self.kind == 0:
            return f"uniform(w={self.w})"
        if self.kind == 1:
            return f"general({self.general.tolist()})"
        return f"product({self.within.tolist()}, c={self.scale})"


# ----------------------------------------------------------------- problem
class OmnibusProblem:
    """m dissimilarity matrices over the same n objects (problem.cpp:8-32)."""

    def __init__(self, modalities, validate=True):
        mods = [_f64(d) for d in modalities]
        if not mods:
            raise InvalidArgument("OmnibusProblem: at least one modality required")
        n = mods[0].shape[0]
        if n < 2:
            raise InvalidArgument("OmnibusProblem: need at least two objects")
        if validate:
            for i, d in enumerate(mods):
                tag = f"modality {i}"
                if d.ndim != 2 or d.shape != (n, n):
                    raise InvalidArgument(f"OmnibusProblem: {tag} has wrong shape")
                if not np.all(np.isfinite(d)):
                    raise InvalidArgument(f"OmnibusProblem: {tag} has non-finite entries")
                scale = max(1.0, float(np.max(np.abs(d))))
                if float(np.max(np.abs(d - d.T))) > 1e-9 * scale:
                    raise InvalidArgument(f"OmnibusProblem: {tag} is not symmetric")
                if np.any(np.diagonal(d) != 0.0):
                    raise InvalidArgument(f"OmnibusProblem: {tag} has nonzero diagonal")
                if np.any(d < 0.0):
                    raise InvalidArgument(f"OmnibusProblem: {tag} has a negative entry")
        self.modalities = mods
        self._version = object()

    def modality_count(self):
        return len(self.modalities)

    def object_count(self):
        return self.modalities[0].shape[0]

    def normalized(self):
        out = []
        for d in self.modalities:
            nrm = math.sqrt(float(np.sum(d * d)))
            out.append(d if nrm == 0.0 else d / nrm)
        return OmnibusProblem(out, validate=False)

    def leading_objects(self, count):
        n = self.object_count()
        if count < 2 or count > n:
            raise InvalidArgument("OmnibusProblem: invalid restriction size")
        return OmnibusProblem([d[:count, :count] for d in self.modalities], validate=False)


class ResidentProblem:
    """A problem that lives only in HBM: loaded by load_dissimilarities straight
    from files into one Device's packed layout (no host n x n copy).  Usable
    wherever an OmnibusProblem is accepted, with that device."""

    def __init__(self, device, m, n, key):
        self.device, self._m, self._n, self._key = device, m, n, key

    def modality_count(self):
        return self._m

    def object_count(self):
        return self._n


def load_dissimilarities(paths, device=None, normalize=False):
    """proj/include/jofc/io.hpp:19-23 (load_dissimilarities), streamed on the
    device: one CSV per modality or a single .jofc problem file.  Returns a
    ResidentProblem bound to `device` (default device 0)."""
    dev = device or default_device()
    if isinstance(paths, (str, bytes)):
        paths = [paths]
    return dev.load_files(list(paths), normalize=normalize)


def stress_pair_count(m, n):
    mn = float(m) * float(n)
    return mn * (mn - 1.0) / 2.0


class InitKind(enum.Enum):
    imputed_cmds = 0
    averaged_procrustes = 1
    provided = 2


class Termination(enum.Enum):
    converged = 0
    max_iterations = 1


@dataclass
class SolveOptions:
    dim: int = 2
    eps: float = 1e-6
    max_iterations: int = 1000
    parallel: bool = False
    init: InitKind = InitKind.averaged_procrustes
    init_config: Optional[np.ndarray] = None
    normalize: bool = False
    keep_config_trace: bool = False
    dense_cap: int = 4096


@dataclass
class EmbeddingResult:
    config: np.ndarray
    stress_trace: list
    normalized_stress_trace: list
    iterations: int
    terminated: Termination
    step_seconds: list = field(default_factory=list)
    config_trace: list = field(default_factory=list)

    def final_stress(self):
        return self.stress_trace[-1]

    def final_normalized_stress(self):
        return self.normalized_stress_trace[-1]


@dataclass
class OosOptions:
    eps: float = 1e-6
    max_iterations: int = 1000


@dataclass
class OosResult:
    y: np.ndarray
    stress_trace: list
    iterations: int
    terminated: Termination


# ------------------------------------------------------------------ device
class Device:
    """One jofc_ctx on one GPU; keeps the packed problem resident in HBM."""

    def __init__(self, device=0, shard=(0, 1)):
        self.lib = _capi.load()
        h = C.c_void_p()
        check(self.lib.jofc_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        if shard != (0, 1):
            check(self.lib.jofc_set_shard(self.h, int(shard[0]), int(shard[1])))
        self._problem_key = None
        self._hook = None

    def close(self):
        if self.h:
            self.lib.jofc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self):
        return self.lib.jofc_ctx_stream(self.h)

    def launches(self):
        return int(self.lib.jofc_launch_count(self.h))

    def stress_evaluations(self):
        """Iterations (stress evaluations) the device executed since creation."""
        v = C.c_uint64()
        check(self.lib.jofc_stress_evaluations(self.h, C.byref(v)))
        return int(v.value)

    def set_fidelity_form(self, direct: bool):
        """False (default): identity-form fidelity where the route allows it
        (include/jofc_gpu.h, jofc_set_fidelity_form); True: always per pair."""
        check(self.lib.jofc_set_fidelity_form(self.h, 1 if direct else 0))

    def set_oos_route(self, route: int):
        """0 auto (default), 1 the persistent batch solve, 2 one fused launch per
        update (include/jofc_gpu.h, jofc_set_oos_route)."""
        check(self.lib.jofc_set_oos_route(self.h, int(route)))

    def profile(self, enable: bool):
        """CUDA events around every pass launch (also forces per-iteration
        stream launches: no CUDA graph, no single-launch persistent solve)."""
        check(self.lib.jofc_profile(self.h, 1 if enable else 0))

    def set_allreduce(self, fn):
        """fn(ptr: int, count: int, stream: int) -> None, sums in place over ranks."""
        def tramp(buf, count, stream, user):
            try:
                fn(C.cast(buf, C.c_void_p).value, int(count), stream)
                return 0
            except Exception:  # noqa: BLE001 -- reported as JOFC_ECOMM
                return 1
        self._hook = _capi.ALLREDUCE_FN(tramp)
        check(self.lib.jofc_set_allreduce(self.h, self._hook, None))

    # C-native NCCL exchange (include/jofc_gpu.h, jofc_nccl_*): the default
    # multi-GPU path; paper_1502_03391_b200.dist.attach_nccl_native runs the
    # SPMD id broadcast / init sequence
    @staticmethod
    def nccl_unique_id():
        _process_nccl()
        buf = C.create_string_buffer(128)
        check(_capi.load().jofc_nccl_unique_id(buf))
        return buf.raw

    @staticmethod
    def nccl_version():
        _process_nccl()
        v = C.c_int()
        check(_capi.load().jofc_nccl_version(C.byref(v)))
        return int(v.value)

    def nccl_init(self, uid, rank, world):
        if len(uid) != 128:
            raise InvalidArgument("NCCL exchange: the unique id is 128 bytes")
        _process_nccl()
        check(self.lib.jofc_nccl_init(self.h, uid, int(rank), int(world)))

    def nccl_release(self):
        check(self.lib.jofc_nccl_release(self.h))

    # peer-memory exchange (include/jofc_gpu.h, jofc_peer_*): multi-GPU
    # without the all-reduce hook; paper_1502_03391_b200.dist.attach_peers
    # runs the SPMD export / all-gather / attach sequence
    def peer_export(self):
        """(64-byte CUDA IPC handle, device pointer) of this rank's slab."""
        buf = C.create_string_buffer(64)
        slab = C.c_void_p()
        check(self.lib.jofc_peer_export(self.h, buf, C.byref(slab)))
        return buf.raw, slab.value

    def peer_attach(self, rank, world, handles):
        """handles: the world's 64-byte handles, rank order."""
        blob = b"".join(handles)
        if len(blob) != 64 * world:
            raise InvalidArgument("peer exchange: need world x 64-byte handles")
        check(self.lib.jofc_peer_attach(self.h, int(rank), int(world), blob))

    def peer_attach_pointers(self, rank, world, slabs):
        arr = (C.c_void_p * world)(*slabs)
        check(self.lib.jofc_peer_attach_pointers(self.h, int(rank), int(world), arr))

    def peer_detach(self):
        check(self.lib.jofc_peer_detach(self.h))

    def load_files(self, paths, normalize=False):
        enc = [os.fsencode(p) for p in paths]
        arr = (C.c_char_p * len(enc))(*enc)
        check(self.lib.jofc_load_problem_files(self.h, len(enc), arr, int(bool(normalize))))
        key = ("files", tuple(paths), bool(normalize), object())
        self._problem_key = key
        self._keep = None
        m, n = self._resident_shape()
        return ResidentProblem(self, m, n, key)

    def _resident_shape(self):
        m, n = C.c_size_t(), C.c_size_t()
        check(self.lib.jofc_problem_shape(self.h, C.byref(m), C.byref(n)))
        return m.value, n.value

    def upload(self, problem, normalize=False):
        if isinstance(problem, ResidentProblem):
            if problem.device is not self or problem._key != self._problem_key:
                raise InvalidArgument("ResidentProblem: no longer resident on this device")
            if normalize:
                raise InvalidArgument("ResidentProblem: load with normalize=True instead")
            return
        key = (id(problem), problem._version, bool(normalize))
        if key == self._problem_key:
            return
        mods = problem.modalities
        arr = (_capi._dp * len(mods))(*[dptr(d) for d in mods])
        check(self.lib.jofc_set_problem(self.h, len(mods), problem.object_count(), arr,
                                        int(normalize)))
        self._problem_key = key
        self._keep = problem

    def upload_features(self, feats):
        """Delta_l = EDM(feats[l]) built on the device (reference arithmetic)."""
        feats = _f64(feats)
        m, n, p = feats.shape
        check(self.lib.jofc_set_problem_features(self.h, m, n, p, dptr(feats)))
        self._problem_key = ("features", id(feats), object())
        self._keep = None
        return ResidentProblem(self, m, n, self._problem_key)

    def problem_bytes(self):
        return int(self.lib.jofc_problem_bytes(self.h))

    def problem_pairs(self):
        return float(self.lib.jofc_problem_pairs(self.h))


_default_devices = {}


def _process_nccl():
    """Load torch (when installed) before the C library resolves NCCL: its
    bundled libnccl.so.2 is then the process's one NCCL (csrc/capi_nccl.cu
    reuses an already-loaded copy), instead of an older system copy that
    would later satisfy torch's own libnccl.so.2 dependency and break it."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def default_device(device=0):
    if device not in _default_devices:
        _default_devices[device] = Device(device)
    return _default_devices[device]


# --------------------------------------------------------- in-sample entry points
def _require_shapes(config, problem, spec):
    config = _f64(config)
    m, n = problem.modality_count(), problem.object_count()
    if config.ndim != 3:
        raise InvalidArgument("configuration blocks have inconsistent shapes")
    if config.shape[0] != m:
        raise InvalidArgument("configuration/problem modality count mismatch")
    if config.shape[1] != n:
        raise InvalidArgument("configuration/problem object count mismatch")
    return config


def raw_stress(config, problem, spec, parallel=False, device=None):
    """proj/src/stress.cpp:39-74 on the GPU."""
    config = _require_shapes(config, problem, spec)
    dev = device or default_device()
    dev.upload(problem)
    out = C.c_double()
    check(dev.lib.jofc_raw_stress(dev.h, C.byref(spec.c()), config.shape[2], dptr(config),
                                  C.byref(out)))
    return out.value


def guttman_step_fast(config, problem, spec, parallel=False, device=None):
    """proj/src/solver.cpp:154-161 on the GPU."""
    config = _require_shapes(config, problem, spec)
    dev = device or default_device()
    dev.upload(problem)
    out = np.empty_like(config)
    check(dev.lib.jofc_guttman_step(dev.h, C.byref(spec.c()), config.shape[2], dptr(config),
                                    dptr(out)))
    return out


def cmds(problem, modality, d, normalize=False, device=None):
    """proj/src/init.cpp:21-42 on the GPU; modality < 0 = the modality average."""
    dev = device or default_device()
    dev.upload(problem, normalize=normalize)
    out = np.empty((problem.object_count(), int(d)))
    check(dev.lib.jofc_cmds(dev.h, int(modality), int(d), dptr(out)))
    return out


def averaged_procrustes_init(problem, d, normalize=False, device=None):
    """proj/src/init.cpp:57-88 on the GPU (the reference's default init)."""
    dev = device or default_device()
    dev.upload(problem, normalize=normalize)
    out = np.empty((problem.modality_count(), problem.object_count(), int(d)))
    check(dev.lib.jofc_init_averaged_procrustes(dev.h, int(d), dptr(out)))
    return out


def symmetric_top_eigenpairs_subspace(s, k, device=None):
    """proj/include/jofc/linalg.hpp:29-35 with the S Q products on the GPU:
    (values[k], vectors[k, n]) by algebraic value, descending."""
    s = _f64(s)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise InvalidArgument("symmetric_top_eigenpairs_subspace: matrix not square")
    if float(np.max(np.abs(s - s.T), initial=0.0)) > 1e-9 * max(1.0, float(np.max(np.abs(s)))):
        raise InvalidArgument("symmetric_top_eigenpairs_subspace: matrix not symmetric")
    dev = device or default_device()
    n = s.shape[0]
    vals, vecs = np.empty(int(k)), np.empty((int(k), n))
    check(dev.lib.jofc_symmetric_top_eigenpairs_subspace(dev.h, n, dptr(s), int(k), dptr(vals),
                                                         dptr(vecs)))
    return vals, vecs


def imputed_omnibus_init(problem, d, dense_cap=4096, normalize=False, device=None):
    """proj/src/init.cpp:90-116 on the GPU (cmds of the imputed omnibus matrix)."""
    dev = device or default_device()
    dev.upload(problem, normalize=normalize)
    out = np.empty((problem.modality_count(), problem.object_count(), int(d)))
    check(dev.lib.jofc_init_imputed_cmds(dev.h, int(d), int(dense_cap), dptr(out)))
    return out


def fjofc_embed(problem, spec, options: SolveOptions, device=None):
    """proj/src/solver.cpp:223-236 (+ run_majorization :106-150) on the GPU.

    Every InitKind: provided, averaged_procrustes (the default) and
    imputed_cmds, the latter two computed on the GPU."""
    if options.dim < 1:
        raise InvalidArgument("SolveOptions: dim must be positive")
    if not options.eps > 0:
        raise InvalidArgument("SolveOptions: eps must be positive")
    m, n = problem.modality_count(), problem.object_count()
    dev = device or default_device()
    if options.init == InitKind.provided:
        if options.init_config is None:
            raise InvalidArgument("SolveOptions: provided init missing a configuration")
        x0 = _f64(options.init_config)
        if x0.shape != (m, n, options.dim):
            raise InvalidArgument("SolveOptions: provided init has the wrong shape")
        dev.upload(problem, normalize=options.normalize)
    elif options.init == InitKind.averaged_procrustes:
        x0 = averaged_procrustes_init(problem, options.dim, options.normalize, device=dev)
    else:
        x0 = imputed_omnibus_init(problem, options.dim, options.dense_cap, options.normalize,
                                  device=dev)
    T = int(options.max_iterations)
    if options.keep_config_trace:
        return _embed_with_config_trace(problem, spec, options, x0, dev)
    x = np.empty_like(x0)
    trace = np.empty(T + 1)
    steps = np.zeros(max(T, 1))
    its, conv = C.c_size_t(), C.c_int()
    check(dev.lib.jofc_fjofc_embed(dev.h, C.byref(spec.c()), options.dim, dptr(x0),
                                   float(options.eps), T, dptr(x), dptr(trace), C.byref(its),
                                   C.byref(conv), dptr(steps)))
    k = its.value
    pairs = stress_pair_count(m, n)
    tr = trace[: k + 1].tolist()
    return EmbeddingResult(config=x, stress_trace=tr,
                           normalized_stress_trace=[v / pairs for v in tr], iterations=k,
                           terminated=Termination.converged if conv.value else
                           Termination.max_iterations,
                           step_seconds=steps[:k].tolist())


def peer_lockstep_solve(devices, spec, x0, eps, max_iterations):
    """One fJOFC solve over peer-attached contexts of this process (test
    driver of the peer exchange: jofc_peer_lockstep_solve).  Returns, per
    rank, (X, stress trace, iterations, converged)."""
    x0 = _f64(x0)
    m, n, d = x0.shape
    world = len(devices)
    arr = (C.c_void_p * world)(*[dv.h.value for dv in devices])
    lib = devices[0].lib
    check(lib.jofc_peer_lockstep_solve(arr, world, C.byref(spec.c()), d, dptr(x0), float(eps),
                                       int(max_iterations)))
    out = []
    for dv in devices:
        x = np.empty_like(x0)
        trace = np.empty(int(max_iterations) + 1)
        its, conv = C.c_size_t(), C.c_int()
        check(lib.jofc_fetch_result(dv.h, dptr(x), dptr(trace), C.byref(its), C.byref(conv)))
        out.append((x, trace[: its.value + 1].copy(), its.value, bool(conv.value)))
    return out


def _embed_with_config_trace(problem, spec, options, x0, dev):
    """keep_config_trace: the reference loop (proj/src/solver.cpp:106-150)
    driven from the host, one GPU transform and one GPU stress per iteration,
    every iterate kept."""
    m, n = problem.modality_count(), problem.object_count()
    use = problem.normalized() if options.normalize and not isinstance(
        problem, ResidentProblem) else problem
    pairs = stress_pair_count(m, n)
    x = _f64(x0).copy()
    stress = raw_stress(x, use, spec, device=dev)
    if not math.isfinite(stress):
        raise NumericalError("embed: non-finite stress at the initial configuration")
    trace, configs, steps = [stress], [x.copy()], []
    term = Termination.max_iterations
    for it in range(int(options.max_iterations)):
        t0 = time.perf_counter()
        nxt = guttman_step_fast(x, use, spec, device=dev)
        steps.append(time.perf_counter() - t0)
        ns = raw_stress(nxt, use, spec, device=dev)
        if not math.isfinite(ns):
            raise NumericalError(f"embed: non-finite stress at iteration {it + 1}")
        x = nxt
        trace.append(ns)
        configs.append(x.copy())
        decrease = (stress - ns) / pairs
        stress = ns
        if decrease < options.eps:
            term = Termination.converged
            break
    k = len(trace) - 1
    return EmbeddingResult(config=x, stress_trace=trace,
                           normalized_stress_trace=[v / pairs for v in trace], iterations=k,
                           terminated=term, step_seconds=steps, config_trace=configs)


# ------------------------------------------------------------ out-of-sample
def _oos_shapes(y, x, deltas, w):
    x, deltas = _f64(x), _f64(deltas)
    if not w > 0:
        raise InvalidArgument("oos: w must be strictly positive")
    m, n, d = x.shape
    if deltas.shape[0] != m:
        raise InvalidArgument("oos: delta count does not match the configuration")
    if deltas.shape[-1] != n:
        raise InvalidArgument("oos: delta length does not match the configuration")
    if np.any(~(deltas >= 0)) or not np.all(np.isfinite(deltas)):
        raise InvalidArgument("oos: deltas must be finite and nonnegative")
    if y is not None:
        y = _f64(y)
        if y.shape != (m, d):
            raise InvalidArgument("oos: y must be m x d")
    return y, x, deltas


def oos_stress(y, x, deltas, w, device=None):
    """proj/src/oos.cpp:43-71 on the GPU."""
    y, x, deltas = _oos_shapes(y, x, deltas, w)
    m, n, d = x.shape
    dev = device or default_device()
    out = C.c_double()
    check(dev.lib.jofc_oos_stress(dev.h, m, n, d, dptr(y), dptr(x), dptr(deltas), float(w),
                                  C.byref(out)))
    return out.value


def oos_step_fast(y, x, deltas, w, device=None):
    """proj/src/oos.cpp:73-113 on the GPU."""
    y, x, deltas = _oos_shapes(y, x, deltas, w)
    m, n, d = x.shape
    dev = device or default_device()
    out = np.empty((m, d))
    check(dev.lib.jofc_oos_step(dev.h, m, n, d, dptr(y), dptr(x), dptr(deltas), float(w),
                                dptr(out)))
    return out


def oos_start(x, seed):
    """oos_embed's seeded start (proj/src/oos.cpp:189-198)."""
    x = _f64(x)
    m, n, d = x.shape
    out = np.empty((m, d))
    _capi.load().jofc_wl_oos_start(m, n, d, dptr(x), int(seed), dptr(out))
    return out


def oos_embed_batch(x, deltas, w, y0, options: OosOptions, fixed_iterations=False,
                    device=None):
    """k independent out-of-sample embeds in one GPU solve.

    deltas: (k, m, n), y0: (k, m, d).  Returns (y (k, m, d), traces
    (k, max_it+1; entries past each point's stop are unspecified),
    iterations (k,)).
    """
    x, deltas, y0 = _f64(x), _f64(deltas), _f64(y0)
    if not options.eps > 0:
        raise InvalidArgument("OosOptions: eps must be positive")
    k = y0.shape[0]
    _oos_shapes(None, x, deltas.reshape(-1, deltas.shape[-1])[: x.shape[0]], w)
    m, n, d = x.shape
    if deltas.shape != (k, m, n) or y0.shape != (k, m, d):
        raise InvalidArgument("oos: batch shapes disagree")
    if np.any(~(deltas >= 0)) or not np.all(np.isfinite(deltas)):
        raise InvalidArgument("oos: deltas must be finite and nonnegative")
    dev = device or default_device()
    T = int(options.max_iterations)
    y = np.empty_like(y0)
    traces = np.empty((k, T + 1))
    its = np.zeros(k, dtype=np.uint64)
    check(dev.lib.jofc_oos_batch(dev.h, k, m, n, d, dptr(x), dptr(deltas), float(w), dptr(y0),
                                 float(options.eps), T, int(bool(fixed_iterations)), dptr(y),
                                 dptr(traces), its.ctypes.data_as(C.POINTER(C.c_size_t))))
    return y, traces, its.astype(np.int64)


def oos_embed(x, deltas, w, options: OosOptions, seed, device=None):
    """proj/src/oos.cpp:180-229 on the GPU (one point)."""
    _, x, deltas = _oos_shapes(None, x, deltas, w)
    if not options.eps > 0:
        raise InvalidArgument("OosOptions: eps must be positive")
    y0 = oos_start(x, seed)
    y, traces, its = oos_embed_batch(x, deltas[None], w, y0[None], options, device=device)
    k = int(its[0])
    conv = k < options.max_iterations or (
        k >= 1 and (traces[0, k - 1] - traces[0, k]) /
        (x.shape[0] * x.shape[1] + 0.5 * x.shape[0] * (x.shape[0] - 1)) < options.eps)
    return OosResult(y=y[0], stress_trace=traces[0, : k + 1].tolist(), iterations=k,
                     terminated=Termination.converged if conv else Termination.max_iterations)
