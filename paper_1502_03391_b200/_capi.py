"""ctypes binding of libjofc_gpu.so (the C ABI declared in include/jofc_gpu.h).

There is no fallback: if the CUDA library is missing or cannot be loaded,
importing the product API raises.  Status codes map to the exception types
the reference throws (std::invalid_argument -> InvalidArgument(ValueError),
jofc::NumericalError -> NumericalError(RuntimeError)).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libjofc_gpu.so")
HEADER_DIR = os.path.join(os.path.dirname(HERE), "include")

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p


class JofcError(Exception):
    code = -1


class InvalidArgument(JofcError, ValueError):
    code = 1


class NumericalError(JofcError, RuntimeError):
    code = 2


class CudaError(JofcError, RuntimeError):
    code = 3


class CommError(JofcError, RuntimeError):
    code = 4


_ERRORS = {1: InvalidArgument, 2: NumericalError, 3: CudaError, 4: CommError}


class Weights(C.Structure):
    _fields_ = [("kind", C.c_int), ("w", C.c_double), ("general", _dp), ("within", _dp),
                ("scale", C.c_double)]


class WorkloadShape(C.Structure):
    _fields_ = [("m", _sz), ("n", _sz), ("d", _sz), ("p", _sz), ("iterations", _sz),
                ("w", C.c_double), ("general_weights", C.c_int), ("oos_points", _sz)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, _dp, _sz, _vp, _vp)

# name -> (restype, argtypes)
_SIGS = {
    "jofc_last_error": (C.c_char_p, []),
    "jofc_version": (C.c_int, []),
    "jofc_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "jofc_ctx_destroy": (C.c_int, [_vp]),
    "jofc_ctx_stream": (_vp, [_vp]),
    "jofc_set_shard": (C.c_int, [_vp, C.c_int, C.c_int]),
    "jofc_set_allreduce": (C.c_int, [_vp, ALLREDUCE_FN, _vp]),
    "jofc_set_problem": (C.c_int, [_vp, _sz, _sz, C.POINTER(_dp), C.c_int]),
    "jofc_set_problem_features": (C.c_int, [_vp, _sz, _sz, _sz, _dp]),
    "jofc_load_problem_files": (C.c_int, [_vp, _sz, C.POINTER(C.c_char_p), C.c_int]),
    "jofc_problem_shape": (C.c_int, [_vp, _szp, _szp]),
    "jofc_problem_bytes": (_sz, [_vp]),
    "jofc_problem_pairs": (C.c_double, [_vp]),
    "jofc_raw_stress": (C.c_int, [_vp, C.POINTER(Weights), _sz, _dp, _dp]),
    "jofc_guttman_step": (C.c_int, [_vp, C.POINTER(Weights), _sz, _dp, _dp]),
    "jofc_fjofc_embed": (C.c_int, [_vp, C.POINTER(Weights), _sz, _dp, C.c_double, _sz, _dp, _dp,
                                   _szp, C.POINTER(C.c_int), _dp]),
    "jofc_fjofc_enqueue": (C.c_int, [_vp, C.POINTER(Weights), _sz, _dp, C.c_double, _sz]),
    "jofc_fetch_result": (C.c_int, [_vp, _dp, _dp, _szp, C.POINTER(C.c_int)]),
    "jofc_launch_count": (C.c_uint64, [_vp]),
    "jofc_stress_evaluations": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "jofc_profile": (C.c_int, [_vp, C.c_int]),
    "jofc_set_fidelity_form": (C.c_int, [_vp, C.c_int]),
    "jofc_set_oos_route": (C.c_int, [_vp, C.c_int]),
    "jofc_profile_read": (C.c_int, [_vp, _dp, C.POINTER(C.c_uint64)]),
    "jofc_set_exchange_buffer": (C.c_int, [_vp, _vp, _sz]),
    "jofc_exchange_count": (_sz, [_vp, _sz]),
    "jofc_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "jofc_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "jofc_nccl_init": (C.c_int, [_vp, C.c_char_p, C.c_int, C.c_int]),
    "jofc_nccl_release": (C.c_int, [_vp]),
    "jofc_peer_export": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "jofc_peer_attach": (C.c_int, [_vp, C.c_int, C.c_int, C.c_char_p]),
    "jofc_peer_attach_pointers": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "jofc_peer_detach": (C.c_int, [_vp]),
    "jofc_peer_address": (_vp, [_vp, C.c_int]),
    "jofc_peer_lockstep_solve": (C.c_int, [C.POINTER(_vp), C.c_int, C.POINTER(Weights), _sz, _dp,
                                           C.c_double, _sz]),
    "jofc_oos_stress": (C.c_int, [_vp, _sz, _sz, _sz, _dp, _dp, _dp, C.c_double, _dp]),
    "jofc_oos_step": (C.c_int, [_vp, _sz, _sz, _sz, _dp, _dp, _dp, C.c_double, _dp]),
    "jofc_oos_batch": (C.c_int, [_vp, _sz, _sz, _sz, _sz, _dp, _dp, C.c_double, _dp, C.c_double,
                                 _sz, C.c_int, _dp, _dp, _szp]),
    "jofc_cmds": (C.c_int, [_vp, C.c_int, _sz, _dp]),
    "jofc_symmetric_top_eigenpairs_subspace": (C.c_int, [_vp, _sz, _dp, _sz, _dp, _dp]),
    "jofc_init_imputed_cmds": (C.c_int, [_vp, _sz, _sz, _dp]),
    "jofc_init_averaged_procrustes": (C.c_int, [_vp, _sz, _dp]),
    # workload generators (include/jofc_workloads.h)
    "jofc_wl_shape": (C.c_int, [C.c_int, C.POINTER(WorkloadShape)]),
    "jofc_wl_features": (C.c_int, [C.c_int, C.c_uint64, _sz, _dp]),
    "jofc_wl_normals": (None, [C.c_uint64, _sz, C.c_double, _dp]),
    "jofc_wl_distance_matrix": (None, [_sz, _sz, _dp, _dp]),
    "jofc_wl_oos_deltas": (None, [_sz, _sz, _sz, _sz, _dp, _dp]),
    "jofc_wl_oos_start": (None, [_sz, _sz, _sz, _dp, C.c_uint64, _dp]),
}

_lib = None


def load():
    """Load libjofc_gpu.so (once).  Raises if it is absent: no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    # JOFC_GPU_LIB: an alternative in-tree build of the same C ABI (kernel
    # experiments, scripts/diag_pass.py); the default is the shipped library
    path = os.environ.get("JOFC_GPU_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; build it with `make` "
                          "(or __graft_entry__.build()).  There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        if path != LIB_PATH and not hasattr(lib, name):
            continue  # (an older experiment build: A/B timing only)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc:
        msg = load().jofc_last_error().decode()
        raise _ERRORS.get(rc, JofcError)(msg)


def header_symbols(header="jofc_gpu.h"):
    """Function names declared in include/<header> (for the export test)."""
    text = open(os.path.join(HEADER_DIR, header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(jofc_[a-z0-9_]+)\s*\(", text)) - {"jofc_allreduce_fn"})


def dptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None
