"""B200-native fJOFC Guttman loop (arXiv 1502.03391) behind the reference's API.

The product is libjofc_gpu.so (C ABI, include/jofc_gpu.h) with hand-written
sm_100a kernels, plus the C++ drop-in libjofc.so (include/jofc/*.hpp).  This
Python package is the host-side mirror used by the tests and bench.py.
"""
from .api import (  # noqa: F401
    Device,
    EmbeddingResult,
    InitKind,
    OmnibusProblem,
    OosOptions,
    OosResult,
    ResidentProblem,
    SolveOptions,
    Termination,
    WeightSpec,
    averaged_procrustes_init,
    cmds,
    default_device,
    fjofc_embed,
    guttman_step_fast,
    imputed_omnibus_init,
    load_dissimilarities,
    oos_embed,
    oos_embed_batch,
    oos_start,
    oos_step_fast,
    oos_stress,
    peer_lockstep_solve,
    raw_stress,
    stress_pair_count,
    symmetric_top_eigenpairs_subspace,
)
from ._capi import CommError, CudaError, InvalidArgument, NumericalError  # noqa: F401
