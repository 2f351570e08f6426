"""The reference arm's inputs (oracle/workloads_ref.py: the recipes drawn
through the reference's own Rng and euclidean_distance_matrix, without the
product library) are bit-identical to the product's workloads.make."""
import os

import numpy as np
import pytest

from oracle import workloads_ref
from oracle.oracle import PORT_SO, REF_SO, Port, Reference
from paper_1502_03391_b200 import workloads

IMPLS = ["port"] + (["reference"] if os.path.exists(REF_SO) else [])


def impl_of(name):
    return Reference(REF_SO) if name == "reference" else Port(PORT_SO)


@pytest.mark.parametrize("name", IMPLS)
@pytest.mark.parametrize("cfg,n", [(1, 300), (2, 257), (3, 190), (4, 130), (5, 150)])
def test_reference_inputs_bit_identical(name, cfg, n):
    impl = impl_of(name)
    ours = workloads.make(cfg, n=n)
    ref = workloads_ref.make(cfg, n=n, impl=impl)
    assert (ref.m, ref.n, ref.d, ref.iterations) == (ours.m, ours.n, ours.d, ours.iterations)
    assert ref.w == ours.w and ref.general_weights == ours.general_weights
    assert np.array_equal(ref.features, ours.features)
    assert np.array_equal(ref.x0(), ours.x0())
    assert np.array_equal(ref.dense_delta(), ours.dense_delta())


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_shapes_agree(cfg):
    s = workloads.shape(cfg)
    m, n, d, p, its, w, gen, k = workloads_ref.SHAPES[cfg]
    assert (s.m, s.n, s.d, s.p, s.iterations, s.w, bool(s.general_weights), s.oos_points) == \
        (m, n, d, p, its, w, gen, k)
