"""The shared host algebra (csrc/host_linalg.cpp) on CPU: Jacobi eigenpairs,
one-sided Jacobi SVD, Gram-Schmidt, Gauss-Jordan -- against numpy and, where
the reference's contract fixes the arithmetic (W^-1 of general weights), the
reference itself."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1502_03391_b200", "csrc")


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("hla") / "libhla.so")
    subprocess.run(["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-I" + CSRC, "-o", out,
                    os.path.join(CSRC, "host_linalg.cpp"),
                    os.path.join(ROOT, "tests", "cpp", "host_linalg_shim.cpp")], check=True)
    return C.CDLL(out)


def P(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@pytest.mark.parametrize("n", [1, 2, 5, 17, 60])
def test_jacobi_eigh(lib, n):
    rng = np.random.default_rng(n)
    a = rng.normal(size=(n, n))
    a = a + a.T
    w, v = np.empty(n), np.empty((n, n))
    assert lib.t_jacobi(P(a), C.c_size_t(n), P(w), P(v)) == 1
    ref = np.linalg.eigvalsh(a)
    assert np.allclose(np.sort(w), ref, rtol=0, atol=1e-12 * max(1, np.abs(ref).max()))
    assert np.allclose(a @ v, v * w, atol=1e-11 * max(1, np.abs(ref).max()))
    assert np.allclose(v.T @ v, np.eye(n), atol=1e-13)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_svd(lib, n):
    rng = np.random.default_rng(10 + n)
    a = rng.normal(size=(n, n))
    u, s, v = np.empty((n, n)), np.empty(n), np.empty((n, n))
    lib.t_svd(P(a), C.c_size_t(n), P(u), P(s), P(v))
    assert np.allclose(u @ np.diag(s) @ v.T, a, atol=1e-12)
    assert np.allclose(u.T @ u, np.eye(n), atol=1e-12)
    assert np.allclose(v.T @ v, np.eye(n), atol=1e-12)
    assert np.all(np.diff(s) <= 0)
    assert np.allclose(s, np.linalg.svd(a, compute_uv=False), atol=1e-12)


def test_svd_rank_deficient_completion(lib):
    a = np.outer(np.arange(1, 4.0), np.arange(2, 5.0))
    u, s, v = np.empty((3, 3)), np.empty(3), np.empty((3, 3))
    lib.t_svd(P(a), C.c_size_t(3), P(u), P(s), P(v))
    assert np.allclose(u.T @ u, np.eye(3), atol=1e-12)
    assert np.allclose(u @ np.diag(s) @ v.T, a, atol=1e-12)


def test_orthonormalize_with_vanished_column(lib):
    q = np.random.default_rng(4).normal(size=(12, 4))
    q[:, 2] = 2.0 * q[:, 0]  # dependent: replaced by a coordinate direction
    lib.t_orth(P(q), C.c_size_t(12), C.c_size_t(4))
    assert np.allclose(q.T @ q, np.eye(4), atol=1e-12)


def test_gauss_jordan(lib):
    a = np.random.default_rng(7).normal(size=(6, 6))
    inv = np.empty((6, 6))
    assert lib.t_inv(P(a), C.c_size_t(6), P(inv)) == 1
    assert np.allclose(a @ inv, np.eye(6), atol=1e-12)
    sing = np.ones((3, 3))
    assert lib.t_inv(P(sing), C.c_size_t(3), P(np.empty((3, 3)))) == 0


def test_orient(lib):
    x = np.array([0.1, -0.9, 0.9, 0.3])
    lib.t_orient(P(x), C.c_size_t(4))
    assert list(x) == [-0.1, 0.9, -0.9, -0.3]  # first largest-magnitude entry positive
