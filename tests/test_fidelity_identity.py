"""The SMACOF identity behind the identity-form fidelity
(csrc/jofc_kernels.cuh, rho_decide), checked in numpy on the oracle's own
products (CPU, no GPU):

    sum_{i<j} (delta_ij - d_ij)^2 = A + S - 2 R,
    A = sum_{i<j} delta_ij^2,
    S = n sum_i |x_i - x_0|^2 - |sum_i (x_i - x_0)|^2   (= sum_{i<j} d_ij^2),
    R = sum_i x_i . P_i,  P = B(X) X                     (= sum_{i<j} delta_ij d_ij),

including coincident rows (d_ij = 0: b_ij = 0, the reference's guard).
"""
import numpy as np


def products(x, delta):
    diff = x[:, None, :] - x[None, :, :]
    d = np.sqrt((diff ** 2).sum(-1))
    with np.errstate(divide="ignore", invalid="ignore"):
        b = np.where(d > 0, delta / d, 0.0)
    np.fill_diagonal(b, 0.0)
    return (b[:, :, None] * diff).sum(1), d


def test_identity_on_random_and_coincident_rows():
    rng = np.random.default_rng(5)
    for n, dim, offset in [(40, 2, 0.0), (57, 5, 1e3), (33, 3, -7.0)]:
        x = rng.normal(size=(n, dim)) + offset
        x[7] = x[3]  # coincident rows
        f = rng.normal(size=(n, dim + 2))
        delta = np.sqrt(((f[:, None] - f[None]) ** 2).sum(-1))
        P, d = products(x, delta)
        iu = np.triu_indices(n, 1)
        direct = ((delta[iu] - d[iu]) ** 2).sum()
        A = (delta[iu] ** 2).sum()
        dx = x - x[0]
        S = n * (dx ** 2).sum() - (dx.sum(0) ** 2).sum()
        R = (x * P).sum()
        assert abs((A + S - 2 * R) - direct) <= 1e-9 * (A + S + 2 * abs(R))
        assert abs(S - (d[iu] ** 2).sum()) <= 1e-12 * S * max(1.0, offset ** 2)
