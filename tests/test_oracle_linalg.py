"""Pins of the oracle's POD (Eq. 9) and gappy least squares (Eq. 8).

Pinned against closed forms (already-orthogonal columns, rank one, Eckart-Young,
Phi^T X = S V^T, planted spectra) and against numpy.linalg (LAPACK) on small
problems -- a library routine the oracle does not use.
"""
import numpy as np
import pytest


def _principal_sines(A, B):
    Qa, _ = np.linalg.qr(A)
    Qb, _ = np.linalg.qr(B)
    # sines of the principal angles, computed without the 1 - cos^2 cancellation
    return np.linalg.svd(Qb - Qa @ (Qa.T @ Qb), compute_uv=False)


def test_svd_matches_lapack(orc, inputs):
    for (m, n, seed) in [(30, 6, 1), (200, 12, 2), (5, 9, 3)]:
        X = inputs.random_matrix(seed, m, n)
        U, S, V = orc.svd(X)
        Sl = np.linalg.svd(X, compute_uv=False)
        k = min(m, n)
        np.testing.assert_allclose(S[:k], Sl, rtol=1e-13)
        np.testing.assert_allclose(U[:, :k] @ np.diag(S[:k]) @ V[:, :k].T, X, atol=1e-13)
        np.testing.assert_allclose(V.T @ V, np.eye(n), atol=1e-13)
        # sign convention: largest-|.| entry of each right singular vector positive
        for j in range(k):
            i = np.argmax(np.abs(V[:, j]))
            assert V[i, j] > 0


def test_pod_orthonormal_and_reff(orc, inputs):
    X = inputs.random_matrix(4, 500, 10)
    Phi, S, V, reff = orc.pod(X, 6)
    assert reff == 6
    assert np.max(np.abs(Phi.T @ Phi - np.eye(6))) <= 1e-12


def test_pod_orthogonal_columns(orc):
    """orthogonal columns with norms 3 > 2 > 1 -> the first r normalised columns."""
    X = np.zeros((7, 3))
    X[1, 0], X[4, 1], X[6, 2] = 3.0, -2.0, 1.0
    Phi, S, V, reff = orc.pod(X, 2)
    np.testing.assert_allclose(S, [3, 2, 1], rtol=1e-15)
    np.testing.assert_allclose(np.abs(Phi[:, 0]), np.eye(7)[1], atol=1e-15)
    np.testing.assert_allclose(np.abs(Phi[:, 1]), np.eye(7)[4], atol=1e-15)


def test_pod_rank_one(orc):
    """a b^T -> a/|a|; r_eff = 1 (zero trailing singular values are cut, A15)."""
    a = np.array([1.0, -2.0, 0.5, 3.0])
    b = np.array([0.3, 1.0, -0.7])
    Phi, S, V, reff = orc.pod(np.outer(a, b), 3)
    assert reff == 1
    np.testing.assert_allclose(np.abs(Phi[:, 0]), np.abs(a) / np.linalg.norm(a), rtol=1e-14)


def test_pod_vs_lapack_subspace_and_eckart_young(orc, inputs):
    X = inputs.random_matrix(5, 30, 6)
    Phi, S, V, reff = orc.pod(X, 4)
    Ul, Sl, Vl = np.linalg.svd(X, full_matrices=False)
    assert np.max(_principal_sines(Phi, Ul[:, :4])) < 1e-12
    resid = X - Phi @ (Phi.T @ X)
    assert abs(np.sum(resid ** 2) - np.sum(Sl[4:] ** 2)) <= 1e-12 * np.sum(Sl ** 2)
    # Phi^T X = S_r V_r^T
    np.testing.assert_allclose(Phi.T @ X, np.diag(S[:4]) @ V[:, :4].T, atol=1e-13)


def test_pod_planted_spectrum_and_cutoff(orc, inputs):
    m, w = 400, 8
    Q1, _ = np.linalg.qr(inputs.random_matrix(6, m, w))
    Q2, _ = np.linalg.qr(inputs.random_matrix(7, w, w))
    sig = np.array([10.0, 5.0, 2.0, 1.0, 0.5, 2e-4, 1e-5, 1e-7])
    X = Q1 @ np.diag(sig) @ Q2.T
    Phi, S, V, reff = orc.pod(X, 8, cut=1e-8)
    np.testing.assert_allclose(S, sig, rtol=1e-9, atol=1e-14)
    assert reff == 5  # (0.5/10)^2 = 2.5e-3 kept; (2e-4/10)^2 = 4e-10 < 1e-8 cut


def test_pod_cutoff_rule_exact(orc, inputs):
    """r_eff = #{i < r: S_i^2 >= cut S_0^2} (reading A15)."""
    m, w = 300, 6
    Q1, _ = np.linalg.qr(inputs.random_matrix(8, m, w))
    Q2, _ = np.linalg.qr(inputs.random_matrix(9, w, w))
    sig = np.array([1.0, 0.5, 1e-3, 2e-4, 5e-5, 1e-6])  # squares: 1, .25, 1e-6, 4e-8, 2.5e-9, 1e-12
    X = Q1 @ np.diag(sig) @ Q2.T
    assert orc.pod(X, 6, cut=1e-8)[3] == 4
    assert orc.pod(X, 3, cut=1e-8)[3] == 3
    assert orc.pod(X, 6, cut=1e-5)[3] == 2  # 1e-6 < 1e-5


def test_lsq_in_subspace_exact(orc, inputs):
    """v - psi = Phi e_1 -> y = e_1; in-subspace data recovered exactly."""
    Phi, _ = np.linalg.qr(inputs.random_matrix(10, 60, 5))
    rows = np.arange(0, 60, 3)
    for i in range(5):
        b = Phi[rows, i]
        y, rank = orc.lsq(Phi[rows], b)
        np.testing.assert_allclose(y, np.eye(5)[i], atol=1e-12)
        assert rank == 5


def test_lsq_full_sampling_is_projection(orc, inputs):
    """P = all rows, Phi orthonormal -> y = Phi^T (v - psi)."""
    Phi, _ = np.linalg.qr(inputs.random_matrix(11, 80, 6))
    v = inputs.random_values(12, 80, -1, 1)
    y, _ = orc.lsq(Phi, v)
    np.testing.assert_allclose(y, Phi.T @ v, atol=1e-13)


@pytest.mark.parametrize("m,n", [(50, 7), (7, 7), (4, 9)])
def test_lsq_vs_lapack_min_norm(orc, inputs, m, n):
    A = inputs.random_matrix(13 + m, m, n)
    b = inputs.random_values(14 + m, m, -1, 1)
    x, rank = orc.lsq(A, b)
    np.testing.assert_allclose(x, np.linalg.pinv(A) @ b, atol=1e-11)
    assert rank == min(m, n)


def test_lsq_rank_deficient_cutoff(orc, inputs):
    """A13: minimum-norm solution discarding sigma^2 < 1e-12 sigma_1^2."""
    B = inputs.random_matrix(20, 40, 3)
    A = np.hstack([B, B[:, :1] * 2.0 + 1e-9 * inputs.random_matrix(21, 40, 1)])
    b = inputs.random_values(22, 40, -1, 1)
    x, rank = orc.lsq(A, b, cut=1e-12)
    assert rank == 3
    U, S, Vt = np.linalg.svd(A, full_matrices=False)
    keep = S ** 2 >= 1e-12 * S[0] ** 2
    ref = Vt[keep].T @ ((U[:, keep].T @ b) / S[keep])
    np.testing.assert_allclose(x, ref, atol=1e-10)


def test_lsq_empty(orc):
    x, rank = orc.lsq(np.zeros((0, 3)), np.zeros(0))
    assert rank == 0 and np.all(x == 0)


def test_gram_matches_definition(orc, inputs):
    """C = (S - rho)^T (S - rho) (snapshot Gram, P:634 remark) vs LAPACK-free brute force."""
    S = inputs.random_matrix(30, 7, 200).copy()  # 7 columns of 200 rows
    rho = inputs.random_values(31, 200, 0.5, 1.5)
    C = orc.gram(S, rho)
    ref = np.array([[float(np.sum((S[i] - rho) * (S[j] - rho))) for j in range(7)] for i in range(7)])
    np.testing.assert_allclose(C, ref, rtol=1e-13)
    assert np.array_equal(C, C.T)


def test_project_exact_integers_and_coefficients(orc, inputs):
    """orc_project (C = Phi^T S, the config-5 projection op): (i) small-integer Phi and S give the
    exact integer product (every partial sum is an integer < 2^53), checked against int64
    arithmetic, with m != ncol so a transposed operand or swapped index fails; (ii) for
    orthonormal Phi and S = Phi Y + (I - Phi Phi^T) Z the projection returns Y (the POD
    coefficients) to rounding."""
    rng = np.random.default_rng(12)
    D, m, ncol = 257, 5, 7
    Pi = rng.integers(-9, 10, size=(m, D))
    Si = rng.integers(-9, 10, size=(ncol, D))
    C = orc.project(Pi.astype(np.float64), Si.astype(np.float64))
    assert C.shape == (m, ncol)
    assert np.array_equal(C, (Pi @ Si.T).astype(np.float64))
    Q, _ = np.linalg.qr(inputs.random_matrix(13, 2000, 6))
    Y = inputs.random_matrix(14, 6, 9)
    Z = inputs.random_matrix(15, 2000, 9)
    S = Q @ Y + (Z - Q @ (Q.T @ Z))
    C = orc.project(Q.T.copy(), S.T.copy())
    np.testing.assert_allclose(C, Y, rtol=0, atol=1e-13 * np.abs(Y).max())
