"""Pins for oracle/fem.py, oracle/transfer.py (closed forms, invariants, exact identities).

SURVEY 8(c) C.3 rows "element matrices, assembly", "N, N_p", "Transfers and coarse
operators", "Mass bounds".
"""
import numpy as np
import pytest

import synth
from oracle import fem, transfer
from oracle.problem import Problem
from oracle.inner import wathen_bounds


def test_1d_element_matrices_closed_form():
    """Printed 1-D Q2/Q1 element matrices (textbook closed forms)."""
    h = 0.37
    gp, gw = fem.gauss3()
    phi, dphi = fem.q2_basis_1d(gp)
    psi, dpsi = fem.q1_basis_1d(gp)
    M2 = h * np.einsum("q,iq,jq->ij", gw, phi, phi)
    K2 = (1 / h) * np.einsum("q,iq,jq->ij", gw, dphi, dphi)
    M1 = h * np.einsum("q,iq,jq->ij", gw, psi, psi)
    K1 = (1 / h) * np.einsum("q,iq,jq->ij", gw, dpsi, dpsi)
    Mx = h * np.einsum("q,iq,jq->ij", gw, psi, phi)
    Gx = np.einsum("q,iq,jq->ij", gw, psi, dphi)
    np.testing.assert_allclose(M2, h / 30 * np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]), atol=1e-15)
    np.testing.assert_allclose(K2, 1 / (3 * h) * np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]), atol=1e-13)
    np.testing.assert_allclose(M1, h / 6 * np.array([[2, 1], [1, 2]]), atol=1e-15)
    np.testing.assert_allclose(K1, 1 / h * np.array([[1, -1], [-1, 1]]), atol=1e-13)
    np.testing.assert_allclose(Mx, h / 12 * np.array([[2, 4, 0], [0, 4, 2]]), atol=1e-15)
    np.testing.assert_allclose(Gx, 1 / 6 * np.array([[-5, 4, 1], [-1, -4, 5]]), atol=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
def test_tensor_element_matrices_are_kronecker_products(dim):
    """d-dim element loop (genuine d-dim quadrature) equals the Kronecker form of 1-D matrices."""
    L1 = fem.Level(1, 1, 0.0, 1.0)
    Ld = fem.Level(dim, 1, 0.0, 1.0)
    m2, k2 = L1.mass_q2().toarray(), L1.stiff_q2().toarray()
    Mk, Kk = m2, k2
    for _ in range(dim - 1):                    # a new (slower) axis goes on the left
        Kk = np.kron(m2, Kk) + np.kron(k2, Mk)
        Mk = np.kron(m2, Mk)
    np.testing.assert_allclose(Ld.mass_q2().toarray(), Mk, atol=1e-15)
    np.testing.assert_allclose(Ld.stiff_q2().toarray(), Kk, atol=1e-13)


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_mass_sums_to_area_and_stiffness_kills_constants(dim, n):
    L = fem.Level(dim, n, -1.0, 1.0)
    vol = 2.0**dim
    assert abs(L.mass_q2().sum() - vol) < 1e-13
    assert abs(L.mass_q1().sum() - vol) < 1e-13
    assert np.abs(L.stiff_q2() @ np.ones(L.n_s)).max() < 1e-12
    assert np.abs(L.stiff_q1() @ np.ones(L.n_p)).max() < 1e-12


def _q2_xyz(L):
    g = L.lo + (L.hi - L.lo) * np.arange(L.n1q2) / (L.n1q2 - 1)
    n = np.arange(L.n_s)
    return [g[(n // L.n1q2**a) % L.n1q2] for a in range(L.dim)]


def _q1_xyz(L):
    g = L.lo + (L.hi - L.lo) * np.arange(L.n1q1) / (L.n1q1 - 1)
    n = np.arange(L.n_p)
    return [g[(n // L.n1q1**a) % L.n1q1] for a in range(L.dim)]


@pytest.mark.parametrize("dim", [2, 3])
def test_stiffness_of_quadratic_is_minus_laplacian_load(dim):
    """u = x^2 is in Q2: (K u)_i = -int phi_i Lap u = -2 (M 1)_i on interior rows (Green's formula)."""
    L = fem.Level(dim, 4 if dim == 2 else 2, 0.0, 1.0)
    X = _q2_xyz(L)
    u = X[0] ** 2 + 0.5 * X[dim - 1] ** 2
    lhs = (L.stiff_q2() @ u)[L.q2_interior()]
    rhs = -(2.0 + 1.0) * (L.mass_q2() @ np.ones(L.n_s))[L.q2_interior()]
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_divergence_closed_form_and_invariants(dim):
    """B is the NEGATIVE divergence: B (x^2, 0, ..) = -int psi_i 2x = -2 M_p x (x linear, in Q1)."""
    L = fem.Level(dim, 4 if dim == 2 else 2, 0.0, 1.0)
    B = L.div()
    X = _q2_xyz(L)
    v = np.zeros(dim * L.n_s)
    v[: L.n_s] = X[0] ** 2
    np.testing.assert_allclose(B @ v, -2.0 * (L.mass_q1() @ _q1_xyz(L)[0]), atol=1e-13)
    # B kills constant velocities; B^T 1_p = 0 on interior velocity rows (before pinning)
    for c in range(dim):
        v = np.zeros(dim * L.n_s)
        v[c * L.n_s:(c + 1) * L.n_s] = 1.0
        assert np.abs(B @ v).max() < 1e-13
    BT1 = B.T @ np.ones(L.n_p)
    Iv = L.q2_interior()
    assert np.abs(np.concatenate([BT1[c * L.n_s + Iv] for c in range(dim)])).max() < 1e-13


def test_divergence_full_rank_after_pin():
    prob = Problem(synth.small_config("t", 2, 4, 5))
    B = prob.fine.B.toarray()
    assert np.linalg.matrix_rank(B) == B.shape[0]            # n_p - 1 rows, full rank


def test_convection_skew_and_closed_form():
    """c3 wind: div w = 0 and w.n = 0 => N + N^T = 0 on the full grid; N x = M w_x (x linear)."""
    cfg = synth.small_config("t", 2, 4, 5, problem="oseen", lo=-1.0, hi=1.0)
    L = fem.Level(2, 4, -1.0, 1.0)
    w = synth.wind(cfg)
    N = L.conv_q2(w)
    assert abs(N + N.T).max() < 1e-14 * abs(N).max() * 100
    Np = L.conv_q1(w)
    assert abs(Np + Np.T).max() < 1e-14 * abs(Np).max() * 100
    x = _q2_xyz(L)[0]
    np.testing.assert_allclose(N @ x, L.mass_q2() @ w[0], atol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_transfer_interpolates_exactly(dim):
    """P reproduces any coarse Q2 (resp. Q1) function at the fine nodes (P 1 = 1, P x^2 = x^2)."""
    nc = 2
    Lc, Lf = fem.Level(dim, nc, 0.0, 1.0), fem.Level(dim, 2 * nc, 0.0, 1.0)
    P2 = transfer.prolongation(dim, nc, 2, np.arange(Lf.n_s), np.arange(Lc.n_s))
    P1 = transfer.prolongation(dim, nc, 1, np.arange(Lf.n_p), np.arange(Lc.n_p))
    Xc, Xf = _q2_xyz(Lc), _q2_xyz(Lf)
    f = lambda X: 1.0 + X[0] ** 2 * X[dim - 1] - 3 * X[dim - 1] ** 2
    np.testing.assert_allclose(P2 @ f(Xc), f(Xf), atol=1e-14)
    Yc, Yf = _q1_xyz(Lc), _q1_xyz(Lf)
    g = lambda X: 2.0 - X[0] + 0.5 * X[dim - 1]
    np.testing.assert_allclose(P1 @ g(Yc), g(Yf), atol=1e-14)


@pytest.mark.parametrize("dim,n,problem", [(2, 8, "stokes"), (2, 8, "oseen"), (3, 4, "stokes")])
def test_galerkin_equals_rediscretisation(dim, n, problem):
    """P^T A_f P = A_c for M, K, K_p, M_p (and N with the c3 wind) on the eliminated spaces."""
    lo, hi = (-1.0, 1.0) if problem == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("t", dim, n, 5, problem=problem, lo=lo, hi=hi)
    prob = Problem(cfg, synth.wind(cfg))
    for li in range(len(prob.levels) - 1):
        f, c = prob.levels[li], prob.levels[li + 1]
        P2, P1 = prob.P2[li], prob.P1[li]
        pairs = [(f.Ms, c.Ms, P2), (f.Ks, c.Ks, P2), (f.Mp, c.Mp, P1), (f.Kp, c.Kp, P1)]
        if problem == "oseen":
            pairs.append((f.Ns, c.Ns, P2))
        for Af, Ac, P in pairs:
            G = (P.T @ Af @ P).toarray()
            assert np.abs(G - Ac.toarray()).max() <= 1e-13 * np.abs(Ac.toarray()).max()


@pytest.mark.parametrize("dim", [2, 3])
def test_wathen_mass_bounds(dim):
    """eig(D^-1 M) inside the element bounds used by the Chebyshev iteration."""
    prob = Problem(synth.small_config("t", dim, 4 if dim == 2 else 2, 5))
    for A, space in ((prob.fine.Ms, "q2"), (prob.fine.Mp, "q1")):
        A = A.toarray()
        D = np.diag(A)
        ev = np.linalg.eigvalsh(A / np.sqrt(np.outer(D, D)))
        lo, hi = wathen_bounds(space, dim)
        assert ev.min() >= lo - 1e-12 and ev.max() <= hi + 1e-12


def test_dof_counts_match_baseline_json():
    """n_v, n_p stated in BASELINE.json configs c1, c2, c5 (full-grid counts, C.2 #5)."""
    for name, nv, npr in (("c1", 578, 81), ("c2", 33282, 4225), ("c5", 823875, 35937)):
        c = synth.CONFIGS[name]
        assert (c.n_v, c.n_p) == (nv, npr)
    assert synth.CONFIGS["c2"].n_dofs == 4725882          # = paper's 4.73e6 row (h_f, n_t = 63)


@pytest.mark.parametrize("dim", [2, 3])
def test_pressure_convection_closed_form(dim):
    """N_p (C.2 #9) against a closed form: for a bilinear (Q1) wind w and the coordinate functions
    x_a (in Q1), int psi_i (w . grad x_a) = int psi_i w_a, i.e. N_p x_a = M_p w_a (exact); N_p 1 = 0.
    Pins the scale, sign and quadrature of conv_q1 (a dropped h-power or a factor on N_p fails)."""
    n = 4 if dim == 2 else 2
    L = fem.Level(dim, n, -1.0, 1.0)
    X2, X1 = _q2_xyz(L), _q1_xyz(L)
    lin = lambda X, a: 0.3 + 0.7 * X[0] - 0.4 * X[dim - 1] + (0.9 + a) * X[0] * X[dim - 1]
    w = np.stack([lin(X2, a) for a in range(dim)])              # Q2 nodal values of a Q1 field
    wp = np.stack([lin(X1, a) for a in range(dim)])             # the same field at the Q1 nodes
    Np, Mp = L.conv_q1(w), L.mass_q1()
    for a in range(dim):
        np.testing.assert_allclose(Np @ X1[a], Mp @ wp[a], atol=1e-13)
    assert np.abs(Np @ np.ones(L.n_p)).max() < 1e-13
    # Galerkin identity for the pressure convection on the eliminated spaces (coarse wind = injection)
    Lc = fem.Level(dim, n // 2, -1.0, 1.0)
    wc = fem.inject_wind(w, dim, n)
    P1 = transfer.prolongation(dim, n // 2, 1, L.q1_unknowns(), Lc.q1_unknowns())
    Nf = fem.restrict(Np, L.q1_unknowns(), L.q1_unknowns())
    Nc = fem.restrict(Lc.conv_q1(wc), Lc.q1_unknowns(), Lc.q1_unknowns())
    assert np.abs((P1.T @ Nf @ P1 - Nc).toarray()).max() <= 1e-13 * np.abs(Nc.toarray()).max()
