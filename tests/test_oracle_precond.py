"""Pins for oracle/inner.py and oracle/precond.py.

SURVEY 8(c) C.3 rows: T-factorisation and c1/c2, Stokes Schur, P-hat bound,
Pearson-Wathen, Algorithm 3 structure, Uzawa, Chebyshev, MG, SOR,
FFT-diagonalised circulant solve, conjugate symmetry, Theorems 3.3/3.5.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import precond, timeops
from oracle.inner import Chebyshev, MultiColourSOR, Multigrid, wathen_bounds
from oracle.problem import Problem
import dense_ops
from dense_ops import DenseSolve


def make(problem="stokes", dim=2, n=4, n_t=6, beta=1e-2, nu=0.05):
    lo, hi = (-1.0, 1.0) if problem == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("t", dim, n, n_t, problem=problem, lo=lo, hi=hi, beta=beta, nu=nu)
    return Problem(cfg, synth.wind(cfg))


# ------------------------------------------------------------------ c1/c2 and T factorisation
@pytest.mark.parametrize("k", [0, 1, 2, 4])
def test_G_equals_Tl_Z_Tr_with_squared_reading(k):
    """G_j = T_l Z_j T_r holds with c1 = d_r / sqrt(tau^2/beta + d_c^2) (C.2 #1) ..."""
    prob = make(n=2, n_t=6)
    d = timeops.spectrum(prob.n_b)[k]
    c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
    Tl, Tr = dense_ops.T_matrices(prob, d, c2)
    G = dense_ops.G_block(prob, d)
    np.testing.assert_allclose(Tl @ dense_ops.Z_block(prob, c1, c2) @ Tr, G, atol=1e-13 * np.abs(G).max())


def test_G_factorisation_fails_with_printed_c1():
    """... and NOT with the exponent as printed at P:402 (the garble)."""
    prob = make(n=2, n_t=6)
    d = timeops.spectrum(prob.n_b)[1]
    _, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
    c1_printed = d.real / np.sqrt(prob.tau**2 / prob.beta + d.imag)
    Tl, Tr = dense_ops.T_matrices(prob, d, c2)
    G = dense_ops.G_block(prob, d)
    assert np.abs(Tl @ dense_ops.Z_block(prob, c1_printed, c2) @ Tr - G).max() > 1e-4 * np.abs(G).max()


def test_pointwise_T_inverses_equal_dense_solves():
    prob = make(n=2, n_t=6)
    rng = np.random.default_rng(2)
    nv, npu = prob.dim * prob.fine.nI, prob.fine.npu
    for k in (0, 2, 4):
        d = timeops.spectrum(prob.n_b)[k]
        _, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
        Tl, Tr = dense_ops.T_matrices(prob, d, c2)
        r = rng.standard_normal(2 * nv + 2 * npu) + 1j * rng.standard_normal(2 * nv + 2 * npu)
        parts = np.split(r, [nv, 2 * nv, 2 * nv + npu])
        s = precond.OraclePreconditioner.tl_inv(d, prob.tau, prob.beta, *parts)
        np.testing.assert_allclose(np.concatenate(s), np.linalg.solve(Tl, r), atol=1e-12)
        y = precond.OraclePreconditioner.tr_inv(d, prob.tau, prob.beta, *parts)
        np.testing.assert_allclose(np.concatenate(y), np.linalg.solve(Tr, r), atol=1e-12)


# ------------------------------------------------------------------ bounds from the paper
def test_P_hat_bound():
    """|lambda(P_hat_j^{-1} Z_j)| in [1/sqrt(12), (1+sqrt 5)/2]; P_hat SPD."""
    prob = make(n=2, n_t=8, beta=1e-2, nu=0.01)
    s = dense_ops.spatial(prob)
    for d in timeops.spectrum(prob.n_b):
        c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
        W = (1 + c1) * s["M"] + c2 * s["L"]
        S = s["B"] @ np.linalg.solve(W, s["B"].T)
        Ph = sla.block_diag(W, W, S, S)
        assert np.linalg.eigvalsh(Ph).min() > 0
        lam = np.abs(np.linalg.eigvals(np.linalg.solve(Ph, dense_ops.Z_block(prob, c1, c2))))
        assert lam.min() >= 1 / np.sqrt(12) - 1e-8 and lam.max() <= (1 + np.sqrt(5)) / 2 + 1e-8


def test_pearson_wathen_bound_complex_d():
    """lambda(S_hat^{-1} S) in [1/2, 1] for the Oseen (1,1)-block with complex d_j."""
    prob = make("oseen", n=2, n_t=8, beta=1e-3, nu=0.05)
    s = dense_ops.spatial(prob)
    M, L, tau, beta = s["M"], s["L"], prob.tau, prob.beta
    for d in timeops.spectrum(prob.n_b):
        G21 = d * M + tau * L
        S = (tau / beta) * M + (1 / tau) * G21 @ np.linalg.solve(M, G21.conj().T)
        Q = G21 + (tau / np.sqrt(beta)) * M
        Sh = (1 / tau) * Q @ np.linalg.solve(M, Q.conj().T)
        lam = np.linalg.eigvals(np.linalg.solve(Sh, S))
        assert np.abs(lam.imag).max() < 1e-8
        assert lam.real.min() >= 0.5 - 1e-8 and lam.real.max() <= 1 + 1e-8


# ------------------------------------------------------------------ Stokes block with exact inner solves
class ExactStokes(precond.OraclePreconditioner):
    def W_solver(self, k):
        s = dense_ops.spatial(self.prob)
        c1, c2 = timeops.stokes_constants(self.d[k], self.prob.tau, self.prob.beta)
        return DenseSolve(((1 + c1) * self.prob.fine.Ms + c2 * self.prob.nu * self.prob.fine.Ks))

    def Kp_solver(self):
        return DenseSolve(self.prob.fine.Kp)

    def Mp_solver(self):
        return DenseSolve(self.prob.fine.Mp)


def test_stokes_block_with_exact_inner_solves_equals_dense_formula():
    """stokes_block = T_r^{-1} blkdiag(W, W, S_hat, S_hat)^{-1} T_l^{-1} with
    S_hat = M_p ((1+c1) M_p + c2 L_p)^{-1} K_p, L_p = nu K_p."""
    prob = make(n=4, n_t=6)
    pc = ExactStokes(prob)
    s = dense_ops.spatial(prob)
    rng = np.random.default_rng(4)
    nv, npu = prob.dim * prob.fine.nI, prob.fine.npu
    for k in range(prob.n_b):
        d = pc.d[k]
        c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
        W = (1 + c1) * s["M"] + c2 * s["L"]
        Sh = s["Mp"] @ np.linalg.solve((1 + c1) * s["Mp"] + c2 * prob.nu * s["Kp"], s["Kp"])
        Tl, Tr = dense_ops.T_matrices(prob, d, c2)
        P = Tl @ sla.block_diag(W, W, Sh, Sh) @ Tr
        r = rng.standard_normal(2 * nv + 2 * npu) + 1j * rng.standard_normal(2 * nv + 2 * npu)
        R1, R2, R3, R4 = np.split(r, [nv, 2 * nv, 2 * nv + npu])
        y = pc.stokes_block(k, R1.reshape(prob.dim, -1), R2.reshape(prob.dim, -1), R3, R4)
        y = np.concatenate([y[0].reshape(-1), y[1].reshape(-1), y[2], y[3]])
        np.testing.assert_allclose(y, np.linalg.solve(P, r), rtol=0, atol=1e-9 * np.abs(y).max())


class ExactBlocks(precond.OraclePreconditioner):
    """Algorithm 1 with exact dense G_k^{-1} blocks."""

    def block(self, k, R1, R2, R3, R4):
        G = dense_ops.G_block(self.prob, self.d[k])
        nv = R1.size
        r = np.concatenate([R1.reshape(-1), R2.reshape(-1), R3, R4])
        y = np.linalg.solve(G, r)
        return (y[:nv].reshape(R1.shape), y[nv:2 * nv].reshape(R2.shape),
                y[2 * nv:2 * nv + R3.size], y[2 * nv + R3.size:])


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_algorithm1_with_exact_blocks_is_dense_circulant_solve(problem):
    """FFT -> exact G_k^{-1} -> IFFT equals the dense solve with P_C (1.3e-15)."""
    prob = make(problem, n=2, n_t=7)
    pc = ExactBlocks(prob)
    PC = dense_ops.dense_all_at_once(prob, timeops.circulant_C(prob.n_b))
    r = synth.probe_vector(prob.cfg)
    z, zi = pc.apply(r, return_imag=True)
    from oracle import kkt
    V, P = prob.to_reduced(r)
    zd = np.linalg.solve(PC, kkt.reduced_vector(prob, V, P))
    Vz, Pz = prob.to_reduced(z)
    np.testing.assert_allclose(kkt.reduced_vector(prob, Vz, Pz), zd, atol=1e-12 * np.abs(zd).max())
    assert np.abs(zi).max() < 1e-12 * np.abs(z).max()


def test_conjugate_symmetry_of_block_solves():
    """y_hat_{n-k} = conj(y_hat_k) for the full (MG/Chebyshev) preconditioner."""
    prob = make(n=4, n_t=8)
    pc = precond.OraclePreconditioner(prob)
    r = synth.probe_vector(prob.cfg)
    for k in (1, 3):
        Y1, Q1 = pc.freq_block(r, k)
        Y2, Q2 = pc.freq_block(r, prob.n_b - k)
        np.testing.assert_allclose(Y2, Y1.conj(), atol=1e-13 * np.abs(Y1).max())
        np.testing.assert_allclose(Q2, Q1.conj(), atol=1e-13 * np.abs(Q1).max())


# ------------------------------------------------------------------ Oseen Algorithm 3
class ExactOseen(precond.OraclePreconditioner):
    def M_solver(self):
        return DenseSolve(self.prob.fine.Ms)

    def Mp_solver(self):
        return DenseSolve(self.prob.fine.Mp)

    def Kp_solver(self):
        return DenseSolve(self.prob.fine.Kp)

    def Q_solvers(self, k):
        p = self.prob
        shift = self.d[k] + p.tau / np.sqrt(p.beta)
        Q = shift * p.fine.Ms + p.tau * p.L()
        return DenseSolve(Q), DenseSolve(Q.conj().T)


def test_algorithm3_with_exact_inner_solves():
    """Many exact-inner Uzawa steps -> G^(1,1)^{-1}(r1, r2); then (y3, y4) = -S_hat^{-1}(r34 - tau(B y2, B y1))
    with S_hat assembled from the display at P:719-731."""
    prob = make("oseen", n=2, n_t=8, beta=1e-3)
    pc = ExactOseen(prob, uzawa_iters=60)
    s = dense_ops.spatial(prob)
    M, L, B, Mp, Kp, Lp = s["M"], s["L"], s["B"], s["Mp"], s["Kp"], s["Lp"]
    tau, beta = prob.tau, prob.beta
    rng = np.random.default_rng(5)
    nv, npu = M.shape[0], B.shape[0]
    for k in (0, 3):
        d = pc.d[k]
        G11 = np.block([[tau * M, np.conj(d) * M + tau * L.T], [d * M + tau * L, -(tau / beta) * M]])
        Z = np.zeros((npu, npu))
        mid = np.block([[tau * Mp, np.conj(d) * Mp + tau * Lp.T], [d * Mp + tau * Lp, -(tau / beta) * Mp]])
        left = np.block([[Z, tau * Mp], [tau * Mp, Z]])
        right = np.block([[Z, tau * Kp], [tau * Kp, Z]])
        Sh = left @ np.linalg.solve(mid, right)
        r = rng.standard_normal(2 * nv + 2 * npu) + 1j * rng.standard_normal(2 * nv + 2 * npu)
        R1, R2, R3, R4 = np.split(r, [nv, 2 * nv, 2 * nv + npu])
        y1, y2, y3, y4 = pc.oseen_block(k, R1.reshape(prob.dim, -1), R2.reshape(prob.dim, -1), R3, R4)
        y12 = np.linalg.solve(G11, np.concatenate([R1, R2]))
        got12 = np.concatenate([y1.reshape(-1), y2.reshape(-1)])
        np.testing.assert_allclose(got12, y12, atol=1e-8 * np.abs(y12).max())
        q = np.concatenate([R3 - tau * B @ y2.reshape(-1), R4 - tau * B @ y1.reshape(-1)])
        np.testing.assert_allclose(np.concatenate([y3, y4]), -np.linalg.solve(Sh, q), atol=1e-9 * np.abs(y3).max())


def test_algorithm3_minus_sign_gives_unipotent_preconditioner():
    """P = [[G11, 0], [G21, -S]] with the exact Schur S: (P^{-1} G - I)^2 = 0 (C.2 #15)."""
    prob = make("oseen", n=2, n_t=8, beta=1e-3)
    d = timeops.spectrum(prob.n_b)[2]
    G = dense_ops.G_block(prob, d)
    nv = prob.dim * prob.fine.nI
    G11, G12, G21 = G[:2 * nv, :2 * nv], G[:2 * nv, 2 * nv:], G[2 * nv:, :2 * nv]
    S = G21 @ np.linalg.solve(G11, G12)
    P = np.block([[G11, np.zeros_like(G12)], [G21, -S]])
    X = np.linalg.solve(P, G) - np.eye(G.shape[0])
    assert np.abs(X @ X).max() < 1e-8 * np.abs(X).max()


def test_uzawa_contraction_with_exact_inner_solves():
    """mu = 3/4 with lambda(S_hat^{-1} S) in [1/2, 1]: 6 steps reduce the error to <~1e-2."""
    prob = make("oseen", n=2, n_t=8, beta=1e-3)
    s = dense_ops.spatial(prob)
    M, L, tau, beta = s["M"], s["L"], prob.tau, prob.beta
    nv = M.shape[0]
    rng = np.random.default_rng(6)
    for k in (0, 3, 4):
        pc = ExactOseen(prob, uzawa_iters=6)
        d = pc.d[k]
        G11 = np.block([[tau * M, np.conj(d) * M + tau * L.T], [d * M + tau * L, -(tau / beta) * M]])
        b = rng.standard_normal(2 * nv) + 1j * rng.standard_normal(2 * nv)
        x = np.linalg.solve(G11, b)
        npu = prob.fine.npu
        y1, y2, _, _ = pc.oseen_block(k, b[:nv].reshape(prob.dim, -1), b[nv:].reshape(prob.dim, -1),
                                      np.zeros(npu), np.zeros(npu))
        err = np.linalg.norm(np.concatenate([y1.reshape(-1), y2.reshape(-1)]) - x) / np.linalg.norm(x)
        assert err < 3e-2


# ------------------------------------------------------------------ Chebyshev, SOR, MG
@pytest.mark.parametrize("space", ["q2", "q1"])
def test_chebyshev_error_bound_and_linearity(space):
    """A-norm error <= 2 c^K / (1 + c^{2K}), c = (sqrt(kappa)-1)/(sqrt(kappa)+1)."""
    prob = make(n=4)
    A = prob.fine.Ms if space == "q2" else prob.fine.Mp
    lo, hi = wathen_bounds(space, 2)
    ch = Chebyshev(A, lo, hi, iters=10)
    rng = np.random.default_rng(7)
    Ad = A.toarray()
    kappa = hi / lo
    c = (np.sqrt(kappa) - 1) / (np.sqrt(kappa) + 1)
    bound = 2 * c**10 / (1 + c**20)
    for _ in range(3):
        f = rng.standard_normal(A.shape[0])
        x = np.linalg.solve(Ad, f)
        e = ch.solve(f) - x
        assert np.sqrt(e @ Ad @ e) <= bound * np.sqrt(x @ Ad @ x) * (1 + 1e-10)
    f1, f2 = rng.standard_normal((2, A.shape[0]))
    np.testing.assert_allclose(ch.solve(2.5 * f1 + f2), 2.5 * ch.solve(f1) + ch.solve(f2), atol=1e-13)


def test_sor_equals_gauss_seidel_and_colouring_valid():
    """omega = 1 multicolour SOR = Gauss-Seidel in colour-then-index order; no same-colour couplings."""
    prob = make(n=4)
    for A, col, nc in ((prob.fine.Ks + prob.fine.Ms, prob.fine.q2_colour, 9),
                       (prob.fine.Kp, prob.fine.q1_colour, 4)):
        Ad = A.toarray()
        same = col[:, None] == col[None, :]
        np.fill_diagonal(same, False)
        assert np.all(Ad[same] == 0.0)
        rng = np.random.default_rng(8)
        b = rng.standard_normal(A.shape[0])
        x0 = rng.standard_normal(A.shape[0])
        x = MultiColourSOR(A, col, nc).sweep(x0.copy()[:, None], b[:, None], range(nc))[:, 0]
        y = x0.copy()
        for c in range(nc):
            for i in np.flatnonzero(col == c):
                y[i] = (b[i] - Ad[i] @ y + Ad[i, i] * y[i]) / Ad[i, i]
        np.testing.assert_allclose(x, y, atol=1e-13)


def test_multigrid_properties():
    """r = 0 -> 0; V-cycle contraction < 1 on SPD probes; many cycles -> dense solve."""
    prob = make(n=8)
    lv = prob.levels
    pc = precond.OraclePreconditioner(prob)
    d = pc.d[1]
    c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
    opsW = [(1 + c1) * l.Ms + c2 * prob.nu * l.Ks for l in lv]
    cases = [(opsW, prob.P2, [l.q2_colour for l in lv], 9), ([l.Kp for l in lv], prob.P1, [l.q1_colour for l in lv], 4)]
    rng = np.random.default_rng(9)
    for ops, P, col, nc in cases:
        b = rng.standard_normal(ops[0].shape[0])
        x = np.linalg.solve(ops[0].toarray(), b)
        one = Multigrid(ops, P, col, nc, cycles=1)
        assert np.abs(one.solve(np.zeros_like(b))).max() == 0.0
        errs = [np.linalg.norm(Multigrid(ops, P, col, nc, cycles=c).solve(b) - x) for c in (1, 2, 3, 4)]
        assert all(errs[i + 1] < 0.5 * errs[i] for i in range(3))
        many = Multigrid(ops, P, col, nc, cycles=40).solve(b)
        np.testing.assert_allclose(many, x, atol=1e-11 * np.abs(x).max())


def test_multigrid_complex_oseen_operator_converges():
    prob = make("oseen", n=8, beta=1e-3)
    pc = precond.OraclePreconditioner(prob)
    mgQ, mgQH = pc.oseen_Q_mgs(3)
    shift = pc.d[3] + prob.tau / np.sqrt(prob.beta)
    Q = (shift * prob.fine.Ms + prob.tau * prob.L()).toarray()
    rng = np.random.default_rng(10)
    b = rng.standard_normal(Q.shape[0]) + 1j * rng.standard_normal(Q.shape[0])
    for mg, A in ((mgQ, Q), (mgQH, Q.conj().T)):
        x = np.linalg.solve(A, b)
        assert np.linalg.norm(mg.solve(b) - x) < 1e-3 * np.linalg.norm(x)


# ------------------------------------------------------------------ Theorems 3.3 / 3.5
def _dense_precond(pc, prob):
    N = prob.cfg.n_dofs
    mask = synth.full_mask(prob.cfg)
    cols = []
    from oracle import kkt
    for j in np.flatnonzero(mask):
        e = np.zeros(N)
        e[j] = 1.0
        V, P = prob.to_reduced(pc.apply(e))
        cols.append(kkt.reduced_vector(prob, V, P))
    return np.array(cols).T


class PhatBlocks(precond.OraclePreconditioner):
    """Algorithm 1 with Z-bar_j = P-hat_j (exact W, exact B W^{-1} B^T)."""

    def block(self, k, R1, R2, R3, R4):
        s = dense_ops.spatial(self.prob)
        d = self.d[k]
        c1, c2 = timeops.stokes_constants(d, self.prob.tau, self.prob.beta)
        W = (1 + c1) * s["M"] + c2 * s["L"]
        S = s["B"] @ np.linalg.solve(W, s["B"].T)
        s1, s2, s3, s4 = self.tl_inv(d, self.prob.tau, self.prob.beta, R1.reshape(-1), R2.reshape(-1), R3, R4)
        x1, x2 = np.linalg.solve(W, s1), np.linalg.solve(W, s2)
        x3, x4 = np.linalg.solve(S, s3), np.linalg.solve(S, s4)
        y1, y2, y3, y4 = self.tr_inv(d, self.prob.tau, self.prob.beta, x1, x2, x3, x4)
        return y1.reshape(R1.shape), y2.reshape(R2.shape), y3, y4


def test_theorem_3_3_count():
    """#{|mu| in [a_hat, b_hat]} >= N - 4 n_v for P_hat_C^{-1} A, [a_hat, b_hat] from the blocks."""
    prob = make(n=2, n_t=6, beta=1e-2, nu=0.05)
    s = dense_ops.spatial(prob)
    pc = PhatBlocks(prob)
    lam = []
    for d in pc.d:
        c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
        W = (1 + c1) * s["M"] + c2 * s["L"]
        S = s["B"] @ np.linalg.solve(W, s["B"].T)
        lam.append(np.abs(np.linalg.eigvals(np.linalg.solve(sla.block_diag(W, W, S, S),
                                                            dense_ops.Z_block(prob, c1, c2)))))
    lam = np.concatenate(lam)
    a, b = lam.min(), lam.max()
    Pinv = _dense_precond(pc, prob)
    A = dense_ops.dense_all_at_once(prob, timeops.backward_euler_E(prob.n_b))
    mu = np.abs(np.linalg.eigvals(Pinv @ A))
    nv = prob.dim * prob.fine.nI
    assert np.sum((mu >= a - 1e-8) & (mu <= b + 1e-8)) >= A.shape[0] - 4 * nv
