"""Pins for oracle/nonlinear.py: Algorithm 2 and FGMRES."""
import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import gmres, kkt, precond, timeops
from oracle.nonlinear import OracleNonlinearPreconditioner, fgmres, inner_gmres
from oracle.problem import Problem
import dense_ops


def make(problem="stokes", n=4, n_t=6, beta=1e-2, nu=0.05):
    lo, hi = (-1.0, 1.0) if problem == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("t", 2, n, n_t, problem=problem, lo=lo, hi=hi, beta=beta, nu=nu)
    return Problem(cfg, synth.wind(cfg))


def test_inner_gmres_textbook():
    rng = np.random.default_rng(0)
    n = 40
    A = 3 * np.eye(n) + (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x, its = inner_gmres(lambda v: A @ v, lambda v: v, b, 1e-12, 200)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-10)
    assert its <= n
    Ainv = np.linalg.inv(A)
    x, its = inner_gmres(lambda v: A @ v, lambda v: Ainv @ v, b, 1e-12, 200)
    assert its == 1
    x, its = inner_gmres(lambda v: A @ v, lambda v: v, b, 1e-2, 200)
    assert np.linalg.norm(b - A @ x) <= 1e-2 * np.linalg.norm(b) * (1 + 1e-10)


def test_fgmres_with_fixed_preconditioner_equals_gmres():
    """with a fixed linear preconditioner FGMRES iterates are those of GMRES."""
    rng = np.random.default_rng(1)
    n = 60
    A = 4 * np.eye(n) + rng.standard_normal((n, n)) / np.sqrt(n)
    P = np.eye(n) + 0.1 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    x1, h1, i1 = gmres.gmres(lambda v: A @ v, lambda v: P @ v, b, tol=1e-10, restart=10)
    x2, h2, i2 = fgmres(lambda v: A @ v, lambda v: P @ v, b, tol=1e-10, restart=10)
    assert i1["iterations"] == i2["iterations"]
    np.testing.assert_allclose(h1, h2, rtol=1e-9)
    np.testing.assert_allclose(x1, x2, atol=1e-10)


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_block_operators_equal_displays(problem):
    """Z_apply = Z_j of P:392-397, G_apply = G_j of eq. (SubBlockG) (dense displays)."""
    prob = make(problem, n=2, n_t=6)
    pc = OracleNonlinearPreconditioner(prob)
    rng = np.random.default_rng(2)
    nv, npu = prob.dim * prob.fine.nI, prob.fine.npu
    v = rng.standard_normal(2 * nv + 2 * npu) + 1j * rng.standard_normal(2 * nv + 2 * npu)
    for k in (0, 2):
        d = pc.d[k]
        got = pc._pack(pc.G_apply(k, pc._unpack(v)))
        np.testing.assert_allclose(got, dense_ops.G_block(prob, d) @ v, atol=1e-13)
        if problem == "stokes":
            c1, c2 = timeops.stokes_constants(d, prob.tau, prob.beta)
            got = pc._pack(pc.Z_apply(k, pc._unpack(v)))
            np.testing.assert_allclose(got, dense_ops.Z_block(prob, c1, c2) @ v, atol=1e-13)


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_tight_inner_tolerance_gives_the_exact_circulant_solve(problem):
    """eps -> 0: Algorithm 2 = F^{-1} blkdiag(G_k^{-1}) F = P_C^{-1} (dense)."""
    prob = make(problem, n=2, n_t=6)
    pc = OracleNonlinearPreconditioner(prob, inner_eps=1e-13, inner_maxit=400)
    PC = dense_ops.dense_all_at_once(prob, timeops.circulant_C(prob.n_b))
    r = synth.probe_vector(prob.cfg)
    z = pc.apply(r)
    V, P = prob.to_reduced(r)
    zd = np.linalg.solve(PC, kkt.reduced_vector(prob, V, P))
    Vz, Pz = prob.to_reduced(z)
    np.testing.assert_allclose(kkt.reduced_vector(prob, Vz, Pz), zd, atol=1e-8 * np.abs(zd).max())


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_fgmres_with_nonlinear_preconditioner_converges_fast(problem):
    """Order-of-magnitude anchor (Tables 2-5: 3-10 outer FGMRES iterations at eps = 1e-2)."""
    prob = make(problem, n=4, n_t=8, beta=1e-3, nu=0.05)
    pc = OracleNonlinearPreconditioner(prob, inner_eps=1e-2)
    b = kkt.build_rhs(prob, np.random.default_rng(3).standard_normal((2, prob.n_s)))
    x, hist, info = fgmres(lambda v: kkt.kkt_apply(prob, v), pc.apply, b, tol=1e-6, restart=10)
    assert info["converged"] and info["iterations"] <= 15
    lin = precond.OraclePreconditioner(prob)
    _, _, info_lin = gmres.gmres(lambda v: kkt.kkt_apply(prob, v), lin.apply, b, tol=1e-6, restart=30)
    assert info["iterations"] < info_lin["iterations"]


def test_Pt_apply_equals_dense_blockdiag_with_exact_inner_solves():
    """Pt_apply (Algorithm 2's inner preconditioner P~_j^{-1}) with exact inner solves equals the
    dense blkdiag(W, W, S~, S~)^{-1}, W = (1 + c1) M + c2 L, S~^{-1} = (1 + c1) K_p^{-1} + nu c2 M_p^{-1}
    (P:424), built here from dense_ops' spatial matrices; and with the multigrid inner solves it is the
    Algorithm-1 block between the T transforms: T_r^{-1} Pt_apply(T_l^{-1} r) = stokes_block(r)."""
    prob = make("stokes", n=2, n_t=6)
    pc = OracleNonlinearPreconditioner(prob)
    s = dense_ops.spatial(prob)
    rng = np.random.default_rng(9)
    nI, npu = prob.fine.nI, prob.fine.npu
    S = (rng.standard_normal((prob.dim, nI)) + 1j * rng.standard_normal((prob.dim, nI)),
         rng.standard_normal((prob.dim, nI)) + 1j * rng.standard_normal((prob.dim, nI)),
         rng.standard_normal(npu) + 1j * rng.standard_normal(npu),
         rng.standard_normal(npu) + 1j * rng.standard_normal(npu))
    for k in (1, 2):
        # multigrid inner solves: consistency with the (pinned) Algorithm-1 Stokes block
        d = pc.d[k]
        sl = pc.tl_inv(d, prob.tau, prob.beta, *S)
        got = pc.tr_inv(d, prob.tau, prob.beta, *pc.Pt_apply(k, sl))
        ref = pc.stokes_block(k, *S)
        for g_, r_ in zip(got, ref):
            np.testing.assert_allclose(g_, r_, atol=1e-13 * np.abs(r_).max())
    # exact inner solves
    pe = OracleNonlinearPreconditioner(prob)
    Ms, Ks = prob.fine.Ms.toarray(), prob.nu * prob.fine.Ks.toarray()
    for k in (1, 2):
        c1, c2 = timeops.stokes_constants(pe.d[k], prob.tau, prob.beta)
        Wk = (1.0 + c1) * Ms + c2 * Ks
        pe.W_solver = lambda kk, Wk=Wk: dense_ops.DenseSolve(Wk)
        pe.Kp_solver = lambda: dense_ops.DenseSolve(s["Kp"])
        pe.Mp_solver = lambda: dense_ops.DenseSolve(s["Mp"])
        got = pe.Pt_apply(k, S)
        Wd = (1.0 + c1) * s["M"] + c2 * s["L"]
        Sinv = (1.0 + c1) * np.linalg.inv(s["Kp"]) + prob.nu * c2 * np.linalg.inv(s["Mp"])
        ref = (np.linalg.solve(Wd, S[0].reshape(-1)).reshape(prob.dim, -1),
               np.linalg.solve(Wd, S[1].reshape(-1)).reshape(prob.dim, -1), Sinv @ S[2], Sinv @ S[3])
        for g_, r_ in zip(got, ref):
            np.testing.assert_allclose(g_, r_, atol=1e-11 * np.abs(r_).max())
