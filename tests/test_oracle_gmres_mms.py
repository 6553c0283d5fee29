"""Pins for oracle/gmres.py and the manufactured solution of P:812-824 (oracle/manufactured.py)."""
import numpy as np
import pytest

import synth
from oracle import gmres, kkt, precond, timeops
from oracle.manufactured import solve_manufactured
from oracle.problem import Problem
import dense_ops
from test_oracle_precond import ExactBlocks


def test_gmres_identity_one_iteration():
    b = np.random.default_rng(0).standard_normal(20)
    x, hist, info = gmres.gmres(lambda v: v, lambda v: v, b)
    assert info["iterations"] == 1 and info["converged"]
    np.testing.assert_allclose(x, b, atol=1e-14)


def test_gmres_zero_rhs():
    x, hist, info = gmres.gmres(lambda v: v, lambda v: v, np.zeros(7))
    assert info["iterations"] == 0 and np.all(x == 0)


def test_gmres_matches_dense_solve_with_restarts():
    """Random well-conditioned 50x50, identity preconditioner, tol 1e-10, restart 10."""
    rng = np.random.default_rng(1)
    A = np.eye(50) * 4 + rng.standard_normal((50, 50)) / np.sqrt(50)
    b = rng.standard_normal(50)
    x, hist, info = gmres.gmres(lambda v: A @ v, lambda v: v, b, tol=1e-10, restart=10)
    assert info["converged"] and info["restarts"] >= 1
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-8)
    assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1)
               if (i + 1) % 10 != 0)     # monotone within a cycle
    # right preconditioning with the exact inverse -> 1 iteration
    Ainv = np.linalg.inv(A)
    x, hist, info = gmres.gmres(lambda v: A @ v, lambda v: Ainv @ v, b, tol=1e-10)
    assert info["iterations"] == 1


def test_gmres_with_exact_circulant_preconditioner_is_fast():
    """P_C^{-1} A has >= N - 2 n_v unit eigenvalues (Theorem 3.1): GMRES needs at most 2 n_v + 1 steps."""
    cfg = synth.small_config("t", 2, 2, 6, beta=1e-2, nu=0.05)
    prob = Problem(cfg)
    pc = ExactBlocks(prob)
    b = kkt.build_rhs(prob, synth.desired_state(synth.small_config("t", 2, 2, 6, index=1)))
    x, hist, info = gmres.gmres(lambda v: kkt.kkt_apply(prob, v), pc.apply, b, tol=1e-10, restart=60)
    nv = prob.dim * prob.fine.nI
    assert info["converged"] and info["iterations"] <= 2 * nv + 1
    A = dense_ops.dense_all_at_once(prob, timeops.backward_euler_E(prob.n_b))
    Vb, Pb = prob.to_reduced(b)
    xd = np.linalg.solve(A, kkt.reduced_vector(prob, Vb, Pb))
    Vx, Px = prob.to_reduced(x)
    np.testing.assert_allclose(kkt.reduced_vector(prob, Vx, Px), xd, atol=1e-8 * np.abs(xd).max())


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_full_oracle_solve_converges_to_dense_solution(problem):
    """Linear-mode Algorithm 1 (P~_C, P~_C^(UZ)) inside GMRES(30) reaches tol 1e-6 on a tiny case."""
    lo, hi = (-1.0, 1.0) if problem == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("t", 2, 4, 8, problem=problem, lo=lo, hi=hi, beta=1e-2, nu=0.05)
    prob = Problem(cfg, synth.wind(cfg))
    pc = precond.OraclePreconditioner(prob)
    rng = np.random.default_rng(2)
    b = kkt.build_rhs(prob, rng.standard_normal((2, prob.n_s)))
    x, hist, info = gmres.gmres(lambda v: kkt.kkt_apply(prob, v), pc.apply, b)
    assert info["converged"] and info["true_relres"][-1] < 2e-6
    A = dense_ops.dense_all_at_once(prob, timeops.backward_euler_E(prob.n_b))
    Vb, Pb = prob.to_reduced(b)
    xd = np.linalg.solve(A, kkt.reduced_vector(prob, Vb, Pb))
    Vx, Px = prob.to_reduced(x)
    xs = kkt.reduced_vector(prob, Vx, Px)
    assert np.linalg.norm(xs - xd) < 1e-3 * np.linalg.norm(xd)


def test_manufactured_solution_converges():
    """P:824 "we used this solution to verify the correctness and convergence": nodal errors of v and of
    the closed-form adjoint lambda fall under simultaneous (h, tau) halving, and lambda's
    error falls under tau-halving alone (backward Euler in time)."""
    errs = [solve_manufactured(n, nt) for n, nt in ((2, 4), (4, 8), (8, 16))]
    ev = [e[0] for e in errs]
    el = [e[1] for e in errs]
    assert ev[0] > 4 * ev[1] > 16 * ev[2] and ev[2] < 2e-3
    assert el[0] > 4 * el[1] > 16 * el[2] and el[2] < 2e-2
    lt = [solve_manufactured(8, nt)[1] for nt in (8, 16, 32)]
    assert lt[0] > lt[1] > lt[2]


def test_arnoldi_relation_and_full_spectrum():
    """Textbook Arnoldi pins: A P^{-1} V_m = V_{m+1} H_m (MGS), and at m = n the Ritz values are the
    eigenvalues of A P^{-1} (= those of P^{-1} A)."""
    rng = np.random.default_rng(5)
    n = 12
    A = rng.standard_normal((n, n)) + n * np.eye(n)
    P = np.eye(n) + 0.1 * rng.standard_normal((n, n))
    Pinv = np.linalg.inv(P)
    v0 = rng.standard_normal(n)
    H = gmres.arnoldi(lambda v: A @ v, lambda v: Pinv @ v, v0, 6)
    # rebuild V by the same recurrence and check the relation
    V = np.zeros((n, 7))
    V[:, 0] = v0 / np.linalg.norm(v0)
    for k in range(6):
        w = A @ Pinv @ V[:, k] - V[:, :k + 1] @ H[:k + 1, k]
        V[:, k + 1] = w / H[k + 1, k]
    np.testing.assert_allclose(A @ Pinv @ V[:, :6], V @ H, atol=1e-10)
    Hf = gmres.arnoldi(lambda v: A @ v, lambda v: Pinv @ v, v0, n)
    ritz = np.sort_complex(np.linalg.eigvals(Hf[:n, :n]))
    ev = np.sort_complex(np.linalg.eigvals(Pinv @ A))
    np.testing.assert_allclose(ritz, ev, rtol=1e-9, atol=1e-9)
