"""Manufactured Stokes solution of P:812-824 (oracle-only verification; test infrastructure only).

Omega = [-1,1]^2, nu = 1, exact
  v = e^{T-t} [20 x y^3, 5 x^4 - 5 y^4],  p = e^{T-t} (60 x^2 y - 20 y^3) + const,
with v_d and f transcribed from P:815-820, initial and boundary data "given
implicitly by v".  The discrete system is A x = b with the same A as
eq. (FinalA), and a right-hand side that carries the inhomogeneous Dirichlet
data by lifting (boundary columns moved to the RHS) and v^(0) = v_0.
Solved with a sparse direct solver (scipy spsolve) -- a textbook routine --
so this pins the discretisation (A, B's sign, M, K, the time recursion and the
RHS convention), independent of the preconditioner.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import synth
from . import fem
from .problem import Problem
from .timeops import backward_euler_E


def exact_v(x, y, t, T):
    e = np.exp(T - t)
    return np.stack([e * 20 * x * y**3, e * (5 * x**4 - 5 * y**4)])


def forcing(x, y, t, T):
    """f of P:818-820."""
    e = np.exp(T - t)
    a = (x**2 - 1) ** 2 * (y**2 - 1)
    b = (x**2 - 1) * (y**2 - 1) ** 2
    return np.stack([e * (-20 * x * y**3 - 2 * y * a) + 2 * y * a,
                     e * (5 * (y**4 - x**4) + 2 * x * b) - 2 * x * b])


def desired(x, y, t, T, beta):
    """v_d of P:815-817."""
    e = np.exp(T - t)
    c1 = 4 * beta * (y * (2 * (3 * x**2 - 1) * (y**2 - 1) + 3 * (x**2 - 1) ** 2))
    c2 = 4 * beta * (-x * (3 * (y**2 - 1) ** 2 + 2 * (x**2 - 1) * (3 * y**2 - 1)))
    d1 = e * (20 * x * y**3 + 2 * beta * y * ((x**2 - 1) ** 2 * (y**2 - 7) - 4 * (3 * x**2 - 1) * (y**2 - 1) + 2))
    d2 = e * (5 * (x**4 - y**4) - 2 * beta * x * ((y**2 - 1) ** 2 * (x**2 - 7) - 4 * (x**2 - 1) * (3 * y**2 - 1) - 2))
    return np.stack([c1 + d1, c2 + d2])


def exact_lambda(x, y, t, T, beta):
    """lambda = beta (v_t - Lap v + grad p - f) = beta (e^{T-t} - 1) [2y(x^2-1)^2(y^2-1), -2x(x^2-1)(y^2-1)^2]
    (derived from the state equation of P:53-55 with the data above)."""
    g = beta * (np.exp(T - t) - 1.0)
    return np.stack([g * 2 * y * (x**2 - 1) ** 2 * (y**2 - 1), -g * 2 * x * (x**2 - 1) * (y**2 - 1) ** 2])


def solve_manufactured(n_cells, n_t, T=1.0, beta=1e-2):
    """Solve the discrete optimality system; return the max-over-t_j relative nodal errors of v and lambda."""
    cfg = synth.small_config("mms", 2, n_cells, n_t, lo=-1.0, hi=1.0, beta=beta, nu=1.0)
    prob = Problem(cfg)
    f = prob.fine
    Lv = fem.Level(2, n_cells, -1.0, 1.0)
    X = synth.q2_coords(cfg)
    x, y = X[0], X[1]
    tau, n_b = prob.tau, prob.n_b
    Iv, Ip = f.Iv, f.Ip
    Bd = np.setdiff1d(np.arange(Lv.n_s), Iv)
    Mfull, Kfull = Lv.mass_q2(), Lv.stiff_q2()
    Lfull = 1.0 * Kfull                                     # nu = 1, Stokes
    Bfull = Lv.div()
    M_IB, L_IB = Mfull[Iv][:, Bd], Lfull[Iv][:, Bd]
    # sparse A of eq. (FinalA), ordering (half, t, [v comps, p]) as in kkt.dense_kkt
    I_d = sp.identity(2)
    M = sp.kron(I_d, f.Ms)
    L = sp.kron(I_d, prob.L())
    B = f.B
    nv, npu = M.shape[0], B.shape[0]
    Zvp = sp.csr_matrix((nv, npu))
    Zpp = sp.csr_matrix((npu, npu))
    MM = sp.bmat([[M, Zvp], [Zvp.T, Zpp]])
    S1 = sp.bmat([[L, B.T], [B, Zpp]])
    S2 = sp.bmat([[L.T, B.T], [B, Zpp]])
    E = sp.csr_matrix(backward_euler_E(n_b))
    I = sp.identity(n_b)
    O = sp.csr_matrix((n_b, n_b))
    T1 = sp.bmat([[tau * I, E.T], [E, -(tau / beta) * I]])
    A = (sp.kron(T1, MM) + tau * sp.kron(sp.bmat([[O, O], [I, O]]), S1)
         + tau * sp.kron(sp.bmat([[O, I], [O, O]]), S2)).tocsc()
    # right-hand side with lifting, block m = 1..n_b at t_m = m tau
    nb = nv + npu
    b = np.zeros(2 * n_b * nb)
    vB = lambda m: exact_v(x[Bd], y[Bd], m * tau, T)           # boundary values (d, |Bd|)
    for m in range(1, n_b + 1):
        j = m - 1
        # adjoint rows (half 0): tau M (v_d - v); the boundary part of v^(m) stays on the RHS
        vd = desired(x, y, m * tau, T, beta)
        r0 = np.concatenate([tau * ((Mfull @ vd[c])[Iv] - M_IB @ vB(m)[c]) for c in range(2)])
        b[(0 * n_b + j) * nb:(0 * n_b + j) * nb + nv] = r0
        # state rows (half 1): M(v^m - v^{m-1}) + tau L v^m + tau B^T p^m - tau/beta M lam^m = tau M f^m
        fm = forcing(x, y, m * tau, T)
        r1 = []
        for c in range(2):
            rc = tau * (Mfull @ fm[c])[Iv] - M_IB @ vB(m)[c] - tau * (L_IB @ vB(m)[c])
            if m == 1:
                v0 = exact_v(x, y, 0.0, T)[c]                   # v^(0) = v_0, all nodes
                rc = rc + (Mfull @ v0)[Iv]
            else:
                rc = rc + M_IB @ vB(m - 1)[c]
            r1.append(rc)
        b[(1 * n_b + j) * nb:(1 * n_b + j) * nb + nv] = np.concatenate(r1)
        # divergence rows (half 1 pressure): tau B v^m = 0 -> tau B_I v_I = -tau B_B v_B
        vfull = np.zeros(2 * Lv.n_s)
        for c in range(2):
            vfull[c * Lv.n_s + Bd] = vB(m)[c]
        b[(1 * n_b + j) * nb + nv:(1 * n_b + j + 1) * nb] = -tau * (Bfull @ vfull)[Ip]
    sol = spla.spsolve(A, b)
    err, ref, lerr, lref = 0.0, 0.0, 0.0, 0.0
    for m in range(1, n_b + 1):
        j = m - 1
        vh = sol[j * nb:j * nb + nv].reshape(2, -1)
        ve = exact_v(x[Iv], y[Iv], m * tau, T)
        err = max(err, np.sqrt(np.mean((vh - ve) ** 2)))
        ref = max(ref, np.sqrt(np.mean(ve**2)))
        lh = sol[(n_b + j) * nb:(n_b + j) * nb + nv].reshape(2, -1)
        le = exact_lambda(x[Iv], y[Iv], m * tau, T, beta)
        lerr = max(lerr, np.sqrt(np.mean((lh - le) ** 2)))
        lref = max(lref, np.sqrt(np.mean(le**2)))
    return err / ref, lerr / lref
