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


exact_v = synth.mms_velocity        # the paper's data live in synth/ (inputs of both sides)
forcing = synth.mms_forcing
desired = synth.mms_desired


def exact_lambda(x, y, t, T, beta):
    """lambda = beta (v_t - Lap v + grad p - f) = beta (e^{T-t} - 1) [2y(x^2-1)^2(y^2-1), -2x(x^2-1)(y^2-1)^2]
    (derived from the state equation of P:53-55 with the data above)."""
    g = beta * (np.exp(T - t) - 1.0)
    return np.stack([g * 2 * y * (x**2 - 1) ** 2 * (y**2 - 1), -g * 2 * x * (x**2 - 1) * (y**2 - 1) ** 2])


def rhs_with_data(prob, vd, f, g, v0, wind=None):
    """Right-hand side of the optimality system with time-dependent data, paper order.

    vd, f: (n_b, d, n_s) nodal v_d and f at t_m, m = 1..n_b; g: (n_b + 1, d, n_s) Dirichlet data at
    t_0..t_{n_b} (boundary entries used); v0: (d, n_s) initial state on every node (or None: g[0]).
    Boundary columns of the state are moved to the right-hand side (lifting):
      adjoint rows (half 0):  tau M (v_d^m - G^m) |_I
      state rows   (half 1):  [M (tau f^m - G^m + H^{m-1}) - tau L G^m] |_I,  H^0 = v0, H^{m-1} = G^{m-1}
      divergence rows (half 1): -tau B G^m |_Ip
    with G^m = g^m on boundary nodes and 0 inside, L = nu K (Stokes) or nu K + N (Oseen, `wind` the Q2 nodal
    wind of the problem).  Every matrix is the full (un-eliminated) assembled operator restricted to the
    unknown rows."""
    cfg = prob.cfg
    f_lv = fem.Level(cfg.dim, cfg.n_cells, cfg.x_lo, cfg.x_hi)
    fine = prob.fine
    Iv, Ip = fine.Iv, fine.Ip
    n_s, d, n_b, tau = prob.n_s, cfg.dim, prob.n_b, prob.tau
    bmask = np.ones(n_s, dtype=bool)
    bmask[Iv] = False
    Mfull, Kfull, Bfull = f_lv.mass_q2(), f_lv.stiff_q2(), f_lv.div()
    Lfull = cfg.nu * Kfull
    if prob.oseen:
        Lfull = Lfull + f_lv.conv_q2(wind)
    V = np.zeros((2, n_b, d, len(Iv)))
    P = np.zeros((2, n_b, fine.npu))
    G = lambda m, c: np.where(bmask, g[m][c], 0.0) if g is not None else np.zeros(n_s)
    for j in range(n_b):
        m = j + 1
        Gfull = np.zeros(d * n_s)
        for c in range(d):
            Gm = G(m, c)
            Gfull[c * n_s:(c + 1) * n_s] = Gm
            vdm = vd[j][c] if vd is not None else np.zeros(n_s)
            V[0, j, c] = tau * (Mfull @ (vdm - Gm))[Iv]
            fm = f[j][c] if f is not None else np.zeros(n_s)
            if m == 1:
                H = v0[c] if v0 is not None else G(0, c)
            else:
                H = G(m - 1, c)
            V[1, j, c] = (Mfull @ (tau * fm - Gm + H) - tau * (Lfull @ Gm))[Iv]
        P[1, j] = -tau * (Bfull @ Gfull)[Ip]
    return prob.from_reduced(V, P)


def solve_manufactured(n_cells, n_t, T=1.0, beta=1e-2, full=False):
    """Solve the discrete optimality system; return the max-over-t_j relative nodal errors of v and lambda
    (and, with full=True, the solution in paper order)."""
    cfg = synth.mms_config(n_cells, n_t, beta)
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
    # right-hand side with lifting (rhs_with_data), in the ordering of A: blocks (half, t), [v comps, p]
    nb = nv + npu
    vd, fd, gd, v0 = synth.mms_inputs(cfg)
    Vr, Pr = prob.to_reduced(rhs_with_data(prob, vd, fd, gd, v0))
    b = np.concatenate([np.concatenate([Vr[h, j].reshape(-1), Pr[h, j]]) for h in range(2) for j in range(n_b)])
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
    if full:
        V = np.zeros((2, n_b, 2, len(Iv)))
        P = np.zeros((2, n_b, npu))
        for h in range(2):
            for j in range(n_b):
                blk = sol[(h * n_b + j) * nb:(h * n_b + j + 1) * nb]
                V[h, j] = blk[:nv].reshape(2, -1)
                P[h, j] = blk[nv:]
        return err / ref, lerr / lref, prob.from_reduced(V, P)
    return err / ref, lerr / lref
