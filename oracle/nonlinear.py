"""Nonlinear block-circulant preconditioner, Algorithm 2, and FGMRES (oracle; test infrastructure).

Algorithm 2:  r_hat = F r;  per frequency j:
    Stokes: s_j = T_l^{-1} r_hat_j;  x_j = GMRES(Z_j, P~_j, s_j, tol = eps);  y_j = T_r^{-1} x_j
    Oseen:  y_j = GMRES(G_j, P~_j^(UZ), r_hat_j, tol = eps)
  y = F^{-1} y_hat.
Readings: the inner preconditioner is P~_j (the paper's pseudocode names the
dense P^_j, impractical per P:422); inner GMRES is right-preconditioned, x0 = 0, MGS, no restart,
stopping when the recurrence residual <= eps ||s_j||, capped at `inner_maxit`.  eps = 1e-2.
Because the inner solver is a Krylov method the preconditioner is nonlinear, hence the outer
flexible GMRES (FGMRES) with restart 10, which stores the preconditioned vectors.
"""
from __future__ import annotations

import numpy as np

from . import timeops
from .precond import OraclePreconditioner


def inner_gmres(apply_A, apply_P, b, eps, maxit):
    """Right-preconditioned complex GMRES without restart: returns (x, iterations).

    Stops when |g_{k+1}| <= eps ||b|| (recurrence residual), or at maxit, or on breakdown.
    Hermitian inner products <u, v> = u^H v; complex Givens rotations.
    """
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros_like(b), 0
    V = [b / bnorm]
    Zs = []
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    cs = np.zeros(maxit, dtype=complex)
    sn = np.zeros(maxit, dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = bnorm
    k_done = 0
    for k in range(maxit):
        z = apply_P(V[k])
        Zs.append(z)
        w = apply_A(z)
        for i in range(k + 1):                              # modified Gram-Schmidt
            H[i, k] = np.vdot(V[i], w)
            w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        for i in range(k):                                  # previous rotations
            t = np.conj(cs[i]) * H[i, k] + np.conj(sn[i]) * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = t
        a, bb = H[k, k], H[k + 1, k]
        den = np.sqrt(abs(a) ** 2 + abs(bb) ** 2)
        cs[k], sn[k] = a / den, bb / den
        H[k, k] = den
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = np.conj(cs[k]) * g[k]
        k_done = k + 1
        if abs(g[k + 1]) <= eps * bnorm or abs(bb) < 1e-14 * bnorm:
            break
        V.append(w / bb)
    y = np.zeros(k_done, dtype=complex)
    for i in range(k_done - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:k_done] @ y[i + 1:]) / H[i, i]
    x = np.zeros_like(b)
    for i in range(k_done):
        x = x + y[i] * Zs[i]
    return x, k_done


class OracleNonlinearPreconditioner(OraclePreconditioner):
    """Algorithm 2: per-frequency inner GMRES to tolerance eps, preconditioned by P~_j (or P~_j^(UZ))."""

    def __init__(self, prob, inner_eps=1e-2, inner_maxit=200, **kw):
        super().__init__(prob, **kw)
        self.inner_eps, self.inner_maxit = inner_eps, inner_maxit
        self.last_inner = {}

    def _block_extra(self, k):            # the inner iteration count travels back from a worker process
        return self.last_inner.get(k)

    def _block_extra_set(self, k, extra):
        self.last_inner[k] = extra

    # ---- the block operators, written from their displays
    def Z_apply(self, k, X):
        """Z_j of P:392-397 on X = (x1, x2, x3, x4): rows [M, X, 0, B^T], [X, -M, B^T, 0], [0, B, 0, 0], [B, 0, 0, 0],
        X = c1 M + c2 L (Stokes: L = nu K)."""
        p = self.prob
        f = p.fine
        c1, c2 = timeops.stokes_constants(self.d[k], p.tau, p.beta)
        x1, x2, x3, x4 = X
        M, L = f.Ms, p.L()
        vel = lambda op, V: (op @ V.T).T
        BT = lambda q: (f.BT @ q).reshape(p.dim, -1)
        Bv = lambda v: f.B @ v.reshape(-1)
        XM = lambda V: c1 * vel(M, V) + c2 * vel(L, V)
        return (vel(M, x1) + XM(x2) + BT(x4), XM(x1) - vel(M, x2) + BT(x3), Bv(x2), Bv(x1))

    def G_apply(self, k, X):
        """G_j of eq. (SubBlockG)."""
        p = self.prob
        f = p.fine
        tau, beta, d = p.tau, p.beta, self.d[k]
        x1, x2, x3, x4 = X
        M, L = f.Ms, p.L()
        LT = L.T.tocsr()
        vel = lambda op, V: (op @ V.T).T
        BT = lambda q: (f.BT @ q).reshape(p.dim, -1)
        Bv = lambda v: f.B @ v.reshape(-1)
        r1 = tau * vel(M, x1) + np.conj(d) * vel(M, x2) + tau * vel(LT, x2) + tau * BT(x4)
        r2 = d * vel(M, x1) + tau * vel(L, x1) - (tau / beta) * vel(M, x2) + tau * BT(x3)
        return (r1, r2, tau * Bv(x2), tau * Bv(x1))

    def Pt_apply(self, k, S):
        """P~_j^{-1} = blkdiag(W^-1, W^-1, S^-1, S^-1), the same inner solves as Algorithm 1."""
        p = self.prob
        c1, c2 = timeops.stokes_constants(self.d[k], p.tau, p.beta)
        W, Kp, Mp = self.W_solver(k), self.Kp_solver(), self.Mp_solver()
        s1, s2, s3, s4 = S
        return (W.solve(s1.T).T, W.solve(s2.T).T,
                (1.0 + c1) * Kp.solve(s3) + p.nu * c2 * Mp.solve(s3),
                (1.0 + c1) * Kp.solve(s4) + p.nu * c2 * Mp.solve(s4))

    # ---- flatten helpers for the inner Krylov method
    def _pack(self, X):
        return np.concatenate([X[0].reshape(-1), X[1].reshape(-1), X[2], X[3]])

    def _unpack(self, v):
        f = self.prob.fine
        nv = self.dim * f.nI
        return (v[:nv].reshape(self.dim, -1), v[nv:2 * nv].reshape(self.dim, -1),
                v[2 * nv:2 * nv + f.npu], v[2 * nv + f.npu:])

    def block(self, k, R1, R2, R3, R4):
        p = self.prob
        if p.oseen:
            A = lambda v: self._pack(self.G_apply(k, self._unpack(v)))
            P = lambda v: self._pack(self.oseen_block(k, *self._unpack(v)))
            x, its = inner_gmres(A, P, self._pack((R1, R2, R3, R4)), self.inner_eps, self.inner_maxit)
            self.last_inner[k] = its
            return self._unpack(x)
        d = self.d[k]
        s = self.tl_inv(d, p.tau, p.beta, R1, R2, R3, R4)
        A = lambda v: self._pack(self.Z_apply(k, self._unpack(v)))
        P = lambda v: self._pack(self.Pt_apply(k, self._unpack(v)))
        x, its = inner_gmres(A, P, self._pack(s), self.inner_eps, self.inner_maxit)
        self.last_inner[k] = its
        return self.tr_inv(d, p.tau, p.beta, *self._unpack(x))


def fgmres(apply_A, apply_Pinv, b, tol=1e-6, restart=10, max_iters=500):
    """Flexible GMRES (Saad 1993), right preconditioning with a varying preconditioner:
    stores Z_j = P_j^{-1} v_j and updates x += Z_k y.  Same stopping rule and history as gmres()."""
    n = b.shape[0]
    x = np.zeros(n)
    bnorm = np.linalg.norm(b)
    hist = []
    info = dict(iterations=0, restarts=0, converged=False, breakdown=False, true_relres=[])
    if bnorm == 0.0:
        info["converged"] = True
        return x, hist, info
    r = b.copy()
    it = 0
    while True:
        beta0 = np.linalg.norm(r)
        V = [r / beta0]
        Z = []
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta0
        k_done = 0
        stop = False
        for k in range(restart):
            z = apply_Pinv(V[k])
            Z.append(z)
            w = apply_A(z)
            for i in range(k + 1):
                H[i, k] = np.dot(w, V[i])
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            hkk, hk1 = H[k, k], H[k + 1, k]
            den = np.hypot(hkk, hk1)
            cs[k], sn[k] = hkk / den, hk1 / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            it += 1
            k_done = k + 1
            hist.append(abs(g[k + 1]) / bnorm)
            if abs(g[k + 1]) <= tol * bnorm:
                info["converged"] = True
                stop = True
                break
            if hk1 < 1e-14 * bnorm:
                info["breakdown"] = True
                stop = True
                break
            if it >= max_iters:
                stop = True
                break
            V.append(w / hk1)
        y = np.zeros(k_done)
        for i in range(k_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k_done] @ y[i + 1:]) / H[i, i]
        for i in range(k_done):
            x = x + y[i] * Z[i]
        r = b - apply_A(x)
        info["true_relres"].append(np.linalg.norm(r) / bnorm)
        if stop:
            break
        info["restarts"] += 1
    info["iterations"] = it
    return x, hist, info
