"""Block-circulant preconditioner, Algorithm 1 (oracle; test infrastructure only).

precond_apply(r):  r_hat = F r (time DFT of every spatial DOF),
  per frequency k (ALL k < n_b, solved independently as in P:437):
    Stokes:  s = T_l^{-1} r_hat_k;  x = P~_k^{-1} s;  y_k = T_r^{-1} x
    Oseen:   y_k = (P~_k^(UZ))^{-1} r_hat_k                              (Algorithm 3)
  y = F^{-1} y_hat (real up to rounding).

Slots of G_k, order (v, lambda, p, mu): slot 1 = half-0 velocity,
slot 2 = half-1 velocity, slot 3 = half-0 pressure, slot 4 = half-1 pressure.
"""
from __future__ import annotations

import multiprocessing as mp

import numpy as np

from . import timeops
from .inner import Chebyshev, Multigrid, wathen_bounds


class OraclePreconditioner:
    def __init__(self, prob, mg_cycles=4, pre=2, post=2, omega=1.0, cheb_iters=10,
                 uzawa_iters=6, uzawa_mu=0.75, cache_blocks=None, workers=1):
        self.prob = prob
        self.workers = workers        # processes over the independent frequency blocks; 1 = in-process
        self.dim = prob.dim
        self.n_b = prob.n_b
        self.d = timeops.spectrum(prob.n_b)
        self.mg_kw = dict(cycles=mg_cycles, nu1=pre, nu2=post, omega=omega)
        self.cheb_iters = cheb_iters
        self.uzawa_iters, self.uzawa_mu = uzawa_iters, uzawa_mu
        lv = prob.levels
        self.q2col = [l.q2_colour for l in lv]
        self.q1col = [l.q1_colour for l in lv]
        self.nc2, self.nc1 = 3**prob.dim, 2**prob.dim
        f = prob.fine
        # frequency-independent pieces
        self.mg_Kp = Multigrid([l.Kp for l in lv], prob.P1, self.q1col, self.nc1, **self.mg_kw)
        self.cheb_Mp = Chebyshev(f.Mp, *wathen_bounds("q1", prob.dim), iters=cheb_iters)
        self.cheb_M = Chebyshev(f.Ms, *wathen_bounds("q2", prob.dim), iters=cheb_iters)
        # per-frequency solver objects are rebuilt per call unless cached (small problems)
        if cache_blocks is None:
            cache_blocks = prob.n_b * f.nI < 2_000_000
        self.cache = {} if cache_blocks else None

    def _cached(self, key, make):
        if self.cache is None:
            return make()
        if key not in self.cache:
            self.cache[key] = make()
        return self.cache[key]

    # inner-solver factories (tests substitute exact dense solves here)
    def W_solver(self, k):
        return self._cached(("W", k), lambda: self.stokes_W_mg(k))

    def Kp_solver(self):
        return self.mg_Kp

    def Mp_solver(self):
        return self.cheb_Mp

    def M_solver(self):
        return self.cheb_M

    def Q_solvers(self, k):
        return self._cached(("Q", k), lambda: self.oseen_Q_mgs(k))

    # ------------------------------------------------------------------ Stokes
    def stokes_W_mg(self, k):
        """MG for W_k = (1 + c_{k,1}) M + c_{k,2} L with L = nu K."""
        p = self.prob
        c1, c2 = timeops.stokes_constants(self.d[k], p.tau, p.beta)
        ops = [(1.0 + c1) * l.Ms + (c2 * p.nu) * l.Ks for l in p.levels]
        return Multigrid(ops, p.P2, self.q2col, self.nc2, **self.mg_kw)

    @staticmethod
    def tl_inv(d, tau, beta, R1, R2, R3, R4):
        """T_l^{-1} r (block forward substitution with the T_l of P:380-385)."""
        c1, c2 = timeops.stokes_constants(d, tau, beta)
        dc, st = d.imag, np.sqrt(tau)
        s1 = R1 / st
        s2 = (R2 - 1j * (dc / st) * s1) * c2 / st
        s3 = R3 / (st * c2)
        s4 = (R4 - 1j * (dc * c2 / st) * s3) / st
        return s1, s2, s3, s4

    @staticmethod
    def tr_inv(d, tau, beta, X1, X2, X3, X4):
        """T_r^{-1} x (block back substitution with the T_r of P:386-391)."""
        c1, c2 = timeops.stokes_constants(d, tau, beta)
        dc, st = d.imag, np.sqrt(tau)
        y2 = X2 * c2 / st
        y1 = (X1 + 1j * (dc / st) * y2) / st
        y4 = X4 / st
        y3 = (X3 + 1j * (dc * c2 / st) * y4) / (st * c2)
        return y1, y2, y3, y4

    def stokes_block(self, k, R1, R2, R3, R4):
        """y_k = T_r^{-1} P~_k^{-1} T_l^{-1} r_k (Algorithm 1 loop body with Z-bar = P~_k, C.2 #11)."""
        p = self.prob
        d = self.d[k]
        c1, c2 = timeops.stokes_constants(d, p.tau, p.beta)
        s1, s2, s3, s4 = self.tl_inv(d, p.tau, p.beta, R1, R2, R3, R4)
        # P~_k^{-1} = blkdiag(W^{-1}, W^{-1}, S^-1, S^-1) with S^-1 = (1+c1) K_p^{-1} + nu c2 M_p^{-1}
        W, Kp, Mp = self.W_solver(k), self.Kp_solver(), self.Mp_solver()
        x1 = W.solve(s1.T).T
        x2 = W.solve(s2.T).T
        x3 = (1.0 + c1) * Kp.solve(s3) + p.nu * c2 * Mp.solve(s3)
        x4 = (1.0 + c1) * Kp.solve(s4) + p.nu * c2 * Mp.solve(s4)
        return self.tr_inv(d, p.tau, p.beta, x1, x2, x3, x4)

    # ------------------------------------------------------------------ Oseen
    def oseen_Q_mgs(self, k):
        """MG for Q_k = d_k M + tau L + (tau/sqrt(beta)) M and for Q_k^H, per level."""
        p = self.prob
        d = self.d[k]
        shift = d + p.tau / np.sqrt(p.beta)
        opsQ = [shift * l.Ms + (p.tau * p.nu) * l.Ks + p.tau * l.Ns for l in p.levels]
        opsQH = [np.conj(shift) * l.Ms + (p.tau * p.nu) * l.Ks + p.tau * l.Ns.T for l in p.levels]
        return (Multigrid(opsQ, p.P2, self.q2col, self.nc2, **self.mg_kw),
                Multigrid(opsQH, p.P2, self.q2col, self.nc2, **self.mg_kw))

    def oseen_block(self, k, R1, R2, R3, R4):
        """(P~_k^(UZ))^{-1} r_k, Algorithm 3."""
        p = self.prob
        tau, beta, mu = p.tau, p.beta, self.uzawa_mu
        f = p.fine
        d = self.d[k]
        L, LT = p.L(), p.L().T.tocsr()
        M = f.Ms
        G21 = d * M + tau * L                     # d_j M + tau L
        G12 = np.conj(d) * M + tau * LT           # (d_j M + tau L)^H  (M, K real symmetric)
        mgQ, mgQH = self.Q_solvers(k)
        cheb_M = self.M_solver()

        def vel(op, X):                           # per velocity component
            return (op @ X.T).T

        def Shat_inv(Z):                          # S^-1 = tau Q^{-H} M Q^{-1}  (C.2 #14, #25)
            Y = mgQ.solve(Z.T).T
            Y = vel(M, Y)
            Y = mgQH.solve(Y.T).T
            return tau * Y

        b1, b2 = R1, R2
        x1 = np.zeros_like(b1)
        x2 = np.zeros_like(b2)
        for _ in range(self.uzawa_iters):         # eq. (Uzawa11), x^(0) = 0
            x1 = x1 + (1.0 / tau) * cheb_M.solve((b1 - tau * vel(M, x1) - vel(G12, x2)).T).T
            x2 = x2 - (1.0 / mu) * Shat_inv(b2 - vel(G21, x1) + (tau / beta) * vel(M, x2))
        y1, y2 = x1, x2
        # (y3, y4) = -S_hat^{-1} ((r3, r4) - tau (B y2, B y1))
        q3 = R3 - tau * (f.B @ y2.reshape(-1))
        q4 = R4 - tau * (f.B @ y1.reshape(-1))
        y3, y4 = self.oseen_schur_inv(k, q3, q4)
        return y1, y2, -y3, -y4

    def oseen_schur_inv(self, k, q3, q4):
        """S_hat_k^{-1} (q3, q4) for the commutator approximation of P:719-731."""
        p = self.prob
        tau, beta = p.tau, p.beta
        f = p.fine
        d = self.d[k]
        Mp, Lp = f.Mp, p.Lp()
        LpT = Lp.T.tocsr()
        # [[0, tau M_p],[tau M_p, 0]]^{-1}
        Mp_s, Kp_s = self.Mp_solver(), self.Kp_solver()
        s1 = (1.0 / tau) * Mp_s.solve(q4)
        s2 = (1.0 / tau) * Mp_s.solve(q3)
        # middle block [[tau M_p, d^* M_p + tau L_p^T], [d M_p + tau L_p, -(tau/beta) M_p]]
        t1 = tau * (Mp @ s1) + (np.conj(d) * (Mp @ s2) + tau * (LpT @ s2))
        t2 = (d * (Mp @ s1) + tau * (Lp @ s1)) - (tau / beta) * (Mp @ s2)
        # [[0, tau K_p],[tau K_p, 0]]^{-1}
        y3 = (1.0 / tau) * Kp_s.solve(t2)
        y4 = (1.0 / tau) * Kp_s.solve(t1)
        return y3, y4

    # ------------------------------------------------------------------ Algorithm 1
    def block(self, k, R1, R2, R3, R4):
        if self.prob.oseen:
            return self.oseen_block(k, R1, R2, R3, R4)
        return self.stokes_block(k, R1, R2, R3, R4)

    def forward(self, r, ks=None):
        """r_hat = F r on the reduced arrays: Vh (n_k, 2, d, nI), Ph (n_k, 2, npu)."""
        V, P = self.prob.to_reduced(r)
        Vh = timeops.dft(np.moveaxis(V, 1, 0), ks)
        Ph = timeops.dft(np.moveaxis(P, 1, 0), ks)
        return Vh, Ph

    def freq_block(self, r, k):
        """y_hat_k for one frequency (sampled parity): returns (Y (2,d,nI), Q (2,npu))."""
        Vh, Ph = self.forward(r, [k])
        y1, y2, y3, y4 = self.block(k, Vh[0, 0], Vh[0, 1], Ph[0, 0], Ph[0, 1])
        return np.stack([y1, y2]), np.stack([y3, y4])

    def _blocks(self, Vh, Ph):
        """Solve every frequency block k < n_b; with workers > 1 the independent blocks are spread over
        forked processes -- the same block() calls, so the same arithmetic.  Yields (k, block result, extra)."""
        if self.workers <= 1 or self.n_b == 1:
            for k in range(self.n_b):
                yield k, self.block(k, Vh[k, 0], Vh[k, 1], Ph[k, 0], Ph[k, 1]), self._block_extra(k)
            return
        global _WORKER_PC
        _WORKER_PC = self
        ctx = mp.get_context("fork")
        with ctx.Pool(min(self.workers, self.n_b)) as pool:
            args = [(k, (Vh[k, 0], Vh[k, 1], Ph[k, 0], Ph[k, 1])) for k in range(self.n_b)]
            for k, res, extra in pool.imap_unordered(_worker_block, args):
                self._block_extra_set(k, extra)
                yield k, res, extra
        _WORKER_PC = None

    def _block_extra(self, k):
        return None

    def _block_extra_set(self, k, extra):
        pass

    def apply(self, r, return_imag=False):
        """z = P-bar_C^{-1} r on paper-order full vectors (Algorithm 1)."""
        Vh, Ph = self.forward(r)
        Yh = np.zeros_like(Vh)
        Qh = np.zeros_like(Ph)
        for k, (y1, y2, y3, y4), _ in self._blocks(Vh, Ph):
            Yh[k, 0], Yh[k, 1], Qh[k, 0], Qh[k, 1] = y1, y2, y3, y4
        Y = np.moveaxis(timeops.idft(Yh), 0, 1)
        Q = np.moveaxis(timeops.idft(Qh), 0, 1)
        z = self.prob.from_reduced(Y.real, Q.real)
        if return_imag:
            zi = self.prob.from_reduced(Y.imag, Q.imag)
            return z, zi
        return z


_WORKER_PC = None


def _worker_block(arg):
    """Child process of OraclePreconditioner._blocks (fork: the preconditioner object is inherited)."""
    k, R = arg
    res = _WORKER_PC.block(k, *R)
    return k, res, _WORKER_PC._block_extra(k)
