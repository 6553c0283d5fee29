"""One configuration's discrete operators and MG hierarchy (oracle; test infrastructure only).

Assembles, per mesh level N_c, N_c/2, ..., 2, the eliminated
operators M_s, K_s (Q2 scalar, interior rows/cols), N_s (Oseen), M_p, K_p
(Q1, pinned node deleted), and on the finest level B, N_p and the full-grid
mass used by the right-hand side.  Coarse operators are re-discretised with
the same scalars (equal to Galerkin P^T A P, pinned in the tests).

Reduced vectors: one spatial block is [v_0 | ... | v_{d-1} | p] with v_c over
the interior Q2 nodes and p over the unknown Q1 nodes.  The interchange
("paper order", SURVEY DS-01) is the full-grid space-time vector of length N:
index ((half * n_b + t) * (n_v + n_p)) + field offset, half 0 = (v, p),
half 1 = (lambda, mu) (P:96-100 reordered as in eq. FinalA).
"""
from __future__ import annotations

import numpy as np

from . import fem, transfer


def q2_colours(dim, n1, nodes):
    """Colour (i mod 3) + 3 (j mod 3) [+ 9 (k mod 3)] of full-grid Q2 nodes (C.2 #12)."""
    col = np.zeros_like(nodes)
    for axis in range(dim):
        col += ((nodes // n1**axis) % n1 % 3) * 3**axis
    return col


def q1_colours(dim, n1, nodes):
    """Colour (i mod 2) + 2 (j mod 2) [+ 4 (k mod 2)] of full-grid Q1 nodes (C.2 #12)."""
    col = np.zeros_like(nodes)
    for axis in range(dim):
        col += ((nodes // n1**axis) % n1 % 2) * 2**axis
    return col


class LevelOps:
    def __init__(self, dim, n_cells, lo, hi, wind_q2=None, fine=False):
        L = fem.Level(dim, n_cells, lo, hi)
        self.level = L
        self.dim, self.n_cells = dim, n_cells
        self.Iv, self.Ip = L.q2_interior(), L.q1_unknowns()
        self.nI, self.npu = len(self.Iv), len(self.Ip)
        Ms_full = L.mass_q2()
        self.Ms = fem.restrict(Ms_full, self.Iv, self.Iv)
        self.Ks = fem.restrict(L.stiff_q2(), self.Iv, self.Iv)
        self.Mp = fem.restrict(L.mass_q1(), self.Ip, self.Ip)
        self.Kp = fem.restrict(L.stiff_q1(), self.Ip, self.Ip)
        self.Ns = None
        if wind_q2 is not None:
            self.Ns = fem.restrict(L.conv_q2(wind_q2), self.Iv, self.Iv)
        self.q2_colour = q2_colours(dim, L.n1q2, self.Iv)
        self.q1_colour = q1_colours(dim, L.n1q1, self.Ip)
        if fine:
            self.Ms_full_rows = Ms_full[self.Iv].tocsr()        # for the RHS tau (M_full v_d)|_I
            Bfull = L.div()
            cols = np.concatenate([c * L.n_s + self.Iv for c in range(dim)])
            self.B = fem.restrict(Bfull, self.Ip, cols)          # n_pu x (d nI)
            self.BT = self.B.T.tocsr()
            self.Np = None
            if wind_q2 is not None:
                self.Np = fem.restrict(L.conv_q1(wind_q2), self.Ip, self.Ip)


class Problem:
    """All operators of one configuration `cfg` (a synth.Config)."""

    def __init__(self, cfg, wind_q2=None):
        self.cfg = cfg
        self.dim = cfg.dim
        self.n_b = cfg.n_t - 1
        self.tau = cfg.T / cfg.n_t
        self.beta, self.nu = cfg.beta, cfg.nu
        self.oseen = cfg.problem == "oseen"
        if self.oseen and wind_q2 is None:
            raise ValueError("Oseen needs a wind")
        self.n_cells_levels = []
        n = cfg.n_cells
        while n >= 2:
            self.n_cells_levels.append(n)
            n //= 2
        self.levels = []
        w = wind_q2 if self.oseen else None
        for li, nc in enumerate(self.n_cells_levels):
            self.levels.append(LevelOps(cfg.dim, nc, cfg.x_lo, cfg.x_hi, w, fine=(li == 0)))
            if w is not None:
                w = fem.inject_wind(w, cfg.dim, nc)
        # transfers between level li+1 (coarse) and li (fine)
        self.P2, self.P1 = [], []
        for li in range(len(self.levels) - 1):
            f, c = self.levels[li], self.levels[li + 1]
            self.P2.append(transfer.prolongation(cfg.dim, c.n_cells, 2, f.Iv, c.Iv))
            self.P1.append(transfer.prolongation(cfg.dim, c.n_cells, 1, f.Ip, c.Ip))
        f = self.levels[0]
        self.fine = f
        self.n_s = (2 * cfg.n_cells + 1) ** cfg.dim
        self.n_p = (cfg.n_cells + 1) ** cfg.dim
        self.n_block = cfg.dim * self.n_s + self.n_p        # n_v + n_p (full grid)

    # ------------------------------------------------------------ layout helpers
    def to_reduced(self, x):
        """Paper-order full vector (N,) -> V (2, n_b, d, nI), P (2, n_b, npu); masked entries dropped."""
        f = self.fine
        X = x.reshape(2, self.n_b, self.n_block)
        V = np.stack([X[:, :, c * self.n_s + f.Iv] for c in range(self.dim)], axis=2)
        P = X[:, :, self.dim * self.n_s + f.Ip]
        return V, P

    def from_reduced(self, V, P):
        f = self.fine
        X = np.zeros((2, self.n_b, self.n_block), dtype=np.result_type(V, P))
        for c in range(self.dim):
            X[:, :, c * self.n_s + f.Iv] = V[:, :, c]
        X[:, :, self.dim * self.n_s + f.Ip] = P
        return X.reshape(-1)

    def L(self):
        """L = nu K + N on the Q2 scalar space (C.2 #8)."""
        f = self.fine
        return self.nu * f.Ks + (f.Ns if f.Ns is not None else 0 * f.Ks)

    def Lp(self):
        """L_p = nu K_p + N_p (C.2 #9)."""
        f = self.fine
        return self.nu * f.Kp + (f.Np if f.Np is not None else 0 * f.Kp)
