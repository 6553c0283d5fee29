"""Inner solvers: multicolour SOR, geometric multigrid, Chebyshev (oracle; test infrastructure only).

The paper fixes: "multigrid method with successive
over-relaxation for the smoothing", "in each application of MG 4 V-cycles",
"Chebyshev semi-iterations ... set to 10".  Everything it leaves open takes
SURVEY C.2 #12/#13: multicolour SOR with omega = 1, nu1 = nu2 = 2 sweeps, colour
order 0..C-1 before and C-1..0 after the coarse correction, exact LU on the
coarsest level (N_c = 2), prolongation P = nodal interpolation, restriction
P^T, V-cycles started from x = 0.  Chebyshev is the Jacobi-preconditioned
semi-iteration with Wathen's element bounds (recurrence SURVEY C.1 O10).
Each solver is a fixed linear map (no data-dependent stopping).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class MultiColourSOR:
    """One operator's multicolour SOR sweeps: x_i <- x_i + omega (b_i - (A x)_i) / A_ii, colour by colour."""

    def __init__(self, A, colours, n_colours, omega=1.0):
        self.A = A.tocsr()
        self.D = self.A.diagonal()
        self.omega = omega
        self.sets = []
        for c in range(n_colours):
            rows = np.flatnonzero(colours == c)
            self.sets.append((rows, self.A[rows]))

    def sweep(self, x, b, order):
        for c in order:
            rows, Arows = self.sets[c]
            if len(rows) == 0:
                continue
            x[rows] += self.omega * (b[rows] - Arows @ x) / self.D[rows][:, None]
        return x


class Multigrid:
    """Geometric MG: `cycles` V-cycles from x = 0 (C.2 #12)."""

    def __init__(self, ops, prolongations, colours, n_colours, cycles=4, nu1=2, nu2=2, omega=1.0):
        self.ops = [A.tocsr() for A in ops]
        self.P = prolongations
        self.PT = [P.T.tocsr() for P in prolongations]
        self.sor = [MultiColourSOR(A, col, n_colours, omega) for A, col in zip(self.ops[:-1], colours[:-1])]
        self.n_colours = n_colours
        self.cycles, self.nu1, self.nu2 = cycles, nu1, nu2
        self.coarse_lu = sla.lu_factor(self.ops[-1].toarray())   # LU with partial pivoting

    def vcycle(self, l, x, b):
        if l == len(self.ops) - 1:
            return sla.lu_solve(self.coarse_lu, b)
        fwd = list(range(self.n_colours))
        for _ in range(self.nu1):
            x = self.sor[l].sweep(x, b, fwd)
        r = b - self.ops[l] @ x
        bc = self.PT[l] @ r
        ec = self.vcycle(l + 1, np.zeros_like(bc), bc)
        x = x + self.P[l] @ ec
        for _ in range(self.nu2):
            x = self.sor[l].sweep(x, b, fwd[::-1])
        return x

    def solve(self, b):
        b2 = b.reshape(b.shape[0], -1)
        x = np.zeros(b2.shape, dtype=np.result_type(b2, self.ops[0].dtype))
        for _ in range(self.cycles):
            x = self.vcycle(0, x, b2)
        return x.reshape(b.shape)


class Chebyshev:
    """Chebyshev semi-iteration, K x-updates, Jacobi preconditioner, spectrum bounds [lo, hi] of D^-1 A.

    SURVEY C.1 O10: x0 = 0, r0 = f, d0 = D^-1 r0 / theta, rho0 = 1/sigma;
    x_{k+1} = x_k + d_k; r_{k+1} = r_k - A d_k; rho_{k+1} = 1/(2 sigma - rho_k);
    d_{k+1} = rho_{k+1} rho_k d_k + (2 rho_{k+1}/delta) D^-1 r_{k+1}.
    """

    def __init__(self, A, lo, hi, iters=10):
        self.A = A.tocsr()
        self.Dinv = 1.0 / self.A.diagonal()
        self.theta = (hi + lo) / 2.0
        self.delta = (hi - lo) / 2.0
        self.sigma = self.theta / self.delta
        self.iters = iters

    def solve(self, f):
        f2 = f.reshape(f.shape[0], -1)
        Dinv = self.Dinv[:, None]
        x = np.zeros_like(f2)
        r = f2.copy()
        d = Dinv * r / self.theta
        rho = 1.0 / self.sigma
        for k in range(self.iters):
            x = x + d
            if k < self.iters - 1:
                r = r - self.A @ d
                rho_new = 1.0 / (2.0 * self.sigma - rho)
                d = rho_new * rho * d + (2.0 * rho_new / self.delta) * (Dinv * r)
                rho = rho_new
        return x.reshape(f.shape)


def wathen_bounds(space, dim):
    """Bounds of lambda(D^-1 M) for the element mass matrix (Wathen, cited at P:664).

    1-D: Q2 [1/2, 5/4], Q1 [1/2, 3/2]; tensor products multiply.
    """
    lo1, hi1 = (0.5, 1.25) if space == "q2" else (0.5, 1.5)
    return lo1**dim, hi1**dim
