"""Q2-Q1 Taylor-Hood finite elements on a uniform box mesh (oracle; test infrastructure only).

Follows P:77-92: Q2-Q1 elements, M the velocity mass matrix, L the
discretisation of -nu Lap + w.grad (L = nu K + N), B the
discretised NEGATIVE divergence (B_ij = -int psi_i d_c phi_j, C.2 #7),
pressure-space matrices M_p, K_p, N_p (C.2 #9).

Every matrix is assembled by a plain element loop (vectorised over elements
with numpy) with 3^d-point Gauss quadrature on each cell.
Matrices are returned on the FULL node grid (boundary and pinned nodes
included); elimination (Dirichlet velocity, pinned pressure node 0, P:92,
C.2 #5/#6) is done by restricting rows and columns to the unknown sets.

Node numbering: lexicographic with x fastest.  Q2 scalar grid has
(2 N_c + 1)^d nodes, Q1 grid (N_c + 1)^d.
"""
from __future__ import annotations

import itertools
import numpy as np
import scipy.sparse as sp


# ---------------------------------------------------------------- reference element
def gauss3():
    """3-point Gauss-Legendre rule mapped to [0, 1]."""
    xi = np.array([-np.sqrt(3.0 / 5.0), 0.0, np.sqrt(3.0 / 5.0)])
    w = np.array([5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0])
    return (xi + 1.0) / 2.0, w / 2.0


def q2_basis_1d(xi):
    """Quadratic Lagrange basis on [0,1] with nodes 0, 1/2, 1: values and derivatives, shape (3, len(xi))."""
    xi = np.asarray(xi, dtype=float)
    v = np.stack([2 * (xi - 0.5) * (xi - 1), 4 * xi * (1 - xi), 2 * xi * (xi - 0.5)])
    d = np.stack([4 * xi - 3, 4 - 8 * xi, 4 * xi - 1])
    return v, d


def q1_basis_1d(xi):
    """Linear Lagrange basis on [0,1]: values and derivatives, shape (2, len(xi))."""
    xi = np.asarray(xi, dtype=float)
    return np.stack([1 - xi, xi]), np.stack([-np.ones_like(xi), np.ones_like(xi)])


def tensor_basis(dim, basis_1d, pts_1d):
    """Tensor-product basis at tensor points.

    Returns values (n_loc, n_q) and reference gradients (n_loc, n_q, dim);
    local index a_0 + k a_1 + k^2 a_2 (x fastest), point index likewise.
    """
    v1, d1 = basis_1d(pts_1d)
    k, m = v1.shape
    n_loc, n_q = k**dim, m**dim
    val = np.ones((n_loc, n_q))
    grad = np.ones((n_loc, n_q, dim))
    for i, a in enumerate(itertools.product(range(k), repeat=dim)):
        a = a[::-1]  # a[axis], x fastest
        for q, b in enumerate(itertools.product(range(m), repeat=dim)):
            b = b[::-1]
            for axis in range(dim):
                val[i, q] *= v1[a[axis], b[axis]]
                for c in range(dim):
                    grad[i, q, c] *= (d1 if c == axis else v1)[a[axis], b[axis]]
    return val, grad


def tensor_weights(dim, w1):
    w = np.ones(len(w1) ** dim)
    for q, b in enumerate(itertools.product(range(len(w1)), repeat=dim)):
        for axis in range(dim):
            w[q] *= w1[b[axis]]
    return w


# ---------------------------------------------------------------- mesh connectivity
def element_nodes(dim, n_cells, order):
    """Global node numbers of every element's local nodes, shape (E, (order+1)^dim).

    order=2: Q2 grid with 2 N_c + 1 nodes per direction; order=1: Q1 grid.
    Elements numbered lexicographically, x fastest.
    """
    n1 = order * n_cells + 1
    e = np.arange(n_cells**dim)
    ecoord = [(e // n_cells**axis) % n_cells for axis in range(dim)]
    cols = []
    for a in itertools.product(range(order + 1), repeat=dim):
        a = a[::-1]
        g = np.zeros_like(e)
        for axis in range(dim):
            g += (order * ecoord[axis] + a[axis]) * n1**axis
        cols.append(g)
    return np.stack(cols, axis=1)


def _assemble(rows, cols, emats, shape):
    """Sum element matrices emats (E, nr, nc) (or (nr, nc) broadcast) into a CSR matrix."""
    E = rows.shape[0]
    if emats.ndim == 2:
        emats = np.broadcast_to(emats, (E,) + emats.shape)
    R = np.broadcast_to(rows[:, :, None], emats.shape).reshape(-1)
    C = np.broadcast_to(cols[:, None, :], emats.shape).reshape(-1)
    A = sp.coo_matrix((emats.reshape(-1), (R, C)), shape=shape).tocsr()
    A.sum_duplicates()
    return A


class Level:
    """One uniform mesh level: N_c cells per direction on [lo, hi]^dim."""

    def __init__(self, dim, n_cells, lo, hi):
        self.dim, self.n_cells, self.lo, self.hi = dim, n_cells, lo, hi
        self.h = (hi - lo) / n_cells
        self.n1q2, self.n1q1 = 2 * n_cells + 1, n_cells + 1
        self.n_s, self.n_p = self.n1q2**dim, self.n1q1**dim
        self.e2 = element_nodes(dim, n_cells, 2)
        self.e1 = element_nodes(dim, n_cells, 1)
        gp, gw = gauss3()
        self.w = tensor_weights(dim, gw)
        self.phi, self.dphi = tensor_basis(dim, q2_basis_1d, gp)   # (9|27, nq), (.., nq, dim)
        self.psi, self.dpsi = tensor_basis(dim, q1_basis_1d, gp)   # (4|8, nq)

    # -- unknown sets (elimination)
    def q2_interior(self):
        n = self.n1q2
        node = np.arange(self.n_s)
        ok = np.ones(self.n_s, dtype=bool)
        for axis in range(self.dim):
            i = (node // n**axis) % n
            ok &= (i > 0) & (i < n - 1)
        return np.flatnonzero(ok)

    def q1_unknowns(self):
        return np.arange(1, self.n_p)  # node 0 (corner at lo^d) is pinned (C.2 #6)

    # -- constant-coefficient operators on the full grid
    def mass_q2(self):
        em = self.h**self.dim * np.einsum("q,iq,jq->ij", self.w, self.phi, self.phi)
        return _assemble(self.e2, self.e2, em, (self.n_s, self.n_s))

    def stiff_q2(self):
        em = self.h ** (self.dim - 2) * np.einsum("q,iqc,jqc->ij", self.w, self.dphi, self.dphi)
        return _assemble(self.e2, self.e2, em, (self.n_s, self.n_s))

    def mass_q1(self):
        em = self.h**self.dim * np.einsum("q,iq,jq->ij", self.w, self.psi, self.psi)
        return _assemble(self.e1, self.e1, em, (self.n_p, self.n_p))

    def stiff_q1(self):
        em = self.h ** (self.dim - 2) * np.einsum("q,iqc,jqc->ij", self.w, self.dpsi, self.dpsi)
        return _assemble(self.e1, self.e1, em, (self.n_p, self.n_p))

    def div(self):
        """B = [B_0, ..., B_{d-1}], (B_c)_{ij} = -int psi_i d_c phi_j (negative divergence)."""
        blocks = []
        for c in range(self.dim):
            em = -self.h ** (self.dim - 1) * np.einsum("q,iq,jq->ij", self.w, self.psi, self.dphi[:, :, c])
            blocks.append(_assemble(self.e1, self.e2, em, (self.n_p, self.n_s)))
        return sp.hstack(blocks).tocsr()

    # -- convection with a Q2 nodal wind (P:86 w.grad)
    def _wind_at_gauss(self, wind_q2):
        """w_h at each element's Gauss points, shape (E, nq, dim); w_h = Q2 nodal interpolant."""
        we = wind_q2[:, self.e2]                     # (dim, E, 9)
        return np.einsum("ceL,Lq->eqc", we, self.phi)

    def conv_q2(self, wind_q2):
        """N_ij = int phi_i (w_h . grad phi_j) on the Q2 scalar space."""
        wq = self._wind_at_gauss(wind_q2)
        em = self.h ** (self.dim - 1) * np.einsum("q,iq,eqc,jqc->eij", self.w, self.phi, wq, self.dphi)
        return _assemble(self.e2, self.e2, em, (self.n_s, self.n_s))

    def conv_q1(self, wind_q2):
        """N_p,ij = int psi_i (w_h . grad psi_j) on the Q1 pressure space (C.2 #9)."""
        wq = self._wind_at_gauss(wind_q2)
        em = self.h ** (self.dim - 1) * np.einsum("q,iq,eqc,jqc->eij", self.w, self.psi, wq, self.dpsi)
        return _assemble(self.e1, self.e1, em, (self.n_p, self.n_p))


def restrict(A, rows, cols):
    """Elimination: keep the unknown rows and columns of a full-grid matrix."""
    return A[rows][:, cols].tocsr()


def inject_wind(wind_fine, dim, n_cells_fine):
    """Coarse-level wind nodal values = fine values at the coarse nodes (coarse node I <-> fine node 2I)."""
    nf = 2 * n_cells_fine + 1
    nc = n_cells_fine + 1
    idx = np.arange(nc**dim)
    fine = np.zeros_like(idx)
    for axis in range(dim):
        fine += 2 * ((idx // nc**axis) % nc) * nf**axis
    return wind_fine[:, fine]
