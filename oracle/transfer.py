"""Multigrid transfer operators (oracle; test infrastructure only).

The paper uses "a geometric multigrid method" without stating the
transfers; reading SURVEY C.2 #12: prolongation P is nodal interpolation of the
coarse finite-element function at the fine nodes, restriction is P^T.  P is
built here by literally evaluating the coarse Lagrange basis at fine-node
positions (1-D), then taking the tensor product (x fastest) and restricting
rows/columns to the unknown sets of the two levels.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import q1_basis_1d, q2_basis_1d


def _interp_1d(n_cells_coarse, order):
    """P1d[f, I] = coarse basis function I evaluated at fine node f (1-D, full grids)."""
    basis = q2_basis_1d if order == 2 else q1_basis_1d
    n_fine_nodes = order * 2 * n_cells_coarse + 1
    n_coarse_nodes = order * n_cells_coarse + 1
    P = np.zeros((n_fine_nodes, n_coarse_nodes))
    for f in range(n_fine_nodes):
        x = f / (2.0 * order)                    # position in units of the coarse cell width
        e = min(int(np.floor(x)), n_cells_coarse - 1)
        xi = x - e
        vals, _ = basis(np.array([xi]))
        for a in range(order + 1):
            P[f, order * e + a] += vals[a, 0]
    P[np.abs(P) < 1e-15] = 0.0
    return P


def prolongation(dim, n_cells_coarse, order, fine_rows, coarse_cols):
    """Prolongation coarse -> fine on the unknown sets, as a CSR matrix."""
    P1 = sp.csr_matrix(_interp_1d(n_cells_coarse, order))
    P = P1
    for _ in range(dim - 1):
        P = sp.kron(P1, P, format="csr")         # later axes are slower: kron(P_y, P_x)
    return P[fine_rows][:, coarse_cols].tocsr()
