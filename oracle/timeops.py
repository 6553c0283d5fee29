"""Circulant time structure (oracle; test infrastructure only).

P:288-301: C is the circulant with first column c_1 = (1, -1, 0, ..., 0)^T,
C = F^{-1} D F with D = diag(F c_1).  Reading SURVEY C.2 #2: F is the
unnormalised DFT with kernel omega^{kt}, omega = exp(-2 pi i / n_b); F^{-1}
carries 1/n_b.  Hence d_k = 1 - omega^k.
P:399-403: constants c_{j,1}, c_{j,2}; the printed c_{j,1} has a garbled
exponent, read as d_{j,c}^2 (pinned by G_j = T_l Z_j T_r).
"""
from __future__ import annotations

import numpy as np


def omega(n_b):
    return np.exp(-2j * np.pi / n_b)


def dft_matrix(n_b):
    """F_{kt} = omega^{kt} = exp(-2 pi i (k t mod n_b) / n_b) (plain definition, k, t = 0..n_b-1)."""
    k = np.arange(n_b)
    return np.exp(-2j * np.pi * (np.outer(k, k) % n_b) / n_b)


def circulant_C(n_b):
    """C of P:290-295: 1 on the diagonal, -1 on the subdiagonal and in the top-right corner."""
    C = np.eye(n_b)
    for j in range(1, n_b):
        C[j, j - 1] = -1.0
    C[0, n_b - 1] = -1.0
    return C


def backward_euler_E(n_b):
    """E of P:110-117: 1 on the diagonal, -1 on the subdiagonal."""
    E = np.eye(n_b)
    for j in range(1, n_b):
        E[j, j - 1] = -1.0
    return E


def spectrum(n_b):
    """d = diag(D) = F c_1 with c_1 the first column of C."""
    c1 = circulant_C(n_b)[:, 0]
    return dft_matrix(n_b) @ c1


def dft(x, ks=None):
    """Naive DFT along axis 0: xhat_k = sum_t x_t omega^{k t}; only rows `ks` if given."""
    n_b = x.shape[0]
    F = dft_matrix(n_b)
    if ks is not None:
        F = F[np.asarray(ks)]
    return np.tensordot(F, x, axes=(1, 0))


def idft(xhat):
    """Inverse DFT along axis 0: x_t = (1/n_b) sum_k xhat_k omega^{-k t}."""
    n_b = xhat.shape[0]
    return np.tensordot(np.conj(dft_matrix(n_b)), xhat, axes=(1, 0)) / n_b


def stokes_constants(d, tau, beta):
    """(c_{j,1}, c_{j,2}) of P:401-402, with the squared reading of d_{j,c} in c_{j,1} (C.2 #1)."""
    dr, dc = d.real, d.imag
    c1 = dr / np.sqrt(tau**2 / beta + dc**2)
    c2 = 1.0 / np.sqrt(1.0 / beta + dc**2 / tau**2)
    return c1, c2
