"""Dense matrices written literally from the paper's displays, for oracle pins on tiny sizes.

Each function transcribes one display; they are deliberately independent of
the block-by-block code paths in oracle/ (that is what makes them pins).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from oracle import timeops


def spatial(prob):
    """Dense reduced M (I_d (x) M_s), L, B, M_p, K_p, K (I_d (x) K_s), L_p on the finest level."""
    f = prob.fine
    I_d = np.eye(prob.dim)
    M = np.kron(I_d, f.Ms.toarray())
    K = np.kron(I_d, f.Ks.toarray())
    L = np.kron(I_d, prob.L().toarray())
    B = f.B.toarray()
    return dict(M=M, K=K, L=L, B=B, Mp=f.Mp.toarray(), Kp=f.Kp.toarray(), Lp=prob.Lp().toarray())


def G_block(prob, d):
    """G_j of eq. (SubBlockG), order (v, lambda, p, mu)."""
    s = spatial(prob)
    tau, beta = prob.tau, prob.beta
    M, L, B = s["M"], s["L"], s["B"]
    nv, npu = M.shape[0], B.shape[0]
    Z = lambda a, b: np.zeros((a, b))
    return np.block([
        [tau * M, np.conj(d) * M + tau * L.T, Z(nv, npu), tau * B.T],
        [d * M + tau * L, -(tau / beta) * M, tau * B.T, Z(nv, npu)],
        [Z(npu, nv), tau * B, Z(npu, npu), Z(npu, npu)],
        [tau * B, Z(npu, nv), Z(npu, npu), Z(npu, npu)],
    ])


def T_matrices(prob, d, c2):
    """T_j^(l), T_j^(r) of P:380-391."""
    s = spatial(prob)
    nv, npu = s["M"].shape[0], s["B"].shape[0]
    tau = prob.tau
    st = np.sqrt(tau)
    dc = d.imag
    Iv, Ip = np.eye(nv), np.eye(npu)
    Zvv, Zvp, Zpv, Zpp = (np.zeros((nv, nv)), np.zeros((nv, npu)), np.zeros((npu, nv)), np.zeros((npu, npu)))
    Tl = np.block([
        [st * Iv, Zvv, Zvp, Zvp],
        [(dc / st) * 1j * Iv, (st / c2) * Iv, Zvp, Zvp],
        [Zpv, Zpv, st * c2 * Ip, Zpp],
        [Zpv, Zpv, (dc * c2 / st) * 1j * Ip, st * Ip],
    ])
    Tr = np.block([
        [st * Iv, -(dc / st) * 1j * Iv, Zvp, Zvp],
        [Zvv, (st / c2) * Iv, Zvp, Zvp],
        [Zpv, Zpv, st * c2 * Ip, -(dc * c2 / st) * 1j * Ip],
        [Zpv, Zpv, Zpp, st * Ip],
    ])
    return Tl, Tr


def Z_block(prob, c1, c2):
    """Z_j of P:392-397."""
    s = spatial(prob)
    M, L, B = s["M"], s["L"], s["B"]
    nv, npu = M.shape[0], B.shape[0]
    Zvp, Zpp = np.zeros((nv, npu)), np.zeros((npu, npu))
    X = c1 * M + c2 * L
    return np.block([
        [M, X, Zvp, B.T],
        [X, -M, B.T, Zvp],
        [Zvp.T, B, Zpp, Zpp],
        [B, Zvp.T, Zpp, Zpp],
    ])


def dense_all_at_once(prob, time_matrix):
    """A of eq. (FinalA) with E replaced by `time_matrix` (E -> A, C -> P_C), ordering half, t, [v, p]."""
    s = spatial(prob)
    M, L, B = s["M"], s["L"], s["B"]
    nv, npu = M.shape[0], B.shape[0]
    Z = np.zeros
    MM = np.block([[M, Z((nv, npu))], [Z((npu, nv)), Z((npu, npu))]])
    S1 = np.block([[L, B.T], [B, Z((npu, npu))]])
    S2 = np.block([[L.T, B.T], [B, Z((npu, npu))]])
    n_b = prob.n_b
    I, O = np.eye(n_b), np.zeros((n_b, n_b))
    E = time_matrix
    T1 = np.block([[prob.tau * I, E.T], [E, -(prob.tau / prob.beta) * I]])
    return (np.kron(T1, MM) + prob.tau * np.kron(np.block([[O, O], [I, O]]), S1)
            + prob.tau * np.kron(np.block([[O, I], [O, O]]), S2))


def block_perm(prob):
    """Permutation taking the (half, k, [v, p]) ordering to per-k blocks (v, lambda, p, mu)."""
    s = spatial(prob)
    nv, npu = s["M"].shape[0], s["B"].shape[0]
    nb = nv + npu
    n_b = prob.n_b
    idx = []
    for k in range(n_b):
        for h, rng in ((0, range(nv)), (1, range(nv)), (0, range(nv, nb)), (1, range(nv, nb))):
            idx.extend((h * n_b + k) * nb + i for i in rng)
    return np.array(idx)


class DenseSolve:
    """x = A^{-1} b with a dense LU (drop-in for MG / Chebyshev in the oracle)."""

    def __init__(self, A):
        self.lu = sla.lu_factor(np.asarray(A.toarray() if hasattr(A, "toarray") else A))

    def solve(self, b):
        return sla.lu_solve(self.lu, b)


def stokes_constants(prob, d):
    return timeops.stokes_constants(d, prob.tau, prob.beta)
