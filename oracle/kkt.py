"""The all-at-once KKT matrix A of eq. (FinalA), P:120-149 (oracle; test infrastructure only).

A = [[tau I, E^T], [E, -tau/beta I]] (x) [[M, 0], [0, 0]]
    + tau [[0, 0], [I, 0]] (x) [[L, B^T], [B, 0]]
    + tau [[0, I], [0, 0]] (x) [[L^T, B^T], [B, 0]]

acting on x = [(v_j, p_j)_{j=1..n_b} ; (lambda_j, mu_j)_{j=1..n_b}], n_b = n_t - 1
(reading SURVEY C.2 #3/#4).  M, L act per velocity component (I_d (x) M_s).
Applied term by term exactly as written; E acts along the time index.
"""
from __future__ import annotations

import numpy as np

from .timeops import backward_euler_E


def _vel(op, V):
    """Apply a scalar Q2 operator to every (time, component) slice of V (n_b, d, nI)."""
    n_b, d, nI = V.shape
    return (op @ V.reshape(-1, nI).T).T.reshape(n_b, d, nI)


def _BT(prob, P):
    n_b = P.shape[0]
    return (prob.fine.BT @ P.T).T.reshape(n_b, prob.dim, -1)


def _B(prob, V):
    n_b = V.shape[0]
    return (prob.fine.B @ V.reshape(n_b, -1).T).T


def kkt_apply_reduced(prob, V, P):
    """y = A x on reduced arrays V (2, n_b, d, nI), P (2, n_b, npu)."""
    tau, beta = prob.tau, prob.beta
    f = prob.fine
    E = backward_euler_E(prob.n_b)
    L = prob.L()
    LT = L.T.tocsr()
    v, lam = V[0], V[1]
    p, mu = P[0], P[1]
    Mv, Mlam = _vel(f.Ms, v), _vel(f.Ms, lam)
    time = lambda Tm, X: np.tensordot(Tm, X, axes=(1, 0))
    Y = np.zeros_like(V)
    Q = np.zeros_like(P)
    # term 1: [[tau I, E^T], [E, -tau/beta I]] (x) [[M,0],[0,0]]
    Y[0] = tau * Mv + time(E.T, Mlam)
    Y[1] = time(E, Mv) - (tau / beta) * Mlam
    # term 2: tau [[0,0],[I,0]] (x) [[L, B^T],[B, 0]]   (state rows)
    Y[1] += tau * (_vel(L, v) + _BT(prob, p))
    Q[1] += tau * _B(prob, v)
    # term 3: tau [[0,I],[0,0]] (x) [[L^T, B^T],[B, 0]]   (adjoint rows)
    Y[0] += tau * (_vel(LT, lam) + _BT(prob, mu))
    Q[0] += tau * _B(prob, lam)
    return Y, Q


def kkt_apply(prob, x):
    """y = A x on paper-order full vectors (masked entries ignored on input, 0 on output)."""
    V, P = prob.to_reduced(x)
    Y, Q = kkt_apply_reduced(prob, V, P)
    return prob.from_reduced(Y, Q)


def build_rhs(prob, vd_q2):
    """Right-hand side for v0 = 0, f = 0, h = 0.

    Adjoint-velocity rows (half 0): tau * (M_full v_d)|_interior at every block j
    (from tau M (v_d - v) in the adjoint equation); all other rows 0.
    """
    f = prob.fine
    V = np.zeros((2, prob.n_b, prob.dim, f.nI))
    P = np.zeros((2, prob.n_b, f.npu))
    for c in range(prob.dim):
        V[0, :, c] = prob.tau * (f.Ms_full_rows @ vd_q2[c])
    return prob.from_reduced(V, P)


def dense_kkt(prob):
    """Dense A assembled literally from eq. (FinalA) with Kronecker products (tiny sizes; tests)."""
    tau, beta, n_b = prob.tau, prob.beta, prob.n_b
    f = prob.fine
    d = prob.dim
    I_d = np.eye(d)
    M = np.kron(I_d, f.Ms.toarray())
    L = np.kron(I_d, prob.L().toarray())
    B = f.B.toarray()
    nv, npu = M.shape[0], B.shape[0]
    Z = np.zeros
    MM = np.block([[M, Z((nv, npu))], [Z((npu, nv)), Z((npu, npu))]])
    S1 = np.block([[L, B.T], [B, Z((npu, npu))]])
    S2 = np.block([[L.T, B.T], [B, Z((npu, npu))]])
    E = backward_euler_E(n_b)
    I = np.eye(n_b)
    O = np.zeros((n_b, n_b))
    T1 = np.block([[tau * I, E.T], [E, -(tau / beta) * I]])
    T2 = tau * np.block([[O, O], [I, O]])
    T3 = tau * np.block([[O, I], [O, O]])
    return np.kron(T1, MM) + np.kron(T2, S1) + np.kron(T3, S2)


def reduced_vector(prob, V, P):
    """Flatten reduced arrays in the dense_kkt ordering: half, time, [v comps, p]."""
    parts = []
    for h in range(2):
        for t in range(prob.n_b):
            parts.append(V[h, t].reshape(-1))
            parts.append(P[h, t])
    return np.concatenate(parts)
