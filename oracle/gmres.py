"""Restarted right-preconditioned GMRES(m) (oracle; test infrastructure only).

P:827: "GMRES iterative solver ... configured to restart every 30 iterations".
Unstated details take SURVEY C.1 O13 / C.2 #17/#19 and S:162-170: x0 = 0,
modified Gram-Schmidt Arnoldi, Givens rotations, stop when the recurrence
residual |g_{k+1}| <= tol * ||b|| (tol = 1e-6), breakdown when
h_{k+1,k} < 1e-14 ||b||.  At a restart or exit x += P^{-1}(V_k y) and the true
residual b - A x is recomputed.  History: |g_{k+1}| / ||b|| per iteration.
"""
from __future__ import annotations

import numpy as np


def gmres(apply_A, apply_Pinv, b, tol=1e-6, restart=30, max_iters=2000):
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
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta0
        k_done = 0
        stop = False
        for k in range(restart):
            w = apply_A(apply_Pinv(V[k]))
            for i in range(k + 1):                      # modified Gram-Schmidt
                H[i, k] = np.dot(w, V[i])
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            for i in range(k):                          # previous rotations
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
        # x += P^{-1} (V_k y),  H_k y = g_k  (upper triangular)
        y = np.zeros(k_done)
        for i in range(k_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k_done] @ y[i + 1:]) / H[i, i]
        u = np.zeros(n)
        for i in range(k_done):
            u = u + y[i] * V[i]
        x = x + apply_Pinv(u)
        r = b - apply_A(x)
        info["true_relres"].append(np.linalg.norm(r) / bnorm)
        if stop:
            break
        info["restarts"] += 1
    info["iterations"] = it
    return x, hist, info


def arnoldi(apply_A, apply_Pinv, v0, m):
    """m steps of the Arnoldi process on A P^{-1} (right preconditioning, as in gmres above) with modified
    Gram-Schmidt, from v0 / ||v0||.  Returns H ((k+1) x k, unrotated) for the k <= m steps done (stops at
    h_{k+1,k} < 1e-14 ||v0||).  The eigenvalues of H[:k, :k] (Ritz values) estimate those of A P^{-1},
    i.e. of P^{-1} A (similar matrices) -- the spectra of P:607-632."""
    nrm = np.linalg.norm(v0)
    V = [v0 / nrm]
    H = np.zeros((m + 1, m))
    for k in range(m):
        w = apply_A(apply_Pinv(V[k]))
        for i in range(k + 1):
            H[i, k] = np.dot(w, V[i])
            w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        if H[k + 1, k] < 1e-14 * nrm:
            return H[:k + 2, :k + 1]
        V.append(w / H[k + 1, k])
    return H
