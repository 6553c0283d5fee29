"""Pins for oracle/timeops.py and oracle/kkt.py (SURVEY 8(c) C.3 rows DFT, KKT, Exact solve,
Block diagonalisation, Theorem 3.1, Rank of perturbation)."""
import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import kkt, timeops
from oracle.problem import Problem
import dense_ops


def test_dft_equals_library_fft_and_roundtrips():
    rng = np.random.default_rng(0)
    for n in (2, 4, 15, 31, 63):
        x = rng.standard_normal((n, 3))
        np.testing.assert_allclose(timeops.dft(x), np.fft.fft(x, axis=0), atol=1e-12)   # numpy's e^{-2 pi i kt/n}
        np.testing.assert_allclose(timeops.idft(timeops.dft(x)).real, x, atol=1e-13)
        c = np.ones((n, 2))                                                               # constant in time -> k = 0 only
        X = timeops.dft(c)
        assert np.abs(X[1:]).max() < 1e-12 and np.allclose(X[0], n)


def test_spectrum_closed_form_and_examples():
    """d_k = 1 - exp(-2 pi i k / n_b); n_b=2 -> {0, 2}; n_b=4 -> {0, 1+i, 2, 1-i}; sum d_k = n_b."""
    np.testing.assert_allclose(timeops.spectrum(2), [0, 2], atol=1e-15)
    np.testing.assert_allclose(timeops.spectrum(4), [0, 1 + 1j, 2, 1 - 1j], atol=1e-15)
    for n in (3, 15, 63, 127):
        d = timeops.spectrum(n)
        np.testing.assert_allclose(d, 1 - np.exp(-2j * np.pi * np.arange(n) / n), atol=1e-14)
        assert abs(d.sum() - n) < 1e-11
        assert abs(d[0]) == 0.0


def test_circulant_diagonalisation():
    """C = F^{-1} D F and C^T = F^{-1} conj(D) F."""
    for n in (5, 15):
        F = timeops.dft_matrix(n)
        Finv = np.linalg.inv(F)
        D = np.diag(timeops.spectrum(n))
        np.testing.assert_allclose(Finv @ D @ F, timeops.circulant_C(n), atol=1e-13)
        np.testing.assert_allclose(Finv @ np.conj(D) @ F, timeops.circulant_C(n).T, atol=1e-13)


def test_stokes_constants_examples():
    """c1 = 0, c2 = 1 at d = 0, tau = beta = 1; c1 = 2 at d = 2."""
    c1, c2 = timeops.stokes_constants(0j, 1.0, 1.0)
    assert c1 == 0.0 and c2 == 1.0
    c1, _ = timeops.stokes_constants(2 + 0j, 1.0, 1.0)
    assert c1 == 2.0


@pytest.fixture(scope="module", params=["stokes", "oseen"])
def tiny(request):
    lo, hi = (-1.0, 1.0) if request.param == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("tiny", 2, 2, 6, problem=request.param, lo=lo, hi=hi, beta=1e-2, nu=0.05)
    return Problem(cfg, synth.wind(cfg))


def test_kkt_equals_dense_kronecker(tiny):
    """Block-by-block kkt_apply equals eq. (FinalA) assembled densely with Kronecker products."""
    A = dense_ops.dense_all_at_once(tiny, timeops.backward_euler_E(tiny.n_b))
    rng = np.random.default_rng(1)
    x = rng.standard_normal(tiny.cfg.n_dofs)
    V, P = tiny.to_reduced(x)
    y = kkt.reduced_vector(tiny, *kkt.kkt_apply_reduced(tiny, V, P))
    np.testing.assert_allclose(y, A @ kkt.reduced_vector(tiny, V, P), atol=1e-14 * np.abs(A).max() * 10)
    assert np.abs(kkt.kkt_apply(tiny, np.zeros_like(x))).max() == 0.0
    # masked entries ignored on input and zero on output
    xm = x.copy()
    xm[~synth.full_mask(tiny.cfg)] = 0.0
    np.testing.assert_array_equal(kkt.kkt_apply(tiny, x), kkt.kkt_apply(tiny, xm))
    assert np.all(kkt.kkt_apply(tiny, x)[~synth.full_mask(tiny.cfg)] == 0.0)


def test_kkt_symmetric_for_stokes_and_oseen(tiny):
    """A = A^T for Stokes AND Oseen."""
    A = dense_ops.dense_all_at_once(tiny, timeops.backward_euler_E(tiny.n_b))
    assert np.abs(A - A.T).max() < 1e-15 * np.abs(A).max() * 10


def test_block_diagonalisation(tiny):
    """(I_2 (x) F (x) I) P_C (..)^{-1}, permuted to (v, lambda, p, mu) per k, = blkdiag(G_k)."""
    n_b = tiny.n_b
    PC = dense_ops.dense_all_at_once(tiny, timeops.circulant_C(n_b))
    nb = PC.shape[0] // (2 * n_b)
    Fbig = np.kron(np.kron(np.eye(2), timeops.dft_matrix(n_b)), np.eye(nb))
    G = Fbig @ PC @ np.linalg.inv(Fbig)
    perm = dense_ops.block_perm(tiny)
    G = G[np.ix_(perm, perm)]
    d = timeops.spectrum(n_b)
    expect = sla.block_diag(*[dense_ops.G_block(tiny, d[k]) for k in range(n_b)])
    assert np.abs(G - expect).max() < 1e-12 * np.abs(expect).max()
    # Hermitian blocks, G_{n-k} = conj(G_k)
    for k in range(1, n_b):
        Gk = dense_ops.G_block(tiny, d[k])
        np.testing.assert_allclose(Gk, Gk.conj().T, atol=1e-15)
        np.testing.assert_allclose(dense_ops.G_block(tiny, d[n_b - k]), Gk.conj(), atol=1e-15)


def test_theorem_3_1_and_rank(tiny):
    """#{mu = 1} >= 2 (n_t-1)(n_v+n_p) - 2 n_v; rank(A - P_C) = 2 n_v."""
    n_b = tiny.n_b
    A = dense_ops.dense_all_at_once(tiny, timeops.backward_euler_E(n_b))
    PC = dense_ops.dense_all_at_once(tiny, timeops.circulant_C(n_b))
    nv = tiny.dim * tiny.fine.nI
    npu = tiny.fine.npu
    N = 2 * n_b * (nv + npu)
    assert np.linalg.matrix_rank(A - PC) == 2 * nv
    mu = np.linalg.eigvals(np.linalg.solve(PC, A))
    assert np.sum(np.abs(mu - 1) < 1e-6) >= N - 2 * nv


def test_exact_solve_divergence_free_and_zero_data(tiny):
    """Dense LU of A: the discrete state is divergence free, B v_j* = 0; zero data => x* = 0."""
    A = dense_ops.dense_all_at_once(tiny, timeops.backward_euler_E(tiny.n_b))
    rng = np.random.default_rng(3)
    vd = rng.standard_normal((2, tiny.n_s))
    b = kkt.build_rhs(tiny, vd)
    Vb, Pb = tiny.to_reduced(b)
    x = np.linalg.solve(A, kkt.reduced_vector(tiny, Vb, Pb))
    nb = tiny.dim * tiny.fine.nI + tiny.fine.npu
    nv = tiny.dim * tiny.fine.nI
    X = x.reshape(2, tiny.n_b, nb)
    Bm = tiny.fine.B.toarray()
    for t in range(tiny.n_b):
        assert np.abs(Bm @ X[0, t, :nv]).max() < 1e-12 * np.abs(X).max()    # v_t (half 0)
        assert np.abs(Bm @ X[1, t, :nv]).max() < 1e-12 * np.abs(X).max()    # lambda_t
    assert np.abs(np.linalg.solve(A, np.zeros(A.shape[0]))).max() == 0.0
    # the RHS touches only the adjoint-velocity rows (v0 = f = 0)
    assert np.abs(Pb).max() == 0.0 and np.abs(Vb[1]).max() == 0.0


@pytest.mark.parametrize("problem", ["stokes", "oseen"])
def test_build_rhs_equals_general_rhs_with_constant_data(problem):
    """kkt.build_rhs (C.1 O5) is the time-constant, zero-forcing, homogeneous-Dirichlet case of
    manufactured.rhs_with_data, which is pinned by the manufactured-solution convergence test
    (tests/test_oracle_gmres_mms.py): every row must agree, so a wrong factor on tau M v_d fails."""
    from oracle import manufactured
    lo, hi = (-1.0, 1.0) if problem == "oseen" else (0.0, 1.0)
    cfg = synth.small_config("rhs", 2, 4, 7, problem=problem, lo=lo, hi=hi, beta=1e-2, nu=0.05)
    w = synth.wind(cfg)
    prob = Problem(cfg, w)
    vd = np.random.default_rng(8).standard_normal((cfg.dim, prob.n_s))
    b = kkt.build_rhs(prob, vd)
    ref = manufactured.rhs_with_data(prob, np.repeat(vd[None], prob.n_b, axis=0), None, None, None, wind=w)
    np.testing.assert_allclose(b, ref, rtol=0, atol=1e-15 * np.abs(ref).max())
    assert np.abs(ref).max() > 0
