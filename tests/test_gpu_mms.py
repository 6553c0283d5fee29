"""NEXT-2 on the GPU: the paper's manufactured Stokes problem through the C ABI.

aao_build_rhs_general (time-dependent v_d and f, inhomogeneous Dirichlet data by lifting, v_0) is
compared element by element with the oracle's right-hand side (oracle/manufactured.rhs_with_data,
itself pinned by the oracle's direct-solve convergence test); the GPU GMRES solution is compared with
the oracle's sparse direct solution of the same discrete system, and its nodal error against the
exact v falls at the rate the oracle pin asserts."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("nc,nt", [(4, 8), (8, 16), (16, 9)])
def test_rhs_general_matches_oracle(nc, nt):
    _torch()
    from oracle import manufactured
    from oracle.problem import Problem
    from paper_2405_18964_b200 import Context
    cfg = synth.mms_config(nc, nt)
    ctx = Context.from_config(cfg, None)
    vd, f, g, v0 = synth.mms_inputs(cfg)
    b = ctx.build_rhs_general(vd, f, g, v0).cpu().numpy()
    bo = manufactured.rhs_with_data(Problem(cfg), vd, f, g, v0)
    assert rel(b, bo) <= 1e-13
    # partial data: forcing only, and v_d only (null pointers = 0)
    assert rel(ctx.build_rhs_general(None, f, None, None).cpu().numpy(),
               manufactured.rhs_with_data(Problem(cfg), None, f, None, None)) <= 1e-13
    assert rel(ctx.build_rhs_general(vd, None, None, None).cpu().numpy(),
               manufactured.rhs_with_data(Problem(cfg), vd, None, None, None)) <= 1e-13


def _velocity_error(cfg, x):
    """max over t_m of the RMS nodal error of v at the interior nodes, relative (oracle/manufactured.py)."""
    X = synth.q2_coords(cfg)
    inner = synth.q2_interior_mask(cfg)
    tau = cfg.T / cfg.n_t
    blocks = x.reshape(2, cfg.n_b, -1)
    err = ref = 0.0
    for j in range(cfg.n_b):
        ve = synth.mms_velocity(X[0][inner], X[1][inner], (j + 1) * tau, cfg.T)
        vh = np.stack([blocks[0, j, c * cfg.n_s:(c + 1) * cfg.n_s][inner] for c in range(2)])
        err = max(err, np.sqrt(np.mean((vh - ve) ** 2)))
        ref = max(ref, np.sqrt(np.mean(ve ** 2)))
    return err / ref


@pytest.mark.parametrize("nc,nt,tol,xtol,etol", [(4, 8, 1e-10, 1e-5, 1e-3), (8, 16, 1e-10, 1e-5, 1e-3),
                                                    (16, 32, 3e-9, None, None)])
def test_manufactured_solution_gpu_gmres(nc, nt, tol, xtol, etol, monkeypatch):
    """GPU GMRES(30) with the linear preconditioner reaches the direct solution of the same discrete system;
    the system is ill-conditioned (nu = 1 on [-1,1]^2), so a residual of 1e-10 leaves ~1e-7 in x and the
    16 x 16 x 32 case (restarted GMRES(30) crawls there: 1e-7 after 3000 iterations, ~2e-9 after 12000, and how
    far it gets within the cap moves with the rounding order of the preconditioner's stencil sums -- 3e-9 is
    asked, the check it feeds needs the 1e-3 discretisation error; the oracle's sparse direct solve takes
    minutes there) is checked against the exact solution only."""
    _torch()
    from oracle.manufactured import solve_manufactured
    from paper_2405_18964_b200 import Context
    cfg = synth.mms_config(nc, nt)
    # restart update x += P^{-1}(V y) (not the stored-Z sum): the tighter attainable accuracy at 1e-9..1e-10
    monkeypatch.setenv("AAO_STORE_Z", "0")
    ctx = Context.from_config(cfg, None)
    b = ctx.build_rhs_general(*synth.mms_inputs(cfg))
    x, info, hist, rc = ctx.gmres_solve(b, tol=tol, restart=30, max_iters=12000)
    assert info["converged"], info
    xg = x.cpu().numpy()
    e = _velocity_error(cfg, xg)
    if xtol is not None:
        ev_o, _, xo = solve_manufactured(nc, nt, full=True)
        assert rel(xg, xo) <= xtol                      # same discrete solution as the direct solve
        assert abs(e - ev_o) <= etol * ev_o
    _ERRS[(nc, nt)] = e


_ERRS = {}


def test_manufactured_gpu_convergence_rate():
    """the GPU solutions' nodal errors fall under (h, tau) halving as the oracle pin asserts."""
    if len(_ERRS) < 3:
        pytest.skip("needs the three manufactured solves above")
    e = [_ERRS[k] for k in ((4, 8), (8, 16), (16, 32))]
    assert e[0] > 4 * e[1] > 16 * e[2] and e[2] < 2e-3


# ---------------------------------------------------------------- the Oseen lid-driven cavity
@pytest.mark.parametrize("nc,nt", [(8, 8), (16, 9)])
def test_cavity_rhs_matches_oracle(nc, nt):
    """Lifting with convection: the lid data enter the state rows through nu K + N (un-eliminated)."""
    _torch()
    from oracle import manufactured
    from oracle.problem import Problem
    from paper_2405_18964_b200 import Context
    cfg = synth.cavity_config(nc, nt)
    w = synth.cavity_wind(cfg)
    ctx = Context.from_config(cfg, w)
    vd, f, g, v0 = synth.cavity_inputs(cfg)
    b = ctx.build_rhs_general(vd, f, g, v0).cpu().numpy()
    bo = manufactured.rhs_with_data(Problem(cfg, w), vd, f, g, v0, wind=w)
    assert rel(b, bo) <= 1e-13


def test_cavity_solve_gpu():
    """Algorithm 2 + FGMRES(10) solves the cavity optimality system; the converged x
    satisfies the oracle's A x = b (true residual through oracle/kkt.py)."""
    torch = _torch()
    from oracle import kkt
    from oracle.problem import Problem
    from paper_2405_18964_b200 import Context
    cfg = synth.cavity_config(16, 9)
    w = synth.cavity_wind(cfg)
    ctx = Context.from_config(cfg, w, nonlinear=True, inner_eps=1e-2, inner_maxit=60)
    b = ctx.build_rhs_general(*synth.cavity_inputs(cfg))
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-8, restart=10, max_iters=200)
    assert info["converged"], info
    bn = b.cpu().numpy()
    r = bn - kkt.kkt_apply(Problem(cfg, w), x.cpu().numpy())
    assert np.linalg.norm(r) <= 1e-7 * np.linalg.norm(bn)
