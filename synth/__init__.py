"""Seeded synthetic inputs for the five BASELINE.json workloads (c1..c5).

This module is the ONLY code shared by the oracle (`oracle/`) and the CUDA
path (`paper_2405_18964_b200/`).  It holds problem *data* -- configuration
records, desired-state fields, the Oseen wind, random probe vectors and the
grid masks that say which entries are unknowns -- and none of the method's
arithmetic (no operator, transform, solver or right-hand-side assembly).

Recipe:
  * seed = 240518964 + cfg_index (c1 -> 1, ..., c5 -> 5; c2's second beta and
    every c4 n_t share their config's seed), numpy PCG64 (default_rng).
  * T = 1, v0 = 0, f = 0, homogeneous Dirichlet velocity; v_d constant in time.
  * c1/c2/c4: v_d = (psi_y, -psi_x) * (1 + 0.1 xi), psi = x^2(1-x)^2 y^2(1-y)^2,
    xi ~ N(0,1) i.i.d. per velocity nodal DOF.
  * c3: per component sum of 8 sine modes with N(0,1) amplitudes, (k,l) ~ U{1..4}^2;
    wind w = (2y(1-x^2), -2x(1-y^2)) on [-1,1]^2.
  * c5: v_d = curl A, A_c = sum of 6 sine modes, (k,l,n) ~ U{1..3}^3.
No public dataset is involved: the paper's workloads are synthetic PDE data.
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED_BASE = 240518964


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int            # 1..5 (c1..c5); selects the seed
    dim: int
    n_cells: int          # N_c per direction
    x_lo: float
    x_hi: float
    n_t: int              # time steps; n_b = n_t - 1 unknown time blocks
    T: float
    beta: float
    nu: float
    problem: str          # "stokes" | "oseen"

    # ---- derived sizes (structure only) ----
    @property
    def n_b(self) -> int:
        return self.n_t - 1

    @property
    def n_f(self) -> int:
        return self.n_b // 2 + 1

    @property
    def n1q2(self) -> int:
        return 2 * self.n_cells + 1

    @property
    def n1q1(self) -> int:
        return self.n_cells + 1

    @property
    def n_s(self) -> int:
        return self.n1q2 ** self.dim

    @property
    def n_v(self) -> int:
        return self.dim * self.n_s

    @property
    def n_p(self) -> int:
        return self.n1q1 ** self.dim

    @property
    def n_dofs(self) -> int:
        """N = 2 (n_t - 1)(n_v + n_p), counting every grid node (C.2 #5)."""
        return 2 * self.n_b * (self.n_v + self.n_p)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index


def _c(name, index, dim, n_cells, lo, hi, n_t, beta, nu, problem):
    return Config(name, index, dim, n_cells, lo, hi, n_t, 1.0, beta, nu, problem)


CONFIGS = {
    "c1": _c("c1", 1, 2, 8, 0.0, 1.0, 16, 1e-2, 1e-2, "stokes"),
    "c2": _c("c2", 2, 2, 64, 0.0, 1.0, 64, 1e-2, 1e-2, "stokes"),
    "c2b": _c("c2b", 2, 2, 64, 0.0, 1.0, 64, 1e-4, 1e-2, "stokes"),
    "c3": _c("c3", 3, 2, 128, -1.0, 1.0, 128, 1e-3, 1.0 / 20.0, "oseen"),
    "c4_32": _c("c4_32", 4, 2, 256, 0.0, 1.0, 32, 1e-2, 1e-2, "stokes"),
    "c4_64": _c("c4_64", 4, 2, 256, 0.0, 1.0, 64, 1e-2, 1e-2, "stokes"),
    "c4_128": _c("c4_128", 4, 2, 256, 0.0, 1.0, 128, 1e-2, 1e-2, "stokes"),
    "c4_256": _c("c4_256", 4, 2, 256, 0.0, 1.0, 256, 1e-2, 1e-2, "stokes"),
    "c4_512": _c("c4_512", 4, 2, 256, 0.0, 1.0, 512, 1e-2, 1e-2, "stokes"),
    "c5": _c("c5", 5, 3, 32, 0.0, 1.0, 64, 1e-3, 1e-2, "stokes"),
}


def small_config(name: str, dim: int, n_cells: int, n_t: int, problem: str = "stokes",
                 beta: float = 1e-2, nu: float = 1e-2, lo: float = 0.0, hi: float = 1.0,
                 index: int = 1, T: float = 1.0) -> Config:
    """Reduced-size configs for parity cases (several tiles + ragged tails)."""
    return Config(name, index, dim, n_cells, lo, hi, n_t, T, beta, nu, problem)


# ----------------------------------------------------------------------------
# grid structure (node coordinates and masks) -- no method arithmetic
# ----------------------------------------------------------------------------
def q2_coords(cfg: Config) -> list[np.ndarray]:
    """Coordinates of the full Q2 grid, lexicographic with x fastest; list per axis."""
    n1 = cfg.n1q2
    g = cfg.x_lo + (cfg.x_hi - cfg.x_lo) * np.arange(n1) / (n1 - 1)
    node = np.arange(cfg.n_s)
    return [g[(node // n1**axis) % n1] for axis in range(cfg.dim)]


def q2_interior_mask(cfg: Config) -> np.ndarray:
    """True where a Q2 scalar node is an unknown (interior; Dirichlet elsewhere)."""
    n = cfg.n1q2
    i = np.arange(n)
    inner = (i > 0) & (i < n - 1)
    m = inner
    for _ in range(cfg.dim - 1):
        m = np.multiply.outer(inner, m)
    return m.reshape(-1)


def q1_unknown_mask(cfg: Config) -> np.ndarray:
    """True where a Q1 pressure node is an unknown (all but node 0, the pinned corner)."""
    m = np.ones(cfg.n_p, dtype=bool)
    m[0] = False
    return m


def unknown_mask(cfg: Config) -> np.ndarray:
    """Mask over one paper-order spatial block [v comps | p] (length n_v + n_p)."""
    return np.concatenate([np.tile(q2_interior_mask(cfg), cfg.dim), q1_unknown_mask(cfg)])


def full_mask(cfg: Config) -> np.ndarray:
    """Mask over a whole paper-order space-time vector (length N)."""
    return np.tile(unknown_mask(cfg), 2 * cfg.n_b)


# ----------------------------------------------------------------------------
# problem data
# ----------------------------------------------------------------------------
def desired_state(cfg: Config) -> np.ndarray:
    """v_d as Q2 nodal values on the full grid, shape (dim, n_s), time-constant."""
    rng = np.random.default_rng(cfg.seed)
    X = q2_coords(cfg)
    if cfg.index in (1, 2, 4):
        x, y = X[0], X[1]
        psi_y = x**2 * (1 - x) ** 2 * 2 * y * (1 - y) * (1 - 2 * y)
        psi_x = 2 * x * (1 - x) * (1 - 2 * x) * y**2 * (1 - y) ** 2
        xi = rng.standard_normal((2, cfg.n_s))
        return np.stack([psi_y, -psi_x]) * (1.0 + 0.1 * xi)
    if cfg.index == 3:
        x, y = X[0], X[1]
        out = np.zeros((2, cfg.n_s))
        for c in range(2):
            a = rng.standard_normal(8)
            kl = rng.integers(1, 5, size=(8, 2))
            for m in range(8):
                out[c] += a[m] * np.sin(kl[m, 0] * np.pi * (x + 1) / 2) * np.sin(kl[m, 1] * np.pi * (y + 1) / 2)
        return out
    if cfg.index == 5:
        x, y, z = X[0], X[1], X[2]
        pi = np.pi
        # A_c = sum_m a sin(k pi x) sin(l pi y) sin(n pi z); curl A analytic
        dA = np.zeros((3, 3, cfg.n_s))  # dA[c, axis] = d A_c / d x_axis
        for c in range(3):
            a = rng.standard_normal(6)
            kln = rng.integers(1, 4, size=(6, 3))
            for m in range(6):
                k, l, n = kln[m]
                sx, sy, sz = np.sin(k * pi * x), np.sin(l * pi * y), np.sin(n * pi * z)
                cx, cy, cz = np.cos(k * pi * x), np.cos(l * pi * y), np.cos(n * pi * z)
                dA[c, 0] += a[m] * k * pi * cx * sy * sz
                dA[c, 1] += a[m] * l * pi * sx * cy * sz
                dA[c, 2] += a[m] * n * pi * sx * sy * cz
        return np.stack([dA[2, 1] - dA[1, 2], dA[0, 2] - dA[2, 0], dA[1, 0] - dA[0, 1]])
    raise ValueError(cfg.name)


def wind(cfg: Config) -> np.ndarray | None:
    """Q2 nodal wind (dim, n_s) for Oseen configs; None for Stokes."""
    if cfg.problem != "oseen":
        return None
    X = q2_coords(cfg)
    x, y = X[0], X[1]
    return np.stack([2 * y * (1 - x**2), -2 * x * (1 - y**2)])


def probe_vector(cfg: Config, seed_offset: int = 0) -> np.ndarray:
    """r ~ N(0,1) on unknown entries and 0 on masked entries (paper order, length N)."""
    rng = np.random.default_rng(cfg.seed * 1000 + 17 + seed_offset)
    r = rng.standard_normal(cfg.n_dofs)
    r[~full_mask(cfg)] = 0.0
    return r


# ----------------------------------------------------------------------------
# the paper's manufactured Stokes problem: data only (exact state, forcing, desired state);
# both the oracle (direct solve) and the GPU path (aao_build_rhs_general) consume these arrays
# ----------------------------------------------------------------------------
def mms_config(n_cells: int, n_t: int, beta: float = 1e-2, nu: float = 1.0, T: float = 1.0) -> Config:
    """Omega = [-1,1]^2; nu = 1, T = 1 for the manufactured solution.  The paper's Stokes
    experiments keep v_d and f with nu = 1e-2 and T = 10: mms_config(n, n_t, beta, 1e-2, 10)."""
    return small_config(f"mms{n_cells}x{n_t}", 2, n_cells, n_t, lo=-1.0, hi=1.0, beta=beta, nu=nu, T=T)


def mms_velocity(x, y, t, T=1.0):
    """v = e^{T-t} [20 x y^3, 5 x^4 - 5 y^4]."""
    e = np.exp(T - t)
    return np.stack([e * 20 * x * y**3, e * (5 * x**4 - 5 * y**4)])


def mms_forcing(x, y, t, T=1.0):
    """f of P:818-820."""
    e = np.exp(T - t)
    a = (x**2 - 1) ** 2 * (y**2 - 1)
    b = (x**2 - 1) * (y**2 - 1) ** 2
    return np.stack([e * (-20 * x * y**3 - 2 * y * a) + 2 * y * a,
                     e * (5 * (y**4 - x**4) + 2 * x * b) - 2 * x * b])


def mms_desired(x, y, t, T, beta):
    """v_d of P:815-817."""
    e = np.exp(T - t)
    c1 = 4 * beta * (y * (2 * (3 * x**2 - 1) * (y**2 - 1) + 3 * (x**2 - 1) ** 2))
    c2 = 4 * beta * (-x * (3 * (y**2 - 1) ** 2 + 2 * (x**2 - 1) * (3 * y**2 - 1)))
    d1 = e * (20 * x * y**3 + 2 * beta * y * ((x**2 - 1) ** 2 * (y**2 - 7) - 4 * (3 * x**2 - 1) * (y**2 - 1) + 2))
    d2 = e * (5 * (x**4 - y**4) - 2 * beta * x * ((y**2 - 1) ** 2 * (x**2 - 7) - 4 * (x**2 - 1) * (3 * y**2 - 1) - 2))
    return np.stack([c1 + d1, c2 + d2])


def mms_inputs(cfg: Config):
    """Nodal data on the full Q2 grid at t_m = m tau: v_d (n_b, d, n_s) and f (n_b, d, n_s) for m = 1..n_b,
    Dirichlet data g (n_b + 1, d, n_s) for m = 0..n_b (exact v; only boundary entries are data), and
    v0 (d, n_s) = v(t = 0) on every node (initial and boundary data given by v)."""
    X = q2_coords(cfg)
    x, y = X[0], X[1]
    tau = cfg.T / cfg.n_t
    n_b = cfg.n_b
    vd = np.stack([mms_desired(x, y, m * tau, cfg.T, cfg.beta) for m in range(1, n_b + 1)])
    f = np.stack([mms_forcing(x, y, m * tau, cfg.T) for m in range(1, n_b + 1)])
    g = np.stack([mms_velocity(x, y, m * tau, cfg.T) for m in range(0, n_b + 1)])
    return vd, f, g, g[0].copy()


# ----------------------------------------------------------------------------
# the paper's Oseen lid-driven cavity: data only
# ----------------------------------------------------------------------------
def cavity_config(n_cells: int, n_t: int, beta: float = 1e-3, nu: float = 1e-2, T: float = 10.0) -> Config:
    """Omega = [-1,1]^2, Oseen; nu = 1e-2 and T = 10 "for this and all subsequent experiments"
    (P:827), kept for the Oseen runs ("the same iterative solver and associated settings")."""
    return small_config(f"cavity{n_cells}x{n_t}", 2, n_cells, n_t, problem="oseen", lo=-1.0, hi=1.0,
                        beta=beta, nu=nu, index=3, T=T)


def cavity_wind(cfg: Config) -> np.ndarray:
    """Two-vortex wind of P:908-913 (DESIGN.md reading: the second vortex uses (x1 + 1/2), the printed
    (x1 - 1/2) does not vanish at its own centre c_2 = 1)."""
    X = q2_coords(cfg)
    x1, x2 = X[0], X[1]
    a, b = (100 / 99) ** 2, (100 / 49) ** 2
    c1 = 1 - np.sqrt((100 / 49 * (x1 - 0.5)) ** 2 + (100 / 99 * x2) ** 2)
    c2 = 1 - np.sqrt((100 / 49 * (x1 + 0.5)) ** 2 + (100 / 99 * x2) ** 2)
    w = np.zeros((2, cfg.n_s))
    m1, m2 = c1 >= 0, (c2 >= 0) & ~(c1 >= 0)
    w[0, m1] = c1[m1] * a * x2[m1]
    w[1, m1] = -c1[m1] * b * (x1[m1] - 0.5)
    w[0, m2] = c2[m2] * a * x2[m2]
    w[1, m2] = c2[m2] * b * (x1[m2] + 0.5)
    return w


def cavity_inputs(cfg: Config):
    """v_d, f (time-independent) on t_1..t_{n_b}, lid data h = [1, 0] on x2 = 1 at
    t_0..t_{n_b}, v0 = [1, 0] where |x1| < x2; same shapes as mms_inputs."""
    X = q2_coords(cfg)
    x1, x2 = X[0], X[1]
    q = (1 - x1**4) * (1 - x2**4)
    vd = np.stack([2 * x2 * q + np.where(x2 >= 0.8, 5 * x2 - 4, 0.0), -2 * x1 * q])
    f = np.stack([-20 * x1 * x2**3 - 2 * x2 * (x1**2 - 1) ** 2 * (x2**2 - 1),
                  5 * (x2**4 - x1**4) + 2 * x1 * (x1**2 - 1) * (x2**2 - 1) ** 2])
    lid = np.isclose(x2, 1.0)
    h = np.stack([np.where(lid, 1.0, 0.0), np.zeros(cfg.n_s)])
    v0 = np.stack([np.where((x1 > -x2) & (x1 < x2), 1.0, 0.0), np.zeros(cfg.n_s)])
    n_b = cfg.n_b
    return (np.repeat(vd[None], n_b, axis=0), np.repeat(f[None], n_b, axis=0),
            np.repeat(h[None], n_b + 1, axis=0), v0)
