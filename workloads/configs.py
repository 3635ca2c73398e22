"""The five BASELINE.json configurations (C1-C5) and their scaled variants.

Each builder returns a `Workload`: the forest, the patch geometry, the problem parameters, the
initial interior state q0[P][meqn][m][m] (x fastest), optional aux, and the dt policy.
Everything is deterministic (analytic ICs, no noise); randomised unit-test inputs use
numpy.random.default_rng(1308147 + k) in the tests themselves.

Readings of the paper/BASELINE wording that these builders fix are listed in DESIGN.md
("Readings"), numbered as in SURVEY.md §8(c.7).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .forests import (Forest, OUTFLOW, WALL, brick, cell_centres, forest_refined, forest_uniform,
                      periodic_unit_square, walled_unit_square)

# problem kinds / limiters (numbering shared by DESIGN.md, include/fc.h and oracle/oracle.h,
# which each define them independently)
ADV_CONST, ADV_EDGEVEL_CAPA, SWE_ROE, EULER_ROE, EULER_HLLE = 0, 1, 2, 3, 4
LIM_NONE, LIM_MINMOD, LIM_MC = 0, 1, 2

CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")


@dataclass
class Workload:
    name: str
    forest: Forest
    m: int
    meqn: int
    maux: int
    kind: int
    params: tuple            # (p0, p1): (u, v) | (unused) | (g, 0) | (gamma, efix)
    q0: np.ndarray | None    # [P, meqn, m, m] (None until materialised for lazy workloads)
    aux: np.ndarray | None   # [P, maux, m+4, m+4] or None
    steps: int
    dt0: float
    dt_policy: str           # "fixed" | "cfl"
    cfl_target: float = 0.9
    limiter: int = LIM_MC
    method2: int = 2
    method3: int = 2
    cfl_reject: float = 1.0
    reflux: int = 0          # conservative coarse/fine flux correction
    mbc: int = 2
    info: dict = field(default_factory=dict)
    ic: object = None        # ic(forest, m, p0, p1) -> q0[p1-p0] (analytic, deterministic)

    def q0_range(self, p0: int, p1: int) -> np.ndarray:
        """Initial state of patches [p0, p1) only (multi-rank runs build just their shard)."""
        if self.q0 is not None:
            return np.ascontiguousarray(self.q0[p0:p1])
        return self.ic(self.forest, self.m, p0, p1)

    def materialise(self):
        if self.q0 is None:
            self.q0 = self.ic(self.forest, self.m, 0, self.num_patches)
        return self

    @property
    def num_patches(self) -> int:
        return self.forest.num_patches

    @property
    def cells(self) -> int:
        return self.num_patches * self.m * self.m

    def next_dt(self, dt: float, cfl: float) -> float:
        """Clawpack's variable-dt rule dt_{n+1} = dt_n * target / CFL_n."""
        if self.dt_policy == "fixed" or cfl <= 0.0:
            return dt
        return dt * self.cfl_target / cfl


def _gaussian_ic(forest: Forest, m: int) -> np.ndarray:
    X, Y = cell_centres(forest, m)
    q = np.exp(-100.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))
    return q[:, None, :, :].astype(np.float64)


def c1(level: int = 2, m: int = 8, steps: int = 20) -> Workload:
    """C1: periodic advection u=1, v=0.5, uniform level 2, m=8 (BASELINE configs[0])."""
    f = forest_uniform(periodic_unit_square(), level)
    dx = 0.5 ** level / m
    dt = 0.9 * dx / 1.0
    return Workload("C1" if (level, m) == (2, 8) else f"C1_L{level}_m{m}", f, m, 1, 0, ADV_CONST,
                    (1.0, 0.5), _gaussian_ic(f, m), None, steps, dt, "fixed")


def c2(base_level: int = 3, m: int = 16, steps: int = 100, radius: float = 0.25) -> Workload:
    """C2: same physics as C1 on a static two-level forest: a level-`base` quadrant is refined
    iff its centre is at distance < radius from (0.5, 0.5) (reading 11: 100 patches)."""
    f = forest_refined(periodic_unit_square(), base_level,
                       lambda t, xc, yc, h: (xc - 0.5) ** 2 + (yc - 0.5) ** 2 < radius ** 2)
    dx_fine = 0.5 ** (base_level + 1) / m
    dt = 0.9 * dx_fine
    return Workload("C2" if (base_level, m) == (3, 16) else f"C2_L{base_level}_m{m}", f, m, 1, 0,
                    ADV_CONST, (1.0, 0.5), _gaussian_ic(f, m), None, steps, dt, "fixed")


def c3_ic(f: Forest, m: int, p0: int, p1: int) -> np.ndarray:
    X, Y = cell_centres(_subforest(f, p0, p1), m)
    q = np.zeros((p1 - p0, 3, m, m))
    q[:, 0] = np.where((X - 0.5) ** 2 + (Y - 0.5) ** 2 < 0.2 ** 2, 2.0, 1.0)
    return q


def c3(level: int = 6, m: int = 32, steps: int = 200, lazy: bool = False) -> Workload:
    """C3: shallow water (g=1) radial dam break with reflecting walls, uniform level 6, m=32."""
    f = forest_uniform(walled_unit_square(WALL), level)
    q = None if lazy else c3_ic(f, m, 0, f.num_patches)
    dx = 0.5 ** level / m
    dt0 = 0.9 * dx / math.sqrt(1.0 * 2.0)   # max(|u|+c) = sqrt(g*h) at h = 2
    return Workload("C3" if (level, m) == (6, 32) else f"C3_L{level}_m{m}", f, m, 3, 0, SWE_ROE,
                    (1.0, 0.0), q, None, steps, dt0, "cfl", ic=c3_ic)


GAMMA = 1.4


def euler_shock_bubble_state(X, Y, x_shock: float = 1.29):
    """Mach-3 planar shock at x_shock moving +x into rho=1, p=1 gas at rest, plus a rho=0.1,
    p=1 bubble of radius 0.2 at (1.5, 0.5) (reading 13).  Returns conserved (rho, rhou, rhov, E)."""
    g = GAMMA
    rho_post, p_post = 27.0 / 7.0, 31.0 / 3.0          # Rankine-Hugoniot at M = 3, gamma = 1.4
    u_post = 20.0 / 9.0 * math.sqrt(g)
    post = X < x_shock
    bubble = (X - 1.5) ** 2 + (Y - 0.5) ** 2 < 0.2 ** 2
    rho = np.where(post, rho_post, np.where(bubble, 0.1, 1.0))
    u = np.where(post, u_post, 0.0)
    p = np.where(post, p_post, 1.0)
    E = p / (g - 1.0) + 0.5 * rho * u * u
    return rho, rho * u, np.zeros_like(rho), E


def _subforest(f: Forest, p0: int, p1: int) -> Forest:
    return Forest(f.levels[p0:p1], f.tree_ids[p0:p1], f.ix[p0:p1], f.iy[p0:p1], f.conn)


def c5_ic(f: Forest, m: int, p0: int, p1: int, x_shock: float = 1.29) -> np.ndarray:
    out = np.empty((p1 - p0, 4, m, m))
    step = 16384
    for a in range(p0, p1, step):            # chunked: the full C5 IC is 2.15 GB
        b = min(p1, a + step)
        sf = _subforest(f, a, b)
        X, Y = cell_centres(sf, m)
        X = X + sf.tree_ids[:, None, None].astype(np.float64)   # tree t covers [t, t+1] x [0, 1]
        for k, v in enumerate(euler_shock_bubble_state(X, Y, x_shock)):
            out[a - p0:b - p0, k] = v
    return out


def c5(level: int = 8, m: int = 16, steps: int = 100, x_shock: float = 1.29,
       lazy: bool = False) -> Workload:
    """C5: 2D Euler (gamma=1.4, Roe + Harten-Hyman), 4-tree brick [0,4]x[0,1], outflow,
    uniform level 8 in each tree (262,144 patches of m=16, 67.1M cells)."""
    conn = brick(4, 1, bc=OUTFLOW)
    f = forest_uniform(conn, level)
    ic = lambda ff, mm, p0, p1: c5_ic(ff, mm, p0, p1, x_shock)
    q = None if lazy else ic(f, m, 0, f.num_patches)
    dx = 0.5 ** level / m
    rho_post, p_post = 27.0 / 7.0, 31.0 / 3.0
    smax = 20.0 / 9.0 * math.sqrt(GAMMA) + math.sqrt(GAMMA * p_post / rho_post)
    dt0 = 0.9 * dx / smax
    return Workload("C5" if (level, m) == (8, 16) else f"C5_L{level}_m{m}", f, m, 4, 0, EULER_ROE,
                    (GAMMA, 1.0), q, None, steps, dt0, "cfl", ic=ic)


def c4(base_level: int = 4, m: int = 16, steps: int = 500, band: float = 0.6) -> Workload:
    from .cubed_sphere import c4_workload
    return c4_workload(base_level=base_level, m=m, steps=steps, band=band)


def make_config(name: str, **kw) -> Workload:
    return {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[name](**kw)
