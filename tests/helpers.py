"""Shared test inputs (seeded) and reference-style configurations."""
from __future__ import annotations

import os

import numpy as np

from oracle.api import BGK, ES_BGK, SHAKHOV, Ctx, Grid, Oracle, count, uniform_field  # noqa: F401
from paper_2206_13164_b200.synthetic import c5_field, index_degrees  # noqa: F401

HAVE_REF = os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                                       "libmomg_ref.so"))

# Hermite roots C_{M+1} as the reference computes them (max_hermite_root,
# tables.cpp:22-41); pinned against the closed forms in test_oracle_pin.py.
_CB = {}


def c_bound(M: int) -> float:
    if M not in _CB:
        _CB[M] = Oracle("port").max_hermite_root(M + 1)
    return _CB[M]


def random_grad_rep(rng, M: int, scale: float = 0.1):
    """test_helpers.hpp:12-30 restated: rho, theta ~ U[0.5,2], u ~ 0.5 U[-1,1],
    |alpha|>=2 coefficients scale*rho/sqrt(alpha!) U[-1,1], trace fixed."""
    return random_rep(rng, M, scale, uz=True)


def _fact_table(M):
    import math
    return np.array([math.factorial(a1) * math.factorial(a2) * math.factorial(a3)
                     for a1, a2, a3 in index_degrees(M)], dtype=float)


def random_rep(rng, M: int, scale: float = 0.1, uz: bool = True):
    idx = index_degrees(M)
    fact = _fact_table(M)
    n = len(idx)
    rho = rng.uniform(0.5, 2.0)
    theta = rng.uniform(0.5, 2.0)
    u = 0.5 * rng.uniform(-1, 1, 3)
    if not uz:
        u[2] = 0.0
    c = np.zeros(n)
    c[0] = rho
    for k in range(4, n):
        c[k] = scale * rho / np.sqrt(fact[k]) * rng.uniform(-1, 1)
    k1 = _find(idx, 2, 0, 0); k2 = _find(idx, 0, 2, 0); k3 = _find(idx, 0, 0, 2)
    c[k3] = -(c[k1] + c[k2])
    return c, np.array([u[0], u[1], u[2], theta])


def _find(idx, a1, a2, a3):
    return int(np.nonzero((idx[:, 0] == a1) & (idx[:, 1] == a2) & (idx[:, 2] == a3))[0][0])


def smooth_field(g: Grid, M: int, seed: int, amp: float = 0.05, uz: bool = False):
    """A seeded, smoothly varying Grad-normalized field (mild gradients keep FS
    sweeps physical): low-order Fourier modes on rho/u/theta plus c5-style
    higher coefficients."""
    rng = np.random.default_rng(seed)
    c, p = c5_field(g.nx, g.ny, M, seed=seed + 1000, coeff_sigma=1e-3 * (amp / 0.05))
    x = np.tile(g.xc, g.ny)
    y = np.repeat(g.yc, g.nx)
    ph = rng.uniform(0, 2 * np.pi, 8)
    c[:, 0] = 1.0 + amp * np.sin(2 * np.pi * x + ph[0]) * np.cos(2 * np.pi * y + ph[1])
    p[:, 0] = amp * np.sin(2 * np.pi * y + ph[2])
    p[:, 1] = amp * np.cos(2 * np.pi * x + ph[3])
    p[:, 2] = amp * np.sin(2 * np.pi * (x + y) + ph[6]) if uz else 0.0
    p[:, 3] = 1.0 + amp * np.cos(2 * np.pi * x + ph[4]) * np.sin(2 * np.pi * y + ph[5])
    return np.ascontiguousarray(c), np.ascontiguousarray(p)


def cavity_ctx(M: int, order: int = 1, model: int = BGK, kn: float = 0.1, lid: float = 0.1,
               prandtl: float = 1.0, bottom_theta: float = 1.0) -> Ctx:
    """Lid-driven / bottom-heated cavity in solver units (scenario.cpp:401-430;
    SURVEY.md §8(d) C1-C4)."""
    cb = c_bound(M)
    return Ctx(M=M, space_order=order, c_bound=cb, cfl=0.9, cfl_c_bound=cb, collision=model,
               prandtl=prandtl, knudsen=kn, viscosity_index=0.81,
               wall_speed=(0.0, 0.0, 0.0, lid), wall_theta=(1.0, 1.0, bottom_theta, 1.0))


def max_rel_diff(a, b, ref_c0=None):
    """max |a-b| / max(1, |f0|) per cell (the tolerance idiom of
    test_projection.cpp:144-145)."""
    a = np.asarray(a); b = np.asarray(b)
    if a.ndim == 1:
        return float(np.max(np.abs(a - b)) / max(1.0, abs(b[0])))
    scale = np.maximum(1.0, np.abs(b[:, :1]))
    return float(np.max(np.abs(a - b) / scale))
