"""Seeded synthetic moment fields (bench / test inputs, not an oracle).

``c5_field`` follows the C5 throughput-field recipe of SURVEY.md §8(d) /
BASELINE.json configs[4]: rho ~ U[0.9,1.1], u_x,u_y ~ N(0,0.05), u_z = 0,
theta ~ U[0.9,1.1], f_0 = rho, f_{e_d} = 0, f_alpha ~ N(0,1e-3)*0.5^|alpha| for
|alpha| >= 2, then the Grad trace is fixed by f_{2e3} = -(f_{2e1}+f_{2e2})
(as test_helpers.hpp:27-28) so every cell has grad_defect = 0.  The paper's
cavity benchmarks use deterministic uniform-Maxwellian starts instead
(grid.hpp:79-85); this field stands in for "seeded random fields" at any size.
Cell order is j-outer, i-inner (grid.hpp:64).  numpy's PCG64 replaces the
survey's mt19937_64: the arrays are generated once per run and handed to both
the CPU oracle and the GPU, so RNG implementations cannot diverge.
"""
from __future__ import annotations

import numpy as np


def index_degrees(M: int) -> np.ndarray:
    """Degrees of the graded-lex multi-indices (multi_index.hpp:31-34)."""
    out = []
    for deg in range(M + 1):
        for a1 in range(deg, -1, -1):
            for a2 in range(deg - a1, -1, -1):
                out.append((a1, a2, deg - a1 - a2))
    return np.array(out, dtype=np.int64)


def c5_field(nx: int, ny: int, M: int, seed: int = 2206, coeff_sigma: float = 1e-3,
             u_sigma: float = 0.05, uz: bool = False):
    rng = np.random.default_rng(seed)
    idx = index_degrees(M)
    n = len(idx)
    deg = idx.sum(axis=1)
    cells = nx * ny
    rho = rng.uniform(0.9, 1.1, cells)
    params = np.zeros((cells, 4))
    params[:, 0] = rng.normal(0.0, u_sigma, cells)
    params[:, 1] = rng.normal(0.0, u_sigma, cells)
    if uz:
        params[:, 2] = rng.normal(0.0, u_sigma, cells)
    params[:, 3] = rng.uniform(0.9, 1.1, cells)
    coeffs = rng.normal(0.0, coeff_sigma, (cells, n)) * (0.5 ** deg)[None, :]
    coeffs[:, deg < 2] = 0.0
    coeffs[:, 0] = rho
    k1 = _find(idx, 2, 0, 0); k2 = _find(idx, 0, 2, 0); k3 = _find(idx, 0, 0, 2)
    coeffs[:, k3] = -(coeffs[:, k1] + coeffs[:, k2])
    return np.ascontiguousarray(coeffs), np.ascontiguousarray(params)


def c5_rhs(nx: int, ny: int, M: int, seed: int = 2207):
    """Seeded non-empty rhs in the cell basis (coarse-level semantics):
    same distribution as c5_field scaled by 1e-3."""
    c, p = c5_field(nx, ny, M, seed=seed)
    return c * 1e-3, p


def _find(idx, a1, a2, a3):
    return int(np.nonzero((idx[:, 0] == a1) & (idx[:, 1] == a2) & (idx[:, 2] == a3))[0][0])
