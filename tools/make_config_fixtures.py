"""Compact GPU-parity fixtures for the BASELINE cavity configs C3 / C4 from the
full oracle fields that tools/oracle_solve_ckpt.py checkpoints into
oracle_runs/ (TEST INFRASTRUCTURE ONLY; the full fields are 50-110 MB and stay
out of the repo).

tests/golden/<name>_<tag>.npz (tag = it1, it2, final) holds
  iteration, ratio, norm, r0_norm, mass   (the oracle's solve_steady scalars)
  row_sums, col_sums   per-row / per-column sums of the 20 order<=3
                       coefficients (rho, momentum, stress, heat flux parts)
  params_sub           basis params (u, theta) on every 8th cell in i and j
  cells, coeff_sub     every coefficient of 64 cells on a regular 8x8 lattice

Usage: python tools/make_config_fixtures.py C3 C4
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNS = os.path.join(ROOT, "oracle_runs")
LOW = 20  # coefficients of order <= 3 (graded-lex prefix, any M >= 3)


def lattice(n):
    s = n // 8
    idx = np.arange(s // 2, n, s)
    return (idx[:, None] * n + idx[None, :]).ravel()


def compact(c, p, n):
    c3 = c.reshape(n, n, -1)
    cells = lattice(n)
    return dict(row_sums=c3[:, :, :LOW].sum(axis=1), col_sums=c3[:, :, :LOW].sum(axis=0),
                params_sub=p.reshape(n, n, 4)[::8, ::8].copy(), cells=cells, coeff_sub=c[cells].copy())


def main():
    for name in sys.argv[1:]:
        hist = json.load(open(os.path.join(RUNS, f"{name}_port_hist.json")))
        n = hist["config"]["n"]
        # residual-ratio history of the oracle's solve_steady loop (and how it ended)
        hout = os.path.join(ROOT, "tests", "golden", f"{name}_history.json")
        json.dump(dict(ratios=[h["ratio"] for h in hist["history"]], r0_norm=hist["r0_norm"],
                       converged=bool(hist.get("converged", False)), error=hist.get("error"),
                       c_bound=hist["config"]["c_bound"]), open(hout, "w"), indent=0)
        print(hout)
        for tag in ("it1", "it2", "final"):
            path = os.path.join(RUNS, f"{name}_port_{tag}.npz")
            if not os.path.exists(path):
                continue
            z = np.load(path)
            c, p = z["coeffs"], z["params"]
            it = {"it1": 1, "it2": 2}.get(tag, hist.get("iterations"))
            h = hist["history"][it - 1]
            out = os.path.join(ROOT, "tests", "golden", f"{name}_{tag}.npz")
            np.savez_compressed(out, iteration=it, ratio=h["ratio"], norm=h["norm"], r0_norm=hist["r0_norm"],
                                target_mass=hist["target_mass"], mass=float(c[:, 0].sum() / (n * n)),
                                converged=bool(hist.get("converged", False)), c_bound=hist["config"]["c_bound"],
                                wall_s=h["wall_s"], **compact(c, p, n))
            print(out, os.path.getsize(out))


if __name__ == "__main__":
    main()
