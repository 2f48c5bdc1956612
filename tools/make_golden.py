"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, i.e.
/root/reference/proj/src compiled against oracle/shim) -- run in the build
container where /root/reference exists; the fixtures are committed so the
tests (and the GPU box) never need the reference sources.

  primitives.npz   project / grad_normalize / half+full flux / face + wall flux /
                   collision (BGK, Shakhov, ES-BGK) on seeded random reps, M = 3, 5
  fields.npz       residual and one fast_sweep_step on seeded 8x8 / 9x7 fields
                   (orders 1, 2; with rhs and a permuted sweep order), restrict /
                   fas on 8x8, M = 3, 5
  c1.npz           C1 (32^2, M=3, order 1, BGK Kn 0.1, lid 0.1, FS to 1e-8):
                   iteration count, residual history, final field
  c2.npz           C2 (128^2, M=5, order 2, BGK Kn 0.1, NMG 4 levels to 1e-8):
                   iteration count, history, final macroscopic fields
                   (from tests/golden/configs_C2_port.json + field: the
                   restatement, itself pinned bitwise to the reference)
Usage: python tools/make_golden.py [--with-c2]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import (BGK, ES_BGK, SHAKHOV, Ctx, Grid, cavity_ctx, random_grad_rep,  # noqa: E402
                     smooth_field, uniform_field)
from oracle.api import Oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def primitives(R):
    out = {}
    for M in (3, 5):
        rng = np.random.default_rng(100 + M)
        reps = [random_grad_rep(rng, M) for _ in range(4)]
        out[f"M{M}_c"] = np.array([r[0] for r in reps])
        out[f"M{M}_p"] = np.array([r[1] for r in reps])
        to = reps[1][1] + np.array([0.1, -0.2, 0.05, 0.3])
        out[f"M{M}_to"] = to
        out[f"M{M}_project"] = R.project(M, reps[0][0], reps[0][1], to)
        cc = reps[2][0].copy(); cc[1] += 0.02; cc[4] += 0.01
        out[f"M{M}_gn_in"] = cc
        out[f"M{M}_gn_c"], out[f"M{M}_gn_p"] = R.grad_normalize(M, cc, reps[2][1])
        for axis in (0, 1):
            out[f"M{M}_half{axis}_up"] = R.half_flux(M, reps[0][0], reps[0][1], axis, True)
            out[f"M{M}_half{axis}_lo"] = R.half_flux(M, reps[0][0], reps[0][1], axis, False)
            out[f"M{M}_full{axis}"] = R.full_flux(M, reps[0][0], reps[0][1], axis)
            out[f"M{M}_face{axis}"], out[f"M{M}_face{axis}_p"] = R.face_flux(
                M, reps[0][0], reps[0][1], reps[3][0], reps[3][1], axis, R.max_hermite_root(M + 1))
            out[f"M{M}_wall{axis}"], _ = R.wall_flux(M, reps[3][0], reps[3][1], axis, 1, 0.1, 1.2)
        for name, model, pr in (("bgk", BGK, 1.0), ("shakhov", SHAKHOV, 2.0 / 3.0), ("es", ES_BGK, 2.0 / 3.0)):
            out[f"M{M}_coll_{name}"] = R.collision(Ctx(M=M, collision=model, prandtl=pr, knudsen=0.3),
                                                   reps[1][0], reps[1][1])
        out[f"M{M}_cbound"] = np.array(R.max_hermite_root(M + 1))
    np.savez_compressed(os.path.join(OUT, "primitives.npz"), **out)


FIELD_CASES = [(3, 1, BGK, 8, 8), (3, 2, BGK, 9, 7), (5, 1, SHAKHOV, 8, 8), (5, 2, BGK, 8, 8)]


def fields(R):
    out = {}
    for (M, order, model, nx, ny) in FIELD_CASES:
        tag = f"M{M}o{order}m{model}_{nx}x{ny}"
        g = Grid.uniform(nx, ny, 1.0, 1.1)
        ctx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                         bottom_theta=1.3)
        ctx.c_bound = ctx.cfl_c_bound = R.max_hermite_root(M + 1)
        c, p = smooth_field(g, M, seed=nx * 10 + ny + M, amp=0.08, uz=(M == 5))
        out[tag + "_c"], out[tag + "_p"] = c, p
        out[tag + "_res"] = R.residual(ctx, g, c, p)
        out[tag + "_fs_c"], out[tag + "_fs_p"], _ = R.fast_sweep(ctx, g, c, p)
        rhs = (c * 1e-3, p.copy())
        out[tag + "_fsr_c"], out[tag + "_fsr_p"], _ = R.fast_sweep(ctx, g, c, p, rhs=rhs, sweep_order=[2, 0, 3, 1])
        if nx % 2 == 0 and ny % 2 == 0:
            cg = g.coarsen()
            cc, cp = R.restrict_solution(M, g, c, p, cg)
            out[tag + "_rs_c"], out[tag + "_rs_p"] = cc, cp
            out[tag + "_rr"] = R.restrict_residual(M, g, -out[tag + "_res"], p, p, cg, cp)
            after = cc.copy(); after[:, 4:] += 1e-4
            out[tag + "_fas_c"], out[tag + "_fas_p"] = R.fas_correct(M, g, c, p, cg, cc, cp, after, cp)
    np.savez_compressed(os.path.join(OUT, "fields.npz"), **out)


def c1(R):
    M = 3
    g = Grid.uniform(32, 32)
    ctx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    ctx.c_bound = ctx.cfl_c_bound = R.max_hermite_root(M + 1)
    c, p = uniform_field(g, M)
    fc, fp, rep = R.solve_steady(ctx, g, c, p, solver=1, tol=1e-8)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), coeffs=fc, params=fp, history=rep["history"],
                        iterations=rep["iterations"], c_bound=ctx.c_bound)


def c2():
    # the reference's own run when present (python tools/run_oracle_configs.py C2 --ref,
    # 99 iterations, ~20 min on one core), else the bitwise-pinned port's
    kind = "reference" if os.path.exists(os.path.join(OUT, "configs_C2_reference.json")) else "port"
    js = os.path.join(OUT, f"configs_C2_{kind}.json")
    fz = os.path.join(OUT, f"configs_C2_{kind}_field.npz")
    if not (os.path.exists(js) and os.path.exists(fz)):
        print("C2 oracle run missing: python tools/run_oracle_configs.py C2")
        return
    rep = json.load(open(js))
    z = np.load(fz)
    c, p = z["coeffs"], z["params"]
    q = np.stack([3 * c[:, 10] + c[:, 13] + c[:, 15], 3 * c[:, 16] + c[:, 11] + c[:, 18]], axis=1)
    macro = np.concatenate([c[:, :1], p, q, 2 * c[:, 4:5], c[:, 5:6], 2 * c[:, 7:8]], axis=1)
    np.savez_compressed(os.path.join(OUT, "c2.npz"), macro=macro, history=np.array(rep["history"]),
                        iterations=rep["iterations"], c_bound=rep["config"]["c_bound"],
                        oracle_seconds=rep["wall_s"], kind=kind)


if __name__ == "__main__":
    R = Oracle("reference")
    os.makedirs(OUT, exist_ok=True)
    primitives(R)
    fields(R)
    c1(R)
    if "--with-c2" in sys.argv:
        c2()
    print(sorted(os.listdir(OUT)))
