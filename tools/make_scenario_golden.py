"""Golden fixtures of the front end's wire formats, made by the REFERENCE itself
(TEST INFRASTRUCTURE ONLY; needs /root/reference and `make -C oracle ref`).

The reference's scenario.cpp is compiled in place into oracle/_ref/libmomg_ref.so
against oracle/shim/json.hpp (its own test_scenario.cpp passes against the
shim: `make -C oracle ref-tests`).  This script drives it through the harness
entry points mo_ref_config_echo / mo_ref_run_scenario / mo_ref_export_field
(oracle/ref_harness.cpp) and writes tests/golden/scenario/:

  parse_cases.json        JSON documents -> (status, message) or config_echo text
  <case>/config.json      a scenario document (output_dir relative: out/<case>)
  <case>/history.tsv      run_scenario's outputs (seconds columns are wall time)
  <case>/report.txt
  <case>/field.tsv.gz     (absent for a run that ends in NonConvergence)
  export_<tag>.npz        a seeded field + the reference's export_field text of it

Usage: python tools/make_scenario_golden.py
"""
import ctypes as C
import gzip
import json
import os
import shutil
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.api import MoErr, Grid, uniform_field  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "scenario")
LIB = os.path.join(ROOT, "oracle", "_ref", "libmomg_ref.so")

# documents for parse_config + config_echo (the reference's test_scenario.cpp
# documents first, then edge cases of the JSON handling)
PARSE_DOCS = [
    """{
    "scenario": "single_lid",
    "collision": "bgk",
    "moment_order": 5,
    "nx": 32, "ny": 24,
    "order": 2,
    "solver": "fs",
    "levels": 3,
    "threads": 4,
    "knudsen": 1.0,
    "init": {"density": 0.0891, "velocity": [1.0, -2.0]},
    "walls": {"top": {"speed": 25.0}},
    "domain": {"Ly": 4.815e-7},
    "s3": 6,
    "output_dir": "elsewhere"
  }""",
    '{"levels": "auto"}', "{}", '{"knudsen_number": 0.1}', '{"walls": {"front": {}}}',
    '{"init": {"pressure": 1.0}}', '{"walls": {"top": {"velocity": 3.0}}}', '{"nx": "sixteen"}',
    '{"levels": 0}', '{"cfl": 1.5}', '{"moment_order": 2}', '{"init": {"temperature": -1.0}}',
    '{"solver": "rk4"}', '{"collision": "boltzmann"}', '{ "nx": }',
    # presets
    '{"scenario": "four_lid"}', '{"scenario": "bottom_heated"}', '{"scenario": "single_lid"}',
    '{"scenario": "triple_lid"}',
    # types: integers vs numbers vs booleans
    '{"nx": 32.0}', '{"nx": true}', '{"cfl": 1}', '{"cfl": false}', '{"prandtl": 0.7, "collision": "es_bgk"}',
    '{"tol": 1e-10, "max_iterations": 500}', '{"max_iterations": -1}', '{"threads": 0}',
    # levels
    '{"levels": " 3"}', '{"levels": "3 "}', '{"levels": "+2"}', '{"levels": "-2"}', '{"levels": "0"}',
    '{"levels": "x"}', '{"levels": 2.0}', '{"levels": 4}', '{"levels": ""}', '{"levels": "99999999999"}',
    # nested objects
    '{"domain": 1.0}', '{"domain": {"Lx": 2e-6, "Ly": 1e-6}}', '{"domain": {"Lz": 1.0}}',
    '{"walls": []}', '{"walls": {"top": 5}}', '{"walls": {"left": {"speed": -3.5, "temperature": 250.0}}}',
    '{"walls": {"bottom": {"temperature": 0.0}}}',
    '{"init": {"velocity": [1.0]}}', '{"init": {"velocity": [1.0, 2.0, 3.0]}}',
    '{"init": {"velocity": [1.0, 2.0, 3.0, 4.0]}}', '{"init": {"velocity": [1.0, "a"]}}',
    '{"init": {"velocity": 1.0}}', '{"init": {"density": 0.0}}', '{"init": 3}',
    # several unknown keys: reported in key order
    '{"zeta": 1, "alpha": 2}', '{"walls": {"zz": {}, "aa": {}}}',
    # cycle / gas / strings
    '{"s1": 0, "s2": 3, "s3": 1, "gamma": 2}', '{"s3": 0}', '{"gamma": 0}', '{"s1": -1}',
    '{"viscosity_index": 0.5, "molecule_mass": 4.65e-26}', '{"molecule_mass": 0}',
    '{"output_dir": 5}', '{"scenario": 3}', '{"collision": 1}', '{"solver": "euler"}', '{"order": 3}',
    '{"nx": 0}', '{"ny": -4}', '{"moment_order": 8, "order": 2, "cfl": 0.5}',
    # documents that are not objects / not JSON
    "[]", "3", '"text"', "", "{", '{"nx": 1,}', '{"cfl": NaN}', '{"nx": 01}', "{} {}",
    '{"output_dir": "d\\u00e9j\\u00e0 vu"}', '{"nx": 16, "nx": 8}',
]

# scenarios run to the end by the reference (small grids: seconds each on one core)
CASES = {
    # the reference's own test_scenario.cpp run (NMG, M=3, 16^2)
    "single_lid_m3": {"scenario": "single_lid", "moment_order": 3, "nx": 16, "ny": 16, "solver": "nmg"},
    # BGK, M=4, second order, a 2:1 cavity, bottom-heated walls, 2 levels
    "bottom_heated_o2": {"scenario": "bottom_heated", "collision": "bgk", "prandtl": 1.0, "moment_order": 4,
                         "nx": 32, "ny": 16, "order": 2, "solver": "nmg", "levels": 2,
                         "domain": {"Ly": 5e-7}},
    # four moving walls, Shakhov M=5, the FS solver
    "four_lid_fs": {"scenario": "four_lid", "moment_order": 5, "nx": 8, "ny": 8, "solver": "fs"},
    # ES-BGK, moving start, a hot moving lid
    "custom_es": {"collision": "es_bgk", "prandtl": 0.7, "moment_order": 3, "nx": 16, "ny": 16,
                  "knudsen": 0.5, "init": {"velocity": [10.0, -5.0]},
                  "walls": {"top": {"speed": 30.0, "temperature": 300.0}}, "solver": "nmg", "levels": 2},
    # the Euler smoother to a loose tolerance
    "euler_loose": {"scenario": "single_lid", "moment_order": 3, "nx": 8, "ny": 8, "solver": "euler",
                    "tol": 1e-3},
    # a hierarchy too deep for the grid: ConfigError before anything is written
    "config_err": {"scenario": "single_lid", "moment_order": 3, "nx": 16, "ny": 8, "solver": "nmg", "levels": 2},
    # NonConvergence at the iteration cap: partial history and report, no field
    "fail_cap": {"scenario": "single_lid", "moment_order": 3, "nx": 16, "ny": 16, "solver": "nmg",
                 "max_iterations": 2},
}


def lib():
    L = C.CDLL(LIB)
    L.mo_ref_config_echo.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(MoErr)]
    L.mo_ref_run_scenario.argtypes = [C.c_char_p, C.POINTER(MoErr)]
    return L


def parse_cases(L):
    out = []
    for doc in PARSE_DOCS:
        buf = C.create_string_buffer(1 << 16)
        err = MoErr()
        rc = L.mo_ref_config_echo(doc.encode(), buf, len(buf), C.byref(err))
        out.append({"doc": doc, "rc": rc, "msg": err.msg.decode(errors="replace") if rc else "",
                    "echo": buf.value.decode() if rc == 0 else ""})
    return out


def run_cases(L):
    cwd = os.getcwd()
    tmp = tempfile.mkdtemp()
    try:
        os.chdir(tmp)
        for name, doc in CASES.items():
            doc = dict(doc, output_dir=f"out/{name}")
            text = json.dumps(doc, indent=1)
            err = MoErr()
            rc = L.mo_ref_run_scenario(text.encode(), C.byref(err))
            d = os.path.join(OUT, name)
            os.makedirs(d, exist_ok=True)
            open(os.path.join(d, "config.json"), "w").write(text + "\n")
            json.dump({"rc": rc, "msg": err.msg.decode(errors="replace")}, open(os.path.join(d, "status.json"), "w"))
            for f in ("history.tsv", "report.txt"):
                if os.path.exists(os.path.join("out", name, f)):
                    shutil.copy(os.path.join("out", name, f), os.path.join(d, f))
            fld = os.path.join("out", name, "field.tsv")
            if os.path.exists(fld):
                with open(fld, "rb") as src, open(os.path.join(d, "field.tsv.gz"), "wb") as raw, \
                        gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as dst:
                    dst.write(src.read())
            print(name, "rc", rc, err.msg.decode(errors="replace")[:80])
    finally:
        os.chdir(cwd)
        shutil.rmtree(tmp)


def export_cases(L):
    """export_field of seeded fields (not a solve): the device table must give the
    same text byte for byte; one field has a nonpositive density (partial file)."""
    L.mo_ref_export_field.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_char_p,
                                      C.POINTER(MoErr)]
    tmp = tempfile.mkdtemp()
    try:
        for tag, (M, nx, ny, preset, bad) in {"m4": (4, 7, 5, "bottom_heated", None),
                                              "m6_lid": (6, 6, 6, "single_lid", None),
                                              "m3_bad": (3, 5, 4, "four_lid", 13)}.items():
            rng = np.random.default_rng(2206 + M)
            g = Grid.uniform(nx, ny, 1.0, 0.8)
            c, p = uniform_field(g, M, 1.0, (0.0, 0.0, 0.0), 1.0)
            c = c + rng.uniform(-0.05, 0.05, c.shape)
            c[:, 0] = rng.uniform(0.5, 1.5, g.cells)
            p[:, :3] = rng.uniform(-0.3, 0.3, (g.cells, 3))
            p[:, 3] = rng.uniform(0.7, 1.4, g.cells)
            if bad is not None:
                c[bad, 0] = -0.25
            doc = json.dumps({"scenario": preset})
            path = os.path.join(tmp, "f.tsv")
            err = MoErr()
            gc = g.c()
            rc = L.mo_ref_export_field(doc.encode(), C.byref(gc), M, c.ctypes.data, p.ctypes.data,
                                       path.encode(), C.byref(err))
            np.savez_compressed(os.path.join(OUT, f"export_{tag}.npz"), M=M, nx=nx, ny=ny, Lx=1.0, Ly=0.8,
                                coeffs=c, params=p, config=doc, rc=rc, msg=err.msg.decode(errors="replace"),
                                text=open(path).read())
            print("export", tag, "rc", rc, err.msg.decode(errors="replace"))
    finally:
        shutil.rmtree(tmp)


def main():
    L = lib()
    os.makedirs(OUT, exist_ok=True)
    json.dump(parse_cases(L), open(os.path.join(OUT, "parse_cases.json"), "w"), indent=1)
    export_cases(L)
    run_cases(L)


if __name__ == "__main__":
    main()
