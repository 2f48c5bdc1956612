"""The front end on the GPU against the reference's
own outputs (tests/golden/scenario, made by the reference's scenario.cpp
compiled here: tools/make_scenario_golden.py):

* run_scenario of each golden document: same outcome (converged / the same
  NonConvergence / the same ConfigError), report.txt's configuration echo and
  status lines byte for byte, iterations +-1 (equal on these cases), the
  residual history at 1e-7 per iteration, field.tsv's coordinates bitwise and
  its macroscopic columns at 1e-8 of each column's scale (the converged-field
  bar), and no field.tsv after a failed run;
* export_field of seeded (unsolved) fields: the text byte for byte, including
  the partial file a nonpositive density leaves behind (NonphysicalState);
* the command line end to end (exit codes 0 / 2, echo, summary line, the
  output files) and a repeated run reproducing field.tsv byte for byte
  (test_scenario.cpp:225-243).
"""
import gzip
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
from paper_2206_13164_b200 import scenario as sc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "scenario")
RUNS = sorted(d for d in os.listdir(GOLD) if os.path.isdir(os.path.join(GOLD, d)))


def _table(text):
    rows = text.splitlines()
    assert rows[0] == "x\ty\trho\tu1\tu2\tT\tsigma11\tsigma12\tsigma22\tq1\tq2"
    return np.array([[float(v) for v in r.split("\t")] for r in rows[1:]]).reshape(-1, 11)


def _report(path):
    out = {}
    for line in open(path).read().splitlines():
        if not line.startswith("# "):
            k, v = line.split(" ", 1)
            out[k] = v
    return out


@pytest.mark.parametrize("name", RUNS)
def test_run_scenario_matches_reference(name, tmp_path, monkeypatch):
    d = os.path.join(GOLD, name)
    status = json.load(open(os.path.join(d, "status.json")))
    cfg = sc.parse_config(open(os.path.join(d, "config.json")).read())
    monkeypatch.chdir(tmp_path)
    out = os.path.join(tmp_path, cfg.output_dir)
    if status["rc"] == 5:  # ConfigError before anything is written
        with pytest.raises(momg.ConfigError) as e:
            sc.run_scenario(cfg)
        assert str(e.value) == status["msg"]
        assert not os.path.exists(os.path.join(out, "report.txt"))
        return
    if status["rc"] == 6:
        with pytest.raises(momg.NonConvergence) as e:
            sc.run_scenario(cfg)
        want = status["msg"]
        assert str(e.value).split(" at ratio ")[0] == want.split(" at ratio ")[0]
        assert float(str(e.value).split(" at ratio ")[1]) == pytest.approx(float(want.split(" at ratio ")[1]),
                                                                              rel=1e-5)
        assert not os.path.exists(os.path.join(out, "field.tsv"))
    else:
        assert status["rc"] == 0
        res = sc.run_scenario(cfg)
        assert res.report.converged
    # report.txt: echo byte for byte, status lines
    got_txt, want_txt = open(os.path.join(out, "report.txt")).read(), open(os.path.join(d, "report.txt")).read()
    head = lambda t: [ln for ln in t.splitlines() if ln.startswith("# ")]  # noqa: E731
    assert head(got_txt) == head(want_txt)
    g, w = _report(os.path.join(out, "report.txt")), _report(os.path.join(d, "report.txt"))
    assert g["converged"] == w["converged"]
    assert abs(int(g["iterations"]) - int(w["iterations"])) <= 1
    assert float(g["initial_residual"]) == pytest.approx(float(w["initial_residual"]), rel=1e-12)
    if g["iterations"] == w["iterations"]:
        assert g["cell_evaluations"] == w["cell_evaluations"]
        assert float(g["final_ratio"]) == pytest.approx(float(w["final_ratio"]), rel=1e-7)
    assert float(g["seconds"]) > 0.0
    # history.tsv: one row per iteration, ratios at 1e-7, seconds increasing
    gh = np.loadtxt(os.path.join(out, "history.tsv"), skiprows=1, ndmin=2)
    wh = np.loadtxt(os.path.join(d, "history.tsv"), skiprows=1, ndmin=2)
    assert len(gh) == int(g["iterations"])
    n = min(len(gh), len(wh))
    assert np.array_equal(gh[:, 0], np.arange(1, len(gh) + 1))
    np.testing.assert_allclose(gh[:n, 1], wh[:n, 1], rtol=1e-7, atol=0)
    assert np.all(np.diff(gh[:, 2]) >= 0) and gh[0, 2] > 0
    if status["rc"] != 0:
        return
    # field.tsv: coordinates bitwise, macroscopic columns at 1e-8 of their scale
    gt = _table(open(os.path.join(out, "field.tsv")).read())
    wt = _table(gzip.open(os.path.join(d, "field.tsv.gz"), "rt").read())
    assert gt.shape == wt.shape == (cfg.nx * cfg.ny, 11)
    assert np.array_equal(gt[:, :2], wt[:, :2])
    for k in range(2, 11):
        scale = max(np.max(np.abs(wt[:, k])), 1e-300)
        assert np.max(np.abs(gt[:, k] - wt[:, k])) <= 1e-8 * scale, f"column {k}"


@pytest.mark.parametrize("tag", ["m4", "m6_lid", "m3_bad"])
def test_export_field_bytes(tag, tmp_path):
    z = np.load(os.path.join(GOLD, f"export_{tag}.npz"))
    M, nx, ny = int(z["M"]), int(z["nx"]), int(z["ny"])
    cfg = sc.parse_config(str(z["config"]))
    g = momg.Grid2D.uniform(nx, ny, float(z["Lx"]), float(z["Ly"]))
    f = momg.CellField.from_host(g, M, z["coeffs"], z["params"])
    path = str(tmp_path / "field.tsv")
    if int(z["rc"]) == 0:
        sc.export_field(f, cfg, sc.unit_scales(cfg), path)
        tab = sc.field_table(f, cfg, sc.unit_scales(cfg))
        assert tab.shape == (nx * ny, 11)
    else:
        with pytest.raises(momg.NonphysicalState, match=str(z["msg"])):
            sc.export_field(f, cfg, sc.unit_scales(cfg), path)
    assert open(path).read() == str(z["text"])


def test_export_field_cannot_open(tmp_path):
    cfg = sc.scenario_preset("single_lid")
    f = momg.uniform_field(momg.Grid2D.uniform(4, 3), 3, 1.0, (0.0, 0.0, 0.0), 1.0)
    with pytest.raises(momg.Error, match="export_field: cannot open"):
        sc.export_field(f, cfg, sc.unit_scales(cfg), str(tmp_path / "no" / "field.tsv"))


def test_uniform_field_export_known_answer(tmp_path):
    """test_scenario.cpp:211-232: a uniform start exports its own lab state."""
    cfg = sc.scenario_preset("single_lid")
    s = sc.unit_scales(cfg)
    g = momg.Grid2D.uniform(4, 3, 1.0, 1.0)
    f = momg.uniform_field(g, 3, 1.0, (0.0, 0.0, 0.0), 1.0)
    sc.export_field(f, cfg, s, str(tmp_path / "field.tsv"))
    t = _table((tmp_path / "field.tsv").read_text())
    assert t.shape == (12, 11)
    for j in range(3):
        for i in range(4):
            row = t[j * 4 + i]
            assert row[0] == pytest.approx(g.xc[i] * 9.63e-7, rel=1e-15)
            assert row[1] == pytest.approx(g.yc[j] * 9.63e-7, rel=1e-15)
            assert row[2] == pytest.approx(0.891, rel=1e-15)
            assert row[3] == 0.0 and row[5] == pytest.approx(273.0, rel=1e-13)


def _cli(*args, cwd):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    return subprocess.run([sys.executable, "-m", "paper_2206_13164_b200", *args], capture_output=True,
                          text=True, cwd=cwd, timeout=600, env=env)


def test_cli_end_to_end(tmp_path):
    d = os.path.join(GOLD, "single_lid_m3")
    r = _cli("solve", "--config", os.path.join(d, "config.json"), "--output", "cli_a", cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    cfg = sc.load_config(os.path.join(d, "config.json"))
    cfg.output_dir = "cli_a"
    assert r.stdout.startswith(sc.config_echo(cfg))
    tail = r.stdout[len(sc.config_echo(cfg)):].splitlines()
    w = _report(os.path.join(d, "report.txt"))
    assert tail[0].startswith(f"converged in {w['iterations']} iterations, final ratio ")
    assert tail[0].endswith(f" {w['cell_evaluations']} cell evaluations")
    assert tail[1] == "wrote history.tsv, field.tsv, report.txt under cli_a"
    first = (tmp_path / "cli_a" / "field.tsv").read_text()
    # a repeated run reproduces field.tsv byte for byte (test_scenario.cpp:239-243)
    r2 = _cli("solve", "--config", os.path.join(d, "config.json"), "--output", "cli_b", cwd=tmp_path)
    assert r2.returncode == 0
    assert (tmp_path / "cli_b" / "field.tsv").read_text() == first
    # NonConvergence: exit 2, partial history left behind (test_scenario.cpp:246-262)
    r3 = _cli("solve", "--config", os.path.join(GOLD, "fail_cap", "config.json"), "--output", "cli_f",
              cwd=tmp_path)
    assert r3.returncode == 2 and r3.stderr.startswith("solver did not converge: iteration cap 2 reached")
    assert len((tmp_path / "cli_f" / "history.tsv").read_text().splitlines()) == 3
    assert "converged no" in (tmp_path / "cli_f" / "report.txt").read_text()
    # overrides: --solver fs --order 2 --levels 3 land in the echo
    r4 = _cli("solve", "--config", os.path.join(d, "config.json"), "--solver", "fs", "--order", "2",
              "--levels", "3", "--output", "cli_o", cwd=tmp_path)
    assert "# solver fs\n" in r4.stdout and "# order 2\n" in r4.stdout and "# levels 3\n" in r4.stdout
