"""The front end's host logic (paper_2206_13164_b200/scenario.py, cli.py) on
CPU, against the reference's own behaviour:

* every document of tests/golden/scenario/parse_cases.json through
  parse_config + config_echo: the echo text byte for byte, or the same
  ConfigError message (the fixture is the reference's scenario.cpp compiled
  here, tools/make_scenario_golden.py);
* the assertions of the reference's test_scenario.cpp that need no solve
  (presets, overrides, rejections, conversions, unit scales, history export);
* the configuration echo of every golden run equals the header of the
  reference's report.txt;
* command-line handling that stops before the GPU (exit codes 1).
"""
import json
import math
import os
import subprocess
import sys

import pytest

from paper_2206_13164_b200 import scenario as sc
from paper_2206_13164_b200.momg import CollisionKind, ConfigError, SolveReport, SolverKind

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "scenario")
PARSE = json.load(open(os.path.join(GOLD, "parse_cases.json")))
RUNS = sorted(d for d in os.listdir(GOLD) if os.path.isdir(os.path.join(GOLD, d)))


@pytest.mark.parametrize("case", PARSE, ids=[f"doc{k}" for k in range(len(PARSE))])
def test_parse_cases_match_reference(case):
    if case["rc"] == 0:
        assert sc.config_echo(sc.parse_config(case["doc"])) == case["echo"]
        return
    assert case["rc"] == 5  # ConfigError
    with pytest.raises(ConfigError) as e:
        sc.parse_config(case["doc"])
    if "parse error" in case["msg"]:  # the JSON parser's own position text differs
        assert str(e.value).startswith("config: [json.exception.parse_error.101] parse error")
    else:
        assert str(e.value) == case["msg"]


@pytest.mark.parametrize("name", RUNS)
def test_golden_run_echo(name):
    """config_echo of each golden run's document = the reference report.txt header."""
    d = os.path.join(GOLD, name)
    cfg = sc.parse_config(open(os.path.join(d, "config.json")).read())
    rep = os.path.join(d, "report.txt")
    if os.path.exists(rep):
        head = "".join(line for line in open(rep).read().splitlines(True) if line.startswith("# "))
        assert sc.config_echo(cfg) == head


def test_presets():
    """test_scenario.cpp:43-91"""
    s = sc.scenario_preset("single_lid")
    assert s.Lx == 9.63e-7 and s.Ly == 9.63e-7
    assert s.wall_top.speed == 50.0 and s.wall_bottom.speed == 0.0
    assert all(w.temperature == 273.0 for w in (s.wall_left, s.wall_right, s.wall_bottom, s.wall_top))
    assert s.init.density == 0.891 and s.init.temperature == 273.0
    assert s.gas.knudsen == 0.1
    assert s.collision.kind == CollisionKind.shakhov and s.collision.prandtl == 2.0 / 3.0
    assert s.cfl == 0.9 and s.tol == 1e-8
    assert (s.cycle.s1, s.cycle.s2, s.cycle.s3, s.cycle.gamma) == (2, 2, 4, 1)
    assert s.gas.viscosity_index == 0.81 and s.gas.molecule_mass == 6.63e-26
    f = sc.scenario_preset("four_lid")
    assert (f.Lx, f.wall_top.speed, f.wall_bottom.speed, f.wall_right.speed, f.wall_left.speed) == \
        (1.0, 50.0, -50.0, 50.0, -50.0)
    assert f.init.density == 1.1044e-7 and f.gas.knudsen == 0.777
    b = sc.scenario_preset("bottom_heated")
    assert (b.Lx, b.wall_bottom.temperature, b.wall_top.temperature, b.wall_left.temperature) == \
        (1e-6, 600.0, 300.0, 300.0)
    assert b.wall_bottom.speed == 0.0 and b.init.density == 0.2733 and b.init.temperature == 300.0
    assert b.gas.knudsen == 0.3
    with pytest.raises(ConfigError):
        sc.scenario_preset("三lid")
    # presets are independent objects
    sc.scenario_preset("single_lid").wall_top.speed = 1.0
    assert sc.scenario_preset("single_lid").wall_top.speed == 50.0


def test_overrides():
    """test_scenario.cpp:93-137"""
    c = sc.parse_config(PARSE[0]["doc"])
    assert c.collision.kind == CollisionKind.bgk and c.moment_order == 5
    assert (c.nx, c.ny, c.space_order, c.solver, c.levels, c.threads) == (32, 24, 2, SolverKind.fs, 3, 4)
    assert c.gas.knudsen == 1.0 and c.init.density == 0.0891
    assert c.init.velocity == [1.0, -2.0, 0.0] and c.init.temperature == 273.0
    assert c.wall_top.speed == 25.0 and c.wall_top.temperature == 273.0
    assert c.Lx == 9.63e-7 and c.Ly == 4.815e-7
    assert c.cycle.s3 == 6 and c.cycle.s1 == 2 and c.output_dir == "elsewhere"
    assert sc.parse_config('{"levels": "auto"}').levels == 0
    assert sc.parse_config("{}").scenario == "custom"


def test_rejections():
    """test_scenario.cpp:139-167"""
    for doc, msg in [('{"knudsen_number": 0.1}', "config: unknown key 'knudsen_number'"),
                     ('{"walls": {"front": {}}}', "config: unknown key 'walls.front'"),
                     ('{"init": {"pressure": 1.0}}', "config: unknown key 'init.pressure'"),
                     ('{"walls": {"top": {"velocity": 3.0}}}', "config: unknown key 'walls.top.velocity'")]:
        with pytest.raises(ConfigError, match=msg.replace(".", r"\.")):
            sc.parse_config(doc)
    for doc in ('{"nx": "sixteen"}', '{"levels": 0}', '{"cfl": 1.5}', '{"moment_order": 2}',
                '{"init": {"temperature": -1.0}}', '{"solver": "rk4"}', '{"collision": "boltzmann"}'):
        with pytest.raises(ConfigError):
            sc.parse_config(doc)
    with pytest.raises(ConfigError, match="parse error"):
        sc.parse_config('{ "nx": }')


def test_conversions_and_scales():
    """test_scenario.cpp:169-189"""
    mass = 6.63e-26
    for kelvin in (1e-3, 1.0, 273.0, 300.0, 600.0, 1e4):
        assert sc.theta_to_kelvin(sc.kelvin_to_theta(kelvin, mass), mass) == pytest.approx(kelvin, rel=1e-14)
    assert sc.kelvin_to_theta(273.0, mass) == 1.380649e-23 * 273.0 / 6.63e-26
    s = sc.unit_scales(sc.scenario_preset("single_lid"))
    assert s.length == 9.63e-7 and s.density == 0.891
    assert s.theta == 1.380649e-23 * 273.0 / 6.63e-26 and s.speed == math.sqrt(s.theta)


def test_export_history_format(tmp_path):
    """test_scenario.cpp:191-209"""
    p = tmp_path / "empty.tsv"
    sc.export_history(SolveReport(), str(p))
    assert p.read_text() == "iter\trel_residual\tseconds\n"
    r = SolveReport(history=[0.5, 0.25, 0.125], history_seconds=[0.01, 0.02, 0.03])
    sc.export_history(r, str(tmp_path / "three.tsv"))
    rows = (tmp_path / "three.tsv").read_text().splitlines()
    assert len(rows) == 4 and rows[1] == "1\t0.5\t0.01"
    assert all(rows[n].startswith(f"{n}\t") for n in (1, 2, 3))
    with pytest.raises(sc.Error, match="export_history: cannot open"):
        sc.export_history(r, str(tmp_path / "missing" / "h.tsv"))


def test_golden_history_format_roundtrip():
    """The reference's history.tsv rows re-formatted by export_history give the
    same bytes (%.17g of the parsed values)."""
    for name in RUNS:
        path = os.path.join(GOLD, name, "history.tsv")
        if not os.path.exists(path):
            continue
        rows = open(path).read().splitlines()[1:]
        vals = [tuple(float(x) for x in r.split("\t")[1:]) for r in rows]
        out = ["iter\trel_residual\tseconds"] + [f"{n + 1}\t{sc.fmt(a)}\t{sc.fmt(b)}" for n, (a, b) in enumerate(vals)]
        assert "\n".join(out) + "\n" == open(path).read()


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2206_13164_b200", *args], capture_output=True,
                          text=True, cwd=cwd or ROOT, timeout=120)


def test_cli_errors_before_the_solve(tmp_path):
    """tools/main.cpp:27-64: command-line and configuration errors exit 1."""
    assert _cli().returncode == 1
    assert _cli("solve").returncode == 1                       # --config is required
    assert _cli("solve", "--config", "x.json", "--order", "3").returncode == 1
    assert _cli("solve", "--config", "x.json", "--threads", "0").returncode == 1
    assert _cli("solve", "--config", "x.json", "--solver", "rk4").returncode == 1
    r = _cli("solve", "--config", str(tmp_path / "absent.json"))
    assert r.returncode == 1 and r.stderr.startswith("configuration error: config: cannot open")
    bad = tmp_path / "bad.json"
    bad.write_text('{"knudsen_number": 0.1}')
    r = _cli("solve", "--config", str(bad))
    assert r.returncode == 1 and "config: unknown key 'knudsen_number'" in r.stderr
    ok = tmp_path / "ok.json"
    ok.write_text('{"scenario": "single_lid"}')
    r = _cli("solve", "--config", str(ok), "--levels", "zero")
    assert r.returncode == 1 and "levels must be" in r.stderr
    assert _cli("--help").returncode == 0
