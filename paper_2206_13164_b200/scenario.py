"""Front end of the solver: scenario configurations in, wire formats out
(SURVEY.md §8(f) row 4).  Mirror of the reference's momg/scenario.hpp
(/root/reference/proj/include/momg/scenario.hpp, src/scenario.cpp) over the
device path:

    kelvin_to_theta / theta_to_kelvin   scenario.cpp:144-150
    ScenarioConfig, WallSetting,
    InitialState                        scenario.hpp:17-55
    scenario_preset                     scenario.cpp:152-184
    parse_config / load_config          scenario.cpp:217-307
    solver_kind_from_string, to_string,
    levels_from_string                  scenario.cpp:186-215
    unit_scales                         scenario.cpp:309-316
    config_echo                         scenario.cpp:318-354
    export_history                      scenario.cpp:356-365
    export_field                        scenario.cpp:367-399 (device table +
                                        the library's TSV writer, momg_export_field)
    run_scenario                        scenario.cpp:401-459 (solve_steady on the GPU)

Names, argument meaning, defaults, error types and messages follow the
reference (ConfigError "config: ..." texts verbatim).  JSON documents are
parsed with the standard library; the reference uses nlohmann::json, whose
behaviour the mirror keeps where it is observable: objects' unknown keys are
reported in sorted key order, integer keys accept only integer literals, a
number is any JSON number (not a boolean), NaN / Infinity are not JSON, and
malformed text raises ConfigError("config: [json.exception.parse_error.101]
parse error at line L, column C: ...").  Values are formatted with %.17g
(scenario.cpp:18-22).
"""
from __future__ import annotations

import json
import math
import os
import re
from dataclasses import dataclass, field

from . import momg
from .momg import (CollisionKind, CollisionModel, ConfigError, CyclePolicy, Error, GasParams,
                   NonConvergence, SolverKind)

K_BOLTZMANN = 1.380649e-23   # J/K (scenario.hpp:10)
MIN_COARSE_CELLS = 8         # multigrid.hpp:11 (echoed as coarsest_floor)


def fmt(v: float) -> str:
    """scenario.cpp:18-22: %.17g."""
    return "%.17g" % v


def kelvin_to_theta(kelvin: float, molecule_mass: float) -> float:
    return K_BOLTZMANN * kelvin / molecule_mass


def theta_to_kelvin(theta: float, molecule_mass: float) -> float:
    return theta * molecule_mass / K_BOLTZMANN


@dataclass
class WallSetting:
    """scenario.hpp:17-23: tangential speed (m/s) and temperature (K)."""
    speed: float = 0.0
    temperature: float = 273.0


@dataclass
class InitialState:
    """scenario.hpp:25-31: uniform Maxwellian start in laboratory units."""
    density: float = 1.0
    velocity: list = field(default_factory=lambda: [0.0, 0.0, 0.0])
    temperature: float = 273.0


@dataclass
class ScenarioConfig:
    """scenario.hpp:33-55 (defaults as there)."""
    scenario: str = "custom"
    collision: CollisionModel = field(default_factory=lambda: CollisionModel(CollisionKind.shakhov, 2.0 / 3.0))
    moment_order: int = 3
    nx: int = 16
    ny: int = 16
    space_order: int = 1
    solver: SolverKind = SolverKind.nmg
    levels: int = 0            # 0 = deepest hierarchy
    cfl: float = 0.9           # CflPolicy{}.cfl
    tol: float = 1e-8          # SolverOptions{}.tol
    max_iterations: int = 0    # 0 = solver default cap
    threads: int = 1
    gas: GasParams = field(default_factory=GasParams)
    Lx: float = 1.0            # metres
    Ly: float = 1.0
    wall_left: WallSetting = field(default_factory=WallSetting)
    wall_right: WallSetting = field(default_factory=WallSetting)
    wall_bottom: WallSetting = field(default_factory=WallSetting)
    wall_top: WallSetting = field(default_factory=WallSetting)
    init: InitialState = field(default_factory=InitialState)
    cycle: CyclePolicy = field(default_factory=CyclePolicy)
    output_dir: str = "out"


@dataclass
class UnitScales:
    """scenario.hpp:76-84"""
    length: float = 1.0
    density: float = 1.0
    theta: float = 1.0
    speed: float = 1.0


@dataclass
class ScenarioResult:
    """scenario.hpp:96-100: the report, the solved field (solver units, on the
    device) and the unit scales."""
    report: momg.SolveReport
    field: momg.CellField
    scales: UnitScales


# ------------------------------------------------------------ presets / names
def scenario_preset(name: str) -> ScenarioConfig:
    """scenario.cpp:148-184: single_lid, four_lid, bottom_heated, custom."""
    c = ScenarioConfig()
    c.scenario = name
    if name == "custom":
        return c
    if name == "single_lid":
        c.Lx = c.Ly = 9.63e-7
        c.wall_top.speed = 50.0
        c.init.density = 0.891
        c.gas.knudsen = 0.1
        return c
    if name == "four_lid":
        c.wall_top.speed = 50.0
        c.wall_bottom.speed = -50.0
        c.wall_right.speed = 50.0
        c.wall_left.speed = -50.0
        c.init.density = 1.1044e-7
        c.gas.knudsen = 0.777
        return c
    if name == "bottom_heated":
        c.Lx = c.Ly = 1e-6
        c.wall_bottom.temperature = 600.0
        c.wall_left.temperature = 300.0
        c.wall_right.temperature = 300.0
        c.wall_top.temperature = 300.0
        c.init.density = 0.2733
        c.init.temperature = 300.0
        c.gas.knudsen = 0.3
        return c
    raise ConfigError(f"config: unknown scenario '{name}'")


_SOLVERS = {"euler": SolverKind.euler, "fs": SolverKind.fs, "nmg": SolverKind.nmg}
_COLLISIONS = {"bgk": CollisionKind.bgk, "es_bgk": CollisionKind.es_bgk, "shakhov": CollisionKind.shakhov}


def solver_kind_from_string(name: str) -> SolverKind:
    if name in _SOLVERS:
        return _SOLVERS[name]
    raise ConfigError(f"config: unknown solver '{name}'")


def to_string(kind: SolverKind) -> str:
    return {SolverKind.euler: "euler", SolverKind.fs: "fs", SolverKind.nmg: "nmg"}.get(kind, "unknown")


def collision_from_string(name: str) -> CollisionKind:
    if name in _COLLISIONS:
        return _COLLISIONS[name]
    raise ConfigError(f"config: unknown collision model '{name}'")


def collision_name(kind: CollisionKind) -> str:
    return {CollisionKind.bgk: "bgk", CollisionKind.es_bgk: "es_bgk",
            CollisionKind.shakhov: "shakhov"}.get(kind, "unknown")


def _int32(v: int) -> int:
    """json get<int>: the integer narrowed to a C int."""
    return (v + 2 ** 31) % 2 ** 32 - 2 ** 31


_STOI = re.compile(r"[ \t\n\v\f\r]*[+-]?[0-9]+")


def levels_from_string(text: str) -> int:
    """scenario.cpp:205-215: "auto" -> 0, else a positive count (std::stoi
    with the whole text consumed)."""
    if text == "auto":
        return 0
    m = _STOI.match(text)
    if m and m.end() == len(text):
        k = int(text)
        if -2 ** 31 <= k < 2 ** 31 and k >= 1:
            return k
    raise ConfigError(f"config: levels must be \"auto\" or a positive count, got '{text}'")


# ------------------------------------------------------------------ parsing
def _is_number(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _is_integer(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _bad_key(key: str, what: str):
    raise ConfigError(f"config: key '{key}' {what}")


def _check_keys(j: dict, where: str, allowed) -> None:
    for k in sorted(j):  # nlohmann's object is a std::map: keys in byte order
        if k not in allowed:
            raise ConfigError(f"config: unknown key '{k if not where else where + '.' + k}'")


def _get_number(j: dict, key: str, fallback: float) -> float:
    if key not in j:
        return fallback
    v = j[key]
    if not _is_number(v):
        _bad_key(key, "must be a number")
    return float(v)


def _get_int(j: dict, key: str, fallback: int) -> int:
    if key not in j:
        return fallback
    v = j[key]
    if not _is_integer(v):
        _bad_key(key, "must be an integer")
    return _int32(v)


def _get_string(j: dict, key: str, fallback: str) -> str:
    if key not in j:
        return fallback
    v = j[key]
    if not isinstance(v, str):
        _bad_key(key, "must be a string")
    return v


def _apply_wall(j, where: str, wall: WallSetting) -> None:
    if not isinstance(j, dict):
        _bad_key(where, "must be an object")
    _check_keys(j, where, ("speed", "temperature"))
    wall.speed = _get_number(j, "speed", wall.speed)
    wall.temperature = _get_number(j, "temperature", wall.temperature)


def validate_config(c: ScenarioConfig) -> None:
    """scenario.cpp:92-124 (same checks, same order, same messages)."""
    if c.moment_order < 3:
        raise ConfigError("config: moment_order must be at least 3")
    if c.nx < 1 or c.ny < 1:
        raise ConfigError("config: nx and ny must be positive")
    if c.space_order not in (1, 2):
        raise ConfigError("config: order must be 1 or 2")
    if not c.cfl > 0.0 or c.cfl > 1.0:
        raise ConfigError("config: cfl must lie in (0, 1]")
    if not c.tol > 0.0:
        raise ConfigError("config: tol must be positive")
    if c.max_iterations < 0:
        raise ConfigError("config: max_iterations must be nonnegative")
    if c.levels < 0:
        raise ConfigError("config: levels must be nonnegative")
    if c.threads < 1:
        raise ConfigError("config: threads must be positive")
    if not c.collision.prandtl > 0.0:
        raise ConfigError("config: prandtl must be positive")
    if not c.gas.knudsen > 0.0:
        raise ConfigError("config: knudsen must be positive")
    if not c.gas.viscosity_index > 0.0:
        raise ConfigError("config: viscosity_index must be positive")
    if not c.gas.molecule_mass > 0.0:
        raise ConfigError("config: molecule_mass must be positive")
    if not c.Lx > 0.0 or not c.Ly > 0.0:
        raise ConfigError("config: domain lengths must be positive")
    if not c.init.density > 0.0 or not c.init.temperature > 0.0:
        raise ConfigError("config: initial density and temperature must be positive")
    for w in (c.wall_left, c.wall_right, c.wall_bottom, c.wall_top):
        if not w.temperature > 0.0:
            raise ConfigError("config: wall temperatures must be positive")
    if c.cycle.s1 < 0 or c.cycle.s2 < 0:
        raise ConfigError("config: s1 and s2 must be nonnegative")
    if c.cycle.s3 < 1:
        raise ConfigError("config: s3 must be positive")
    if c.cycle.gamma < 1:
        raise ConfigError("config: gamma must be positive")


def _reject_constant(name):
    raise ValueError(f"invalid literal '{name}'")


_TOP_KEYS = ("scenario", "collision", "prandtl", "moment_order", "nx", "ny", "order", "solver", "levels",
             "cfl", "tol", "max_iterations", "threads", "knudsen", "viscosity_index", "molecule_mass",
             "domain", "walls", "init", "s1", "s2", "s3", "gamma", "output_dir")


def _loads(text: str):
    try:
        return json.loads(text, parse_constant=_reject_constant)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config: [json.exception.parse_error.101] parse error at line {e.lineno}, "
                          f"column {e.colno}: syntax error - {e.msg}") from None
    except ValueError as e:  # NaN / Infinity: not JSON
        raise ConfigError(f"config: [json.exception.parse_error.101] parse error: syntax error - {e}") from None


def parse_config(text: str) -> ScenarioConfig:
    """scenario.cpp:217-299: the `scenario` key selects the preset whose values
    the remaining keys override; unknown keys are rejected by name."""
    j = _loads(text)
    if not isinstance(j, dict):
        raise ConfigError("config: document must be a JSON object")
    _check_keys(j, "", _TOP_KEYS)
    c = scenario_preset(_get_string(j, "scenario", "custom"))
    if "collision" in j:
        c.collision.kind = collision_from_string(_get_string(j, "collision", ""))
    c.collision.prandtl = _get_number(j, "prandtl", c.collision.prandtl)
    c.moment_order = _get_int(j, "moment_order", c.moment_order)
    c.nx = _get_int(j, "nx", c.nx)
    c.ny = _get_int(j, "ny", c.ny)
    c.space_order = _get_int(j, "order", c.space_order)
    if "solver" in j:
        c.solver = solver_kind_from_string(_get_string(j, "solver", ""))
    if "levels" in j:
        v = j["levels"]
        if isinstance(v, str):
            c.levels = levels_from_string(v)
        elif _is_integer(v) and _int32(v) >= 1:
            c.levels = _int32(v)
        else:
            _bad_key("levels", "must be \"auto\" or a positive count")
    c.cfl = _get_number(j, "cfl", c.cfl)
    c.tol = _get_number(j, "tol", c.tol)
    c.max_iterations = _get_int(j, "max_iterations", c.max_iterations)
    c.threads = _get_int(j, "threads", c.threads)
    c.gas.knudsen = _get_number(j, "knudsen", c.gas.knudsen)
    c.gas.viscosity_index = _get_number(j, "viscosity_index", c.gas.viscosity_index)
    c.gas.molecule_mass = _get_number(j, "molecule_mass", c.gas.molecule_mass)
    if "domain" in j:
        d = j["domain"]
        if not isinstance(d, dict):
            _bad_key("domain", "must be an object")
        _check_keys(d, "domain", ("Lx", "Ly"))
        c.Lx = _get_number(d, "Lx", c.Lx)
        c.Ly = _get_number(d, "Ly", c.Ly)
    if "walls" in j:
        w = j["walls"]
        if not isinstance(w, dict):
            _bad_key("walls", "must be an object")
        _check_keys(w, "walls", ("left", "right", "bottom", "top"))
        for name in ("left", "right", "bottom", "top"):
            if name in w:
                _apply_wall(w[name], "walls." + name, getattr(c, "wall_" + name))
    if "init" in j:
        v = j["init"]
        if not isinstance(v, dict):
            _bad_key("init", "must be an object")
        _check_keys(v, "init", ("density", "velocity", "temperature"))
        c.init.density = _get_number(v, "density", c.init.density)
        c.init.temperature = _get_number(v, "temperature", c.init.temperature)
        if "velocity" in v:
            u = v["velocity"]
            if not isinstance(u, list) or len(u) not in (2, 3):
                _bad_key("init.velocity", "must be an array of 2 or 3 numbers")
            c.init.velocity = [0.0, 0.0, 0.0]
            for d, x in enumerate(u):
                if not _is_number(x):
                    _bad_key("init.velocity", "must be an array of 2 or 3 numbers")
                c.init.velocity[d] = float(x)
    c.cycle.s1 = _get_int(j, "s1", c.cycle.s1)
    c.cycle.s2 = _get_int(j, "s2", c.cycle.s2)
    c.cycle.s3 = _get_int(j, "s3", c.cycle.s3)
    c.cycle.gamma = _get_int(j, "gamma", c.cycle.gamma)
    c.output_dir = _get_string(j, "output_dir", c.output_dir)
    validate_config(c)
    return c


def load_config(path: str) -> ScenarioConfig:
    """scenario.cpp:301-307"""
    try:
        with open(path, "rb") as fh:
            raw = fh.read()
    except OSError:
        raise ConfigError(f"config: cannot open '{path}'") from None
    return parse_config(raw.decode("utf-8", errors="surrogateescape"))


def unit_scales(config: ScenarioConfig) -> UnitScales:
    """scenario.cpp:309-316"""
    theta = kelvin_to_theta(config.init.temperature, config.gas.molecule_mass)
    return UnitScales(config.Lx, config.init.density, theta, math.sqrt(theta))


# ---------------------------------------------------------------- formats
def config_echo(c: ScenarioConfig) -> str:
    """scenario.cpp:318-354: one "# key value" line per setting."""
    lines = [
        f"# scenario {c.scenario}",
        f"# collision {collision_name(c.collision.kind)}",
        f"# prandtl {fmt(c.collision.prandtl)}",
        f"# moment_order {c.moment_order}",
        f"# grid {c.nx} {c.ny}",
        f"# order {c.space_order}",
        f"# solver {to_string(c.solver)}",
        f"# levels {'auto' if c.levels == 0 else c.levels}",
        f"# cycle_s1 {c.cycle.s1}",
        f"# cycle_s2 {c.cycle.s2}",
        f"# cycle_s3 {c.cycle.s3}",
        f"# cycle_gamma {c.cycle.gamma}",
        f"# coarsest_floor {MIN_COARSE_CELLS}",
        f"# cfl {fmt(c.cfl)}",
        f"# tol {fmt(c.tol)}",
        f"# max_iterations {c.max_iterations}",
        f"# threads {c.threads}",
        f"# knudsen {fmt(c.gas.knudsen)}",
        f"# viscosity_index {fmt(c.gas.viscosity_index)}",
        f"# molecule_mass {fmt(c.gas.molecule_mass)}",
        f"# domain {fmt(c.Lx)} {fmt(c.Ly)}",
    ]
    for name in ("left", "right", "bottom", "top"):
        w = getattr(c, "wall_" + name)
        lines.append(f"# wall_{name} {fmt(w.speed)} {fmt(w.temperature)}")
    lines += [
        f"# init_density {fmt(c.init.density)}",
        f"# init_velocity {fmt(c.init.velocity[0])} {fmt(c.init.velocity[1])}",
        f"# init_temperature {fmt(c.init.temperature)}",
        f"# output_dir {c.output_dir}",
    ]
    return "\n".join(lines) + "\n"


def _write(path: str, text: str, who: str) -> None:
    try:
        fh = open(path, "w", newline="\n")
    except OSError:
        raise Error(f"{who}: cannot open '{path}'") from None
    try:
        with fh:
            fh.write(text)
    except OSError:
        raise Error(f"{who}: write failed for '{path}'") from None


def export_history(report: momg.SolveReport, path: str) -> None:
    """scenario.cpp:356-365: header, then (iter, rel_residual, seconds) rows."""
    secs = list(report.history_seconds) + [0.0] * (len(report.history) - len(report.history_seconds))
    rows = ["iter\trel_residual\tseconds"]
    rows += [f"{n + 1}\t{fmt(r)}\t{fmt(s)}" for n, (r, s) in enumerate(zip(report.history, secs))]
    _write(path, "\n".join(rows) + "\n", "export_history")


def export_field(fld: momg.CellField, config: ScenarioConfig, scales: UnitScales, path: str) -> None:
    """scenario.cpp:367-399: the field in laboratory units, one row per cell
    (x, y, rho, u1, u2, T, sigma11, sigma12, sigma22, q1, q2), row-major with j
    outermost.  The per-cell values are computed on the device and the text is
    written by the library (momg_export_field)."""
    momg.export_field_tsv(fld, path, scales.length, scales.density, scales.theta, scales.speed,
                          config.gas.molecule_mass)


def field_table(fld: momg.CellField, config: ScenarioConfig, scales: UnitScales):
    """export_field's values as an array (nx*ny, 11), without the text."""
    return momg.field_table(fld, scales.length, scales.density, scales.theta, scales.speed,
                            config.gas.molecule_mass)


def write_report(c: ScenarioConfig, r: momg.SolveReport, path: str) -> None:
    """scenario.cpp:126-142"""
    text = config_echo(c) + "".join([
        f"converged {'yes' if r.converged else 'no'}\n",
        f"iterations {r.iterations}\n",
        f"initial_residual {fmt(r.r0_norm)}\n",
        f"final_residual {fmt(r.final_norm)}\n",
        f"final_ratio {fmt(r.final_ratio)}\n",
        f"cell_evaluations {r.work}\n",
        f"seconds {fmt(r.seconds)}\n",
    ])
    _write(path, text, "write_report")


# ------------------------------------------------------------------- driver
def solve_context(config: ScenarioConfig, scales: UnitScales) -> momg.SolveContext:
    """The solver-unit SolveContext of a scenario (scenario.cpp:406-424)."""
    def wall(w: WallSetting) -> momg.WallSpec:
        return momg.WallSpec(w.speed / scales.speed,
                             kelvin_to_theta(w.temperature, config.gas.molecule_mass) / scales.theta)

    scheme = momg.SpatialScheme.for_moment_order(config.moment_order, config.space_order)
    return momg.SolveContext(
        walls=momg.Walls(wall(config.wall_left), wall(config.wall_right), wall(config.wall_bottom),
                         wall(config.wall_top)),
        model=CollisionModel(config.collision.kind, config.collision.prandtl),
        gas=GasParams(config.gas.knudsen, config.gas.viscosity_index, config.gas.molecule_mass),
        scheme=scheme,
        cfl=momg.CflPolicy(config.cfl, scheme.c_bound),
        threads=config.threads)


def run_scenario(config: ScenarioConfig) -> ScenarioResult:
    """scenario.cpp:401-459: uniform Maxwellian start, solve_steady on the GPU,
    then history.tsv, field.tsv and report.txt under output_dir; on
    NonConvergence the partial history and the report are written before the
    exception propagates."""
    validate_config(config)
    scales = unit_scales(config)
    grid = momg.Grid2D.uniform(config.nx, config.ny, 1.0, config.Ly / config.Lx)
    ctx = solve_context(config, scales)
    u0 = [u / scales.speed for u in config.init.velocity]
    theta0 = kelvin_to_theta(config.init.temperature, config.gas.molecule_mass) / scales.theta
    fld = momg.uniform_field(grid, config.moment_order, config.init.density / scales.density, u0, theta0)

    os.makedirs(config.output_dir, exist_ok=True)
    history_path = os.path.join(config.output_dir, "history.tsv")
    field_path = os.path.join(config.output_dir, "field.tsv")
    report_path = os.path.join(config.output_dir, "report.txt")
    options = momg.SolverOptions(config.solver, config.tol, config.max_iterations, config.levels,
                                 CyclePolicy(config.cycle.s1, config.cycle.s2, config.cycle.s3,
                                             config.cycle.gamma))
    try:
        report = momg.solve_steady(fld, ctx, options)
    except NonConvergence as e:
        export_history(e.report, history_path)
        write_report(config, e.report, report_path)
        raise
    export_history(report, history_path)
    export_field(fld, config, scales, field_path)
    write_report(config, report, report_path)
    return ScenarioResult(report, fld, scales)
