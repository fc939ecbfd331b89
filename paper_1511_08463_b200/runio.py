"""INI-configured runs and parameter sweeps on the B200 path (reference runio.py, cli.py).

The reference's `phasefrac run|sweep|validate cfg.ini` front end (runio.py:1-60 documents the
grammar) driving the device solvers: the same sections and keys, the same defaults and
validation, the same artifacts (energies.csv, iterations.csv, step_NNNN.vtk, provenance.txt,
summary.csv) and exit codes (0 ok, 2 configuration, 3 non-convergence, 4 I/O).  Differences,
all loud:

* ``[case] name = thermal_shock`` runs on the element-list path (the reference's jittered
  rect_mesh, mesh.py:112-142; cases.setup_thermal_shock): alternate minimisation only (methods am
  and oram); oram_n / newton_only need the coupled Newton step, which that path does not have:
  ConfigError.
* ``[linear] elastic = cg`` with ``elastic_precond = ssor | chebyshev`` has no device form
  (two sparse triangular solves / a stand-alone polynomial): ConfigError.  ``elastic = direct``
  is device PCG at the parity tolerance with the multigrid preconditioner whatever the
  ``elastic_precond`` (SolverConfig docs).
* ``sweep --threads N`` runs the rows in N spawned worker processes, worker w on CUDA device
  w mod (device count): the reference's process-pool sweep (runio.py:550-590) as replicas across
  GPUs.

Reductions on the device are fixed-order, so reruns of one config write bitwise identical
files, as the reference promises (runio.py:478-488).
"""

from __future__ import annotations

import configparser
import dataclasses
import io
import multiprocessing as mp
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass, fields
from pathlib import Path
from typing import Optional

import numpy as np


class ConfigError(ValueError):
    """Invalid or unparsable configuration (exit code 2)."""


CASES = ("traction", "surfing", "thermal_shock")
METHODS = ("am", "oram", "oram_n", "newton_only")
SWEEPABLE = ("omega", "ell", "h", "dT_factor")
# case -> defaults that depend on the case (runio.py:87-91); thermal_shock also defaults ell = 1
CASE_DEFAULTS = {"traction": dict(L=1.0, H=0.3, n_steps=30),
                 "surfing": dict(L=2.0, H=1.0, n_steps=25),
                 "thermal_shock": dict(L=20.0, H=10.0, n_steps=40)}


@dataclass
class RunConfig:
    """A fully resolved run configuration (runio.py:95-137)."""

    case: str = "traction"
    ell: float = 0.1
    h: float = 0.02
    L: float = 1.0
    H: float = 0.3
    n_steps: int = 30
    E: float = 1.0
    nu: float = 0.3
    Gc: float = 1.0
    k_ell: float = 1e-6
    beta: float = 1.0
    load_max_factor: float = 1.5
    t_end: float = 1.0
    dT_factor: float = 1.0
    tau_min: float = 0.05
    tau_max: float = 3.0
    method: str = "am"
    omega: float = 1.0
    outer_atol: float = 1e-7
    am_rtol: float = 0.1
    max_am_iterations: int = 1000
    max_newton_iterations: int = 30
    max_outer_cycles: int = 20
    elastic: str = "direct"
    elastic_precond: str = "ssor"
    elastic_rtol: float = 1e-10
    coupled: str = "fieldsplit"
    fieldsplit_inner: str = "direct"
    fieldsplit_cg_budget: int = 5
    fieldsplit_rtol: float = 1e-6
    directory: str = "out"
    snapshot_stride: int = 1
    seed: int = 0


# INI layout: section -> [(key, attribute)]; the attribute's dataclass type gives the parser
LAYOUT = {
    "case": [("name", "case")] + [(k, k) for k in (
        "ell", "h", "L", "H", "n_steps", "E", "nu", "Gc", "k_ell", "beta", "load_max_factor",
        "t_end", "dT_factor", "tau_min", "tau_max")],
    "solver": [(k, k) for k in ("method", "omega", "outer_atol", "am_rtol", "max_am_iterations",
                                "max_newton_iterations", "max_outer_cycles")],
    "linear": [(k, k) for k in ("elastic", "elastic_precond", "elastic_rtol", "coupled",
                                "fieldsplit_inner", "fieldsplit_cg_budget", "fieldsplit_rtol")],
    "output": [(k, k) for k in ("directory", "snapshot_stride", "seed")],
}
_TYPES = {f.name: f.type for f in fields(RunConfig)}


@dataclass
class SweepSpec:
    """[sweep] parameter and values over a base configuration (runio.py:139-152)."""

    parameter: str
    values: list
    base: RunConfig

    def __post_init__(self):
        if self.parameter not in SWEEPABLE:
            raise ConfigError(f"sweep parameter must be one of {SWEEPABLE}, got {self.parameter!r}")
        if not self.values:
            raise ConfigError("sweep values list must not be empty")


def _ini(text: str) -> configparser.ConfigParser:
    p = configparser.ConfigParser(interpolation=None)
    p.optionxform = str  # keys are case-sensitive (L, H, E, Gc)
    try:
        p.read_string(text)
    except configparser.Error as exc:
        raise ConfigError(f"malformed config: {exc}") from exc
    return p


def _value(section: str, key: str, attr: str, raw: str):
    kind = _TYPES[attr]
    try:
        if kind in (float, "float"):
            return float(raw)
        if kind in (int, "int"):
            return int(raw)
    except ValueError as exc:
        raise ConfigError(f"[{section}] {key}: cannot parse {raw!r}") from exc
    return raw.strip()


def validate_config(cfg: RunConfig) -> None:
    """Choice and range checks (runio.py:204-244)."""
    def need(ok, msg):
        if not ok:
            raise ConfigError(msg)

    need(cfg.case in CASES, f"[case] name must be one of {CASES}, got {cfg.case!r}")
    need(cfg.method in METHODS, f"[solver] method must be one of {METHODS}, got {cfg.method!r}")
    need(0.0 < cfg.omega < 2.0, f"[solver] omega must lie strictly inside (0, 2), got {cfg.omega!r}")
    need(not (cfg.method == "am" and cfg.omega != 1.0),
         "[solver] method 'am' is the unrelaxed scheme (omega = 1); use method 'oram' to set omega")
    for key in ("ell", "h", "L", "H", "E", "Gc", "beta", "outer_atol", "am_rtol", "elastic_rtol",
                "fieldsplit_rtol", "tau_min", "tau_max", "t_end", "load_max_factor", "dT_factor"):
        need(getattr(cfg, key) > 0.0, f"{key} must be positive, got {getattr(cfg, key)!r}")
    need(-1.0 < cfg.nu < 0.5, f"[case] nu must lie in (-1, 0.5), got {cfg.nu!r}")
    need(cfg.k_ell >= 0.0, f"[case] k_ell must be nonnegative, got {cfg.k_ell!r}")
    need(cfg.tau_min < cfg.tau_max, "[case] tau_min must be smaller than tau_max")
    for key in ("n_steps", "max_am_iterations", "max_newton_iterations", "max_outer_cycles",
                "fieldsplit_cg_budget"):
        need(getattr(cfg, key) >= 1, f"{key} must be at least 1, got {getattr(cfg, key)!r}")
    need(cfg.snapshot_stride >= 0, f"snapshot_stride must be nonnegative, got {cfg.snapshot_stride!r}")
    need(cfg.elastic in ("direct", "cg"), f"[linear] elastic must be direct or cg, got {cfg.elastic!r}")
    need(cfg.elastic_precond in ("jacobi", "ssor", "chebyshev"),
         f"[linear] elastic_precond must be jacobi, ssor or chebyshev, got {cfg.elastic_precond!r}")
    need(cfg.coupled in ("direct", "fieldsplit"),
         f"[linear] coupled must be direct or fieldsplit, got {cfg.coupled!r}")
    need(cfg.fieldsplit_inner in ("direct", "cg"),
         f"[linear] fieldsplit_inner must be direct or cg, got {cfg.fieldsplit_inner!r}")


def _resolve(p: configparser.ConfigParser, extra=()) -> RunConfig:
    bad = [s for s in p.sections() if s not in LAYOUT and s not in extra]
    if bad:
        raise ConfigError(f"unknown config sections: {', '.join(bad)}")
    vals = {}
    for section, entries in LAYOUT.items():
        if not p.has_section(section):
            continue
        names = dict(entries)
        unknown = sorted(k for k in p[section] if k not in names)
        if unknown:
            raise ConfigError(f"unknown keys in [{section}]: {', '.join(unknown)}")
        for key, raw in p[section].items():
            vals[names[key]] = _value(section, key, names[key], raw)
    case = vals.get("case", "traction")
    if case not in CASES:
        raise ConfigError(f"[case] name must be one of {CASES}, got {case!r}")
    for attr, dflt in CASE_DEFAULTS[case].items():
        vals.setdefault(attr, dflt)
    vals.setdefault("ell", 1.0 if case == "thermal_shock" else 0.1)
    vals.setdefault("h", vals["ell"] / 5.0)
    cfg = RunConfig(**vals)
    validate_config(cfg)
    return cfg


def parse_config(text: str) -> RunConfig:
    return _resolve(_ini(text))


def parse_sweep(text: str) -> SweepSpec:
    p = _ini(text)
    if not p.has_section("sweep"):
        raise ConfigError("sweep file requires a [sweep] section")
    extra = sorted(k for k in p["sweep"] if k not in ("parameter", "values"))
    if extra:
        raise ConfigError(f"unknown keys in [sweep]: {', '.join(extra)}")
    if not p.has_option("sweep", "parameter"):
        raise ConfigError("[sweep] parameter is required")
    raw = p.get("sweep", "values", fallback="")
    try:
        values = [float(t) for t in raw.replace(",", " ").split()]
    except ValueError as exc:
        raise ConfigError(f"[sweep] values: cannot parse {raw!r}") from exc
    return SweepSpec(p.get("sweep", "parameter").strip(), values, _resolve(p, extra=("sweep",)))


def _fmt(v) -> str:
    return repr(v) if isinstance(v, float) else str(v)


def echo_config(cfg: RunConfig) -> str:
    """Canonical INI text; parse_config(echo_config(c)) == c (runio.py:314-325)."""
    out = []
    for section, entries in LAYOUT.items():
        out.append(f"[{section}]")
        out += [f"{key} = {_fmt(getattr(cfg, attr))}" for key, attr in entries]
        out.append("")
    return "\n".join(out)


# ---- device problem from a config ------------------------------------------------------------

def build_material(cfg: RunConfig):
    from .model import Material
    return Material(E=cfg.E, nu=cfg.nu, Gc=cfg.Gc, ell=cfg.ell, k_ell=cfg.k_ell, beta=cfg.beta)


def build_solver_config(cfg: RunConfig):
    """SolverConfig of the device path; the reference method names map as runio.py:331-352."""
    from .solver import SolverConfig
    if cfg.elastic == "cg" and cfg.elastic_precond in ("ssor", "chebyshev"):
        raise ConfigError(f"[linear] elastic_precond = {cfg.elastic_precond} has no B200 device form "
                          "with elastic = cg; use jacobi (or elastic = direct: multigrid PCG)")
    method = {"am": "am", "oram": "am", "oram_n": "oram_newton", "newton_only": "newton_only"}[cfg.method]
    return SolverConfig(method=method, omega=cfg.omega, outer_atol=cfg.outer_atol, am_rtol=cfg.am_rtol,
                        max_am_iterations=cfg.max_am_iterations,
                        max_newton_iterations=cfg.max_newton_iterations,
                        max_outer_cycles=cfg.max_outer_cycles, elastic_solver=cfg.elastic,
                        elastic_rtol=cfg.elastic_rtol, elastic_precond=cfg.elastic_precond,
                        coupled_solver=cfg.coupled, fieldsplit_inner=cfg.fieldsplit_inner,
                        fieldsplit_cg_budget=cfg.fieldsplit_cg_budget,
                        fieldsplit_rtol=cfg.fieldsplit_rtol)


def build_setup(cfg: RunConfig):
    from .cases import setup_surfing, setup_traction
    mat = build_material(cfg)
    if cfg.case == "traction":
        return setup_traction(mat, L=cfg.L, H=cfg.H, h=cfg.h, n_steps=cfg.n_steps,
                              load_max_factor=cfg.load_max_factor)
    if cfg.case == "surfing":
        return setup_surfing(mat, L=cfg.L, H=cfg.H, h=cfg.h, n_steps=cfg.n_steps, t_end=cfg.t_end)
    from .cases import setup_thermal_shock
    if cfg.method not in ("am", "oram"):
        raise ConfigError(f"[solver] method {cfg.method} needs the coupled Newton step, which the element-list "
                          "path of [case] thermal_shock does not have; use method am or oram")
    return setup_thermal_shock(mat, L=cfg.L, H=cfg.H, h=cfg.h, dT_factor=cfg.dT_factor, n_steps=cfg.n_steps,
                               tau_min=cfg.tau_min, tau_max=cfg.tau_max)


# ---- artifacts ---------------------------------------------------------------------------------

ENERGY_COLUMNS = ("step", "load", "elastic", "dissipated", "total", "am_iters", "newton_iters",
                  "krylov_iters", "omega_bar_min")
ITERATION_COLUMNS = ("step", "phase", "cycle", "iteration", "residual", "omega_bar", "elastic",
                     "dissipated", "total")
SUMMARY_COLUMNS = ("parameter", "value", "total_am_iters", "total_newton_iters",
                   "avg_krylov_per_newton", "wall_time_s", "reduction", "status")


def _write(path: Path, text: str) -> None:
    try:
        path.parent.mkdir(parents=True, exist_ok=True)
        path.write_text(text)
    except OSError as exc:
        raise OSError(f"cannot write {path}: {exc}") from exc


def _csv(columns, rows) -> str:
    lines = [",".join(columns)]
    lines += [",".join(_fmt(r[c]) for c in columns) for r in rows]
    return "\n".join(lines) + "\n"


def write_energies_csv(path: Path, records: list) -> None:
    _write(path, _csv(ENERGY_COLUMNS, [
        dict(step=r.step, load=float(r.load), elastic=float(r.energy.elastic),
             dissipated=float(r.energy.dissipated), total=float(r.energy.total),
             am_iters=r.report.am_iterations, newton_iters=r.report.newton_iterations,
             krylov_iters=r.report.total_krylov_iterations,
             omega_bar_min=float(r.report.omega_bar_min)) for r in records]))


def write_iterations_csv(path: Path, rows: list) -> None:
    _write(path, _csv(ITERATION_COLUMNS, [
        {c: (float(r[c]) if isinstance(r[c], (float, np.floating)) else r[c]) for c in ITERATION_COLUMNS}
        for r in rows]))


def triangles(mesh) -> np.ndarray:
    """(T, 3) vertex triples in the reference element order (mesh.py:95-99): every cell's first
    triangle (I-major), then every second one; crossed: the 4 centre fans in turn.  Element-list
    meshes carry their triangles."""
    if getattr(mesh, "elements", None) is not None:
        return np.asarray(mesh.elements, dtype=np.intp)
    nx, ny = mesh.nx, mesh.ny
    I, J = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij"))
    v00, v10 = I * (ny + 1) + J, (I + 1) * (ny + 1) + J
    v11, v01 = v10 + 1, v00 + 1
    if mesh.pattern == "crossed":
        ctr = (nx + 1) * (ny + 1) + I * ny + J
        parts = [(v00, v10, ctr), (v10, v11, ctr), (v11, v01, ctr), (v01, v00, ctr)]
    elif mesh.pattern == "right":
        parts = [(v00, v10, v11), (v00, v11, v01)]
    else:  # union_jack: the diagonal alternates with the cell parity
        even = (I + J) % 2 == 0
        parts = [(v00, v10, np.where(even, v11, v01)),
                 (np.where(even, v00, v10), v11, v01)]
    return np.vstack([np.column_stack(p) for p in parts]).astype(np.intp)


def write_vtk(path: Path, mesh, alpha: np.ndarray, u: np.ndarray, title: str) -> None:
    """Legacy ASCII VTK: triangles, point damage and displacement (runio.py:406-431 layout)."""
    tri = triangles(mesh)
    xy = mesh.vertices
    buf = io.StringIO()
    buf.write(f"# vtk DataFile Version 3.0\n{title}\nASCII\nDATASET UNSTRUCTURED_GRID\n")
    buf.write(f"POINTS {xy.shape[0]} double\n")
    buf.writelines(f"{float(x)!r} {float(y)!r} 0.0\n" for x, y in xy)
    buf.write(f"CELLS {tri.shape[0]} {4 * tri.shape[0]}\n")
    buf.writelines(f"3 {a} {b} {c}\n" for a, b, c in tri)
    buf.write(f"CELL_TYPES {tri.shape[0]}\n" + "5\n" * tri.shape[0])
    buf.write(f"POINT_DATA {xy.shape[0]}\nSCALARS alpha double 1\nLOOKUP_TABLE default\n")
    buf.writelines(f"{float(a)!r}\n" for a in alpha)
    buf.write("VECTORS displacement double\n")
    buf.writelines(f"{float(u[2 * i])!r} {float(u[2 * i + 1])!r} 0.0\n" for i in range(xy.shape[0]))
    _write(path, buf.getvalue())


def write_provenance(path: Path, cfg: RunConfig, setup) -> None:
    from . import __version__
    material = setup.ops.material if hasattr(setup, "ops") else setup.problem.material
    lines = [f"paper_1511_08463_b200 {__version__} (B200 device path)",
             f"elastic_regime = {material.regime}", f"case = {setup.name}"]
    lines += [f"{k} = {_fmt(setup.params[k])}" for k in sorted(setup.params)
              if isinstance(setup.params[k], (int, float, str))]
    lines += ["", "--- config echo ---", echo_config(cfg)]
    _write(path, "\n".join(lines))


# ---- run / sweep ---------------------------------------------------------------------------------

def _execute(cfg: RunConfig):
    from .cases import StepFailureError, run_quasistatic
    setup = build_setup(cfg)
    scfg = build_solver_config(cfg)
    rows, step = [], [-1]
    apply = setup.apply_load

    def counted(*args):  # (problem, state, t) structured, (ops, t) element-list
        step[0] += 1
        return apply(*args)

    setup.apply_load = counted
    scfg.log_callback = lambda rec: rows.append({"step": step[0], **rec})
    try:
        return setup, run_quasistatic(setup, scfg, snapshot_stride=cfg.snapshot_stride), rows, None
    except StepFailureError as exc:
        return setup, exc.records, rows, exc


def run(cfg: RunConfig, output_dir: Optional[str] = None, snapshot_stride: Optional[int] = None) -> int:
    """Execute one configuration and write its artifacts: 0 converged, 3 solver failure."""
    if output_dir is not None:
        cfg = dataclasses.replace(cfg, directory=output_dir)
    if snapshot_stride is not None:
        cfg = dataclasses.replace(cfg, snapshot_stride=snapshot_stride)
    validate_config(cfg)
    setup, records, rows, err = _execute(cfg)
    out = Path(cfg.directory)
    write_provenance(out / "provenance.txt", cfg, setup)
    write_energies_csv(out / "energies.csv", records)
    write_iterations_csv(out / "iterations.csv", rows)
    for r in records:
        if r.alpha is not None:
            write_vtk(out / f"step_{r.step:04d}.vtk", setup.mesh, r.alpha, r.u,
                      f"{setup.name} step {r.step}")
    if err is not None:
        _write(out / "FAILED.txt", f"{err}\n")
        print(f"solver failure: {err}", file=sys.stderr)
        return 3
    return 0


def _energies_totals(path: Path):
    with open(path) as fh:
        head = fh.readline().strip().split(",")
        cols = [head.index(c) for c in ("am_iters", "newton_iters", "krylov_iters")]
        tot = np.zeros(3, dtype=np.int64)
        for line in fh:
            parts = line.strip().split(",")
            tot += [int(parts[i]) for i in cols]
    return (int(t) for t in tot)


_WORKER = {"device": None}


def _worker_init(counter, lock):
    """Pin a sweep worker process to one GPU (worker w -> device w mod count)."""
    import torch
    with lock:
        w = counter.value
        counter.value += 1
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n:
        _WORKER["device"] = device_for_worker(w, n)
        torch.cuda.set_device(_WORKER["device"])


def device_for_worker(worker: int, n_devices: int) -> int:
    return worker % n_devices


def sweep_row(job) -> dict:
    """One sweep row: run the base config with `parameter = value` into `<dir>/<param>_<value:g>`."""
    cfg, parameter, value = job
    row = dict(parameter=parameter, value=value, total_am_iters=0, total_newton_iters=0,
               avg_krylov_per_newton=0.0, wall_time_s=0.0, reduction=0.0, status="failed")
    t0 = time.perf_counter()
    try:
        rc = dataclasses.replace(cfg, **{parameter: value})
        rc = dataclasses.replace(rc, directory=str(Path(cfg.directory) / f"{parameter}_{value:g}"))
        validate_config(rc)
        status = run(rc)
        am, nw, kr = _energies_totals(Path(rc.directory) / "energies.csv")
        row.update(total_am_iters=am, total_newton_iters=nw,
                   avg_krylov_per_newton=kr / nw if nw else 0.0, status="ok" if status == 0 else "failed")
    except Exception:  # noqa: BLE001  a failed row is reported, the sweep goes on
        pass
    row["wall_time_s"] = time.perf_counter() - t0
    return row


def summarise(parameter: str, rows: list) -> list:
    """Fill the `reduction` column: 1 - AM iterations / those of the reference row (the omega = 1
    row of an omega sweep, else the first row); 0 when either row failed."""
    ref = next((r for r in rows if parameter == "omega" and r["value"] == 1.0 and r["status"] == "ok"),
               rows[0])
    for r in rows:
        ok = ref["status"] == "ok" and r["status"] == "ok" and ref["total_am_iters"] > 0
        r["reduction"] = 1.0 - r["total_am_iters"] / ref["total_am_iters"] if ok else 0.0
    return rows


def sweep(spec: SweepSpec, threads: int = 1, output_dir: Optional[str] = None) -> int:
    """One run per swept value, then summary.csv (runio.py:550-590).  threads > 1: that many
    spawned worker processes, each pinned to a GPU (replicas, no collectives)."""
    base = spec.base if output_dir is None else dataclasses.replace(spec.base, directory=output_dir)
    jobs = [(base, spec.parameter, float(v)) for v in spec.values]
    if threads > 1:
        ctx = mp.get_context("spawn")  # CUDA cannot be forked
        counter, lock = ctx.Value("i", 0), ctx.Lock()
        with ProcessPoolExecutor(max_workers=threads, mp_context=ctx, initializer=_worker_init,
                                 initargs=(counter, lock)) as pool:
            rows = list(pool.map(sweep_row, jobs))
    else:
        rows = [sweep_row(j) for j in jobs]
    _write(Path(base.directory) / "summary.csv", _csv(SUMMARY_COLUMNS, summarise(spec.parameter, rows)))
    return 0


def main(argv: Optional[list] = None) -> int:
    """`python -m paper_1511_08463_b200 run|sweep|validate cfg.ini` (reference cli.py)."""
    import argparse
    from .linalg import LinearSolverError
    ap = argparse.ArgumentParser(prog="paper_1511_08463_b200",
                                 description="Phase-field fracture runs on B200: run, sweep, validate.")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("run", "sweep", "validate"):
        p = sub.add_parser(name)
        p.add_argument("config_file")
        p.add_argument("--output-dir", default=None)
        p.add_argument("--snapshot-stride", type=int, default=None)
        p.add_argument("--threads", type=int, default=1)
    a = ap.parse_args(argv)
    try:
        text = Path(a.config_file).read_text()
    except OSError as exc:
        print(f"error: cannot read {a.config_file}: {exc}", file=sys.stderr)
        return 4
    try:
        if a.command == "validate":
            sys.stdout.write(echo_config(parse_config(text)))
            return 0
        if a.command == "run":
            return run(parse_config(text), output_dir=a.output_dir, snapshot_stride=a.snapshot_stride)
        return sweep(parse_sweep(text), threads=a.threads, output_dir=a.output_dir)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    except (LinearSolverError, ValueError) as exc:
        print(f"solver error: {exc}", file=sys.stderr)
        return 3 if isinstance(exc, LinearSolverError) else 2
    except OSError as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return 4
