"""``python -m paper_2309_04671_b200 run prog.stpy`` — the reference CLI's run path on B200.

Mirrors ``stencilkit run --backend gpu`` (cli.py:246-283): launch-block
parameters overridden by flags (cli.py:65-89), the plan resolved from the
first map (cli.py:121-128), initial grids from zeros / ``--grid name=path`` /
``--random-init`` (cli.py:219-243), every final grid written as STG1 to
``-o`` (``wrote <path>`` on stderr), and ``--oracle`` comparing the first
target grid with the reference executor (needs the reference package) and
printing ``max= rmsd= at=``.  Exit codes: 0 ok, 1 diagnostics/usage, 2
tolerance failure, 3 internal error (cli.py:1-4).
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

from . import stpy
from .backend import ExecutionError, run_gpu
from .grids import GridBuffer, compare, fill_loguniform, load_grid, save_grid
from .planning import PlanError, plan_gpu
from .program import AnalysisError, stmt_kind

DEFAULT_MAX_TOL = 1e-7
DEFAULT_RMSD_TOL = 1e-8


class CliError(Exception):
    pass


def _ints(text: str) -> tuple:
    return tuple(int(p) for p in text.split(","))


def _first_map(stmts):
    for s in stmts:
        k = stmt_kind(s)
        if k == "BoundMap":
            return s
        if k == "BoundFor":
            m = _first_map(s.body)
            if m is not None:
                return m
    return None


def cmd_run(a) -> int:
    t0 = time.perf_counter()
    prog = stpy.load(Path(a.file).read_text(), a.file)
    bound = stpy.bind(prog, a.target, scheme=a.scheme, iters=a.iters)
    params = dict(prog.params) if prog.backend == "gpu" else {}
    for flag, key in (("template", "template"), ("mem_type", "memType"), ("capability", "computeCapability"),
                      ("scheme", "scheme")):
        if getattr(a, flag):
            params[key] = getattr(a, flag)
    if a.block:
        params["threadsPerBlock"] = _ints(a.block)
    if a.plane:
        params["planeDims"] = _ints(a.plane)
    params.setdefault("computeCapability", "10.0")
    first = _first_map(bound.stmts)
    if first is None:
        raise CliError("target has no map invocation to plan")
    plan = plan_gpu(first.info, params)
    t1 = time.perf_counter()

    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in prog.grids.items()}
    for spec in a.grid or []:
        name, _, path = spec.partition("=")
        if not path or name not in grids:
            raise CliError(f"--grid expects name=path of a declared grid, got '{spec}'")
        g = load_grid(path)
        d = prog.grids[name]
        if tuple(g.shape) != tuple(d.shape) or g.order != d.order:
            raise CliError(f"grid file {path} is shape {g.shape}/order {g.order}, declared {d.shape}/order {d.order}")
        grids[name] = g
    if a.random_init is not None:
        firstg = next((x for x in prog.args if isinstance(x, str) and x in grids), next(iter(grids)))
        fill_loguniform(grids[firstg], a.random_init)
    result = run_gpu(bound, plan, grids, precision=a.precision)
    t2 = time.perf_counter()

    out = Path(a.outdir)
    out.mkdir(parents=True, exist_ok=True)
    for name, buf in sorted(result.items()):
        save_grid(out / f"{name}.grid", buf)
        print(f"wrote {out / f'{name}.grid'}", file=sys.stderr)
    code = 0
    if a.oracle:
        try:
            from stencilkit.executor import run_target  # the reference oracle
        except ImportError:
            raise CliError("--oracle needs the reference package (stencilkit) on PYTHONPATH") from None
        ref = run_target(bound, grids)
        main = bound.grid_params[0][1]
        rep = compare(ref[main], result[main])
        print(rep.render())
        if not rep.within(a.max_tol, a.rmsd_tol):
            code = 2
    if a.profile:
        print(f"frontend={t1 - t0:.6f}s codegen=0.000000s execution={t2 - t1:.6f}s")
    return code


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2309_04671_b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="execute a .stpy program on the B200 backend")
    r.add_argument("file")
    r.add_argument("--target")
    r.add_argument("--template")
    r.add_argument("--block")
    r.add_argument("--plane")
    r.add_argument("--mem-type", dest="mem_type", choices=["auto", "registers", "shared"])
    r.add_argument("--capability")
    r.add_argument("--scheme", choices=["unified", "cross_product", "slab7"])
    r.add_argument("--iters", type=int)
    r.add_argument("--grid", action="append")
    r.add_argument("--random-init", type=int, dest="random_init")
    r.add_argument("--oracle", action="store_true")
    r.add_argument("--max-tol", type=float, default=DEFAULT_MAX_TOL, dest="max_tol")
    r.add_argument("--rmsd-tol", type=float, default=DEFAULT_RMSD_TOL, dest="rmsd_tol")
    r.add_argument("--precision", choices=["fast", "exact"], default="fast")
    r.add_argument("-o", "--outdir", default="out")
    r.add_argument("--profile", action="store_true")
    r.set_defaults(func=cmd_run)
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    try:
        return a.func(a)
    except (AnalysisError, PlanError, ExecutionError, CliError, FileNotFoundError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # pragma: no cover
        print(f"internal error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
