"""Time the reference's CPU path (oracle/_ref) — TEST/BENCH INFRASTRUCTURE ONLY.

Loads the reference-emitted OpenMP C for one bench sample (built by
oracle/build_ref.py) through the reference's own C-ABI —
``run_<target>(T *g0, ..., int64_t iter)``, driven with ctypes exactly as the
reference's acceptance criterion 10 does (tests/test_acceptance.py:325-343) —
and times ``steps`` time steps on all host cores.  Run as a subprocess so the
OpenMP environment (OMP_NUM_THREADS / OMP_PROC_BIND=close /
OMP_SCHEDULE=static) is fixed before libgomp starts:

    python -m oracle.ref_runner --name c4_star3d4r_norm --steps 5 --warmup 1

Prints one JSON object: GPts/s, seconds, cores, sample description.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def load_manifest() -> dict:
    p = REF / "manifest.json"
    if not p.exists():
        raise FileNotFoundError("oracle/_ref/manifest.json missing: run oracle/build_ref.py in the build container")
    return json.loads(p.read_text())


def library(entry: dict, strict: bool = False) -> tuple:
    """Prefer a -march=native rebuild of the emitted C on this host.  ``strict`` adds
    -ffp-contract=off: no FMA contraction, so each product and sum rounds separately in
    float64 as in run_target (the bit-exact comparison of precision='exact')."""
    src = REF / entry["source"]
    flags = ["-O3", "-march=native", "-fopenmp"] + (["-ffp-contract=off"] if strict else [])
    if shutil.which("gcc") and src.exists():
        tag = "strict_" if strict else ""
        out = Path(tempfile.gettempdir()) / f"stkb_ref_native_{tag}{os.getpid()}_{entry['lib']}"
        r = subprocess.run(["gcc", *flags, "-fPIC", "-shared", str(src), "-o", str(out)], capture_output=True)
        if r.returncode == 0:
            return out, " ".join(flags)
    if strict:
        raise RuntimeError("the strict (-ffp-contract=off) build of the reference C needs gcc on this host")
    return REF / entry["lib"], " ".join(entry["cflags"])


def _order(builder: str) -> int:
    if builder == "wave":
        return 4
    if builder == "jacobi7":
        return 1
    return int(builder.split("d")[1][0])  # star3d<R>r[_norm]


def fill(arr: np.ndarray, order: int, seed: int) -> None:
    """Log-uniform interior in [1e-4, 1e5] (grids.py:67-72), drawn plane by plane."""
    rng = np.random.default_rng(seed)
    inner = arr[tuple(slice(order, n - order) for n in arr.shape)]
    for z in range(inner.shape[0]):
        inner[z] = (10.0 ** rng.uniform(-4.0, 5.0, size=inner.shape[1:])).astype(arr.dtype)


def run(name: str, steps: int, warmup: int) -> dict:
    entry = load_manifest()[name]
    path, flags = library(entry)
    lib = ctypes.CDLL(str(path))
    fn = getattr(lib, entry["entry"])
    shape = tuple(entry["shape"])
    order = _order(entry["builder"])
    dt = np.float32 if entry["dtype"] == "f32" else np.float64
    cty = ctypes.c_float if entry["dtype"] == "f32" else ctypes.c_double
    padded = tuple(e + 2 * order for e in shape)
    grids = [np.zeros(padded, dt) for _ in entry["grids"]]
    fill(grids[0], order, 7)
    if entry["builder"] == "wave":  # kappa small and positive, u_prev = u
        grids[2][...] = np.float32(0.01)
        grids[1][...] = grids[0]
    fn.argtypes = [ctypes.POINTER(cty)] * len(grids) + [ctypes.c_int64]
    fn.restype = None
    ptrs = [g.ctypes.data_as(ctypes.POINTER(cty)) for g in grids]
    if warmup:
        fn(*ptrs, ctypes.c_int64(warmup))
    t0 = time.perf_counter()
    fn(*ptrs, ctypes.c_int64(steps))
    sec = time.perf_counter() - t0
    pts = int(np.prod(shape)) * steps
    if path.parent != REF:
        path.unlink(missing_ok=True)
    return dict(value=pts / sec / 1e9, unit="GPts/s", seconds=sec, steps=steps, points_per_step=int(np.prod(shape)),
                cores=int(os.environ.get("OMP_NUM_THREADS", host_cores())), kind="reference",
                sample=f"{name}: reference-emitted OpenMP C (template loop, run_{entry['entry'][4:]}) on "
                       f"{'x'.join(map(str, shape))} {entry['dtype']}, {steps} steps, {flags}")


_LOADED: dict = {}


def call(name: str, arrays: list, steps: int, strict: bool = False) -> float:
    """Run the reference-emitted C of manifest entry ``name`` in this process on
    caller-owned padded arrays (in target-parameter order, mutated in place: the
    reference C-ABI, serial.py:126-208) for ``steps`` time steps; returns seconds.
    Test infrastructure: the parity tests' oracle at BASELINE sizes."""
    entry = load_manifest()[name]
    key = (name, strict)
    if key not in _LOADED:
        path, _ = library(entry, strict)
        _LOADED[key] = ctypes.CDLL(str(path))
    fn = getattr(_LOADED[key], entry["entry"])
    cty = ctypes.c_float if entry["dtype"] == "f32" else ctypes.c_double
    dt = np.float32 if entry["dtype"] == "f32" else np.float64
    order = _order(entry["builder"])
    padded = tuple(e + 2 * order for e in entry["shape"])
    if len(arrays) != len(entry["grids"]):
        raise ValueError(f"{name} takes {len(entry['grids'])} grids")
    for a in arrays:
        if a.dtype != dt or tuple(a.shape) != padded or not a.flags.c_contiguous:
            raise ValueError(f"{name}: arrays must be C-contiguous {dt.__name__}{padded}")
    fn.argtypes = [ctypes.POINTER(cty)] * len(arrays) + [ctypes.c_int64]
    fn.restype = None
    t0 = time.perf_counter()
    fn(*[a.ctypes.data_as(ctypes.POINTER(cty)) for a in arrays], ctypes.c_int64(steps))
    return time.perf_counter() - t0


def main(argv=None) -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args(argv)
    print(json.dumps(run(a.name, a.steps, a.warmup)))


def spawn(name: str, steps: int, warmup: int, timeout: float = 600.0) -> dict:
    """Run in a fresh interpreter with the BASELINE.md §3 OpenMP settings."""
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", str(host_cores()))
    env["OMP_PROC_BIND"] = "close"
    env["OMP_SCHEDULE"] = "static"
    r = subprocess.run([sys.executable, "-m", "oracle.ref_runner", "--name", name, "--steps", str(steps),
                        "--warmup", str(warmup)], cwd=str(HERE.parent), env=env, capture_output=True, text=True,
                       timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"ref_runner failed: {r.stderr[-2000:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    main()
