"""Does the fused halo exchange work between two GPUs of this box?

The z-slab engine's default transport (slabs.run_step_p2p) has each rank's
streaming kernel issue TMA loads (cp.async.bulk.tensor) against tensor maps over
its neighbours' buffers, and orders the ranks with stream memory operations on
peer flag words.  Before a multi-GPU run commits to it, rank 0 runs this probe in
a child process (so a fault cannot take the run down): a 2-slab split of a small
star3d4r problem on devices (a, b), wired in-process (slabs.connect_local), run
for a few steps and compared bit for bit with the same program run unsplit on
device a.  The fast path's per-point operation order does not depend on how
d0 is chunked, so the two must be identical.  Any error, mismatch or timeout
means "use the NCCL transport" (slabs.DeviceSlabEngine.connect_ipc).

    python -m paper_2309_04671_b200.peer_probe A B      # prints one JSON line
"""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def run(dev_a: int, dev_b: int, steps: int = 3) -> dict:
    import numpy as np
    import torch

    from . import corpus
    from .backend import DeviceTarget
    from .front import module

    GridBuffer, fill_loguniform = module("grids").GridBuffer, module("grids").fill_loguniform
    from .slabs import DeviceSlabEngine, SlabPlan, connect_local

    shape = (24, 40, 136)
    bound, decls = corpus.config_target("star3d4r_norm", shape, steps, "f32")
    body = next(s for s in bound.stmts if type(s).__name__ == "BoundFor").body
    names = list(decls)
    grids = {n: GridBuffer.zeros(d.shape, d.order, d.dtype) for n, d in decls.items()}
    fill_loguniform(grids["u"], 11)
    order = grids["u"].order

    with DeviceTarget(grids, names, device=dev_a) as dt:
        for n in names:
            dt.upload(n, grids[n].data)
        dt.set_program(body)
        dt.run(steps)
        dt.sync()
        ref = {n: dt.download(n) for n in names}

    engines = []
    for r, dev in enumerate((dev_a, dev_b)):
        plan = SlabPlan(shape[0], 2, r, order)
        eng = DeviceSlabEngine(body, decls, plan, device=dev, transport="p2p")
        for n in names:
            eng.dt.upload(n, np.ascontiguousarray(grids[n].data[plan.global_slice()]))
        engines.append(eng)
    connect_local(engines)
    for _ in range(steps):
        for eng in engines:
            eng.step(None)
    for eng in engines:
        eng.finish()
    for dev in {dev_a, dev_b}:
        torch.cuda.synchronize(dev)
    o = order
    same = True
    for n in names:
        parts = [eng.dt.download(n)[o:-o, o:-o, o:-o] for eng in engines]
        same &= bool(np.array_equal(np.concatenate(parts, axis=0), ref[n][o:-o, o:-o, o:-o]))
    for eng in engines:
        eng.close()
    return {"ok": same, "devices": [dev_a, dev_b], "why": "" if same else "slab result differs from unsplit"}


_VERDICTS: dict = {}  # (dev_a, dev_b) -> (ok, why): one child process per device pair and process
PROBES_RUN = [0]


def probe(dev_a: int, dev_b: int, timeout: float = 240.0) -> tuple:
    """(ok, why) from a child process, cached per device pair; never raises."""
    key = (int(dev_a), int(dev_b))
    if key not in _VERDICTS:
        PROBES_RUN[0] += 1
        _VERDICTS[key] = _probe(dev_a, dev_b, timeout)
    return _VERDICTS[key]


def _probe(dev_a: int, dev_b: int, timeout: float) -> tuple:
    try:
        r = subprocess.run([sys.executable, "-m", "paper_2309_04671_b200.peer_probe", str(dev_a), str(dev_b)],
                           cwd=str(ROOT), capture_output=True, text=True, timeout=timeout)
    except (subprocess.TimeoutExpired, OSError) as exc:
        return False, f"peer-pull probe did not finish ({type(exc).__name__})"
    for line in reversed(r.stdout.strip().splitlines()):
        try:
            d = json.loads(line)
        except ValueError:
            continue
        return bool(d.get("ok")), d.get("why", "")
    tail = (r.stderr.strip().splitlines() or ["no output"])[-1]
    return False, f"peer-pull probe failed (exit {r.returncode}): {tail[:200]}"


if __name__ == "__main__":
    a, b = int(sys.argv[1]), int(sys.argv[2])
    try:
        out = run(a, b)
    except Exception as exc:  # reported to the parent, which falls back to NCCL
        out = {"ok": False, "devices": [a, b], "why": f"{type(exc).__name__}: {exc}"[:300]}
    print(json.dumps(out), flush=True)
