"""Phase timing of one run_gpu-equivalent call (development tool).

    python tools/e2e_phases.py [config]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_04671_b200 import DeviceTarget, corpus  # noqa: E402
from paper_2309_04671_b200.backend import _host_array, dead_on_entry, halo_is_zero  # noqa: E402


def once(bound, grids, names, log):
    t = time.perf_counter
    t0 = t()
    dt = DeviceTarget({n: grids[n] for n in names}, names)
    t1 = t()
    dead = dead_on_entry(bound.stmts, names, {})
    for n in names:
        if n in dead and halo_is_zero(grids[n]):
            continue
        dt.upload(n, grids[n].data, sync=False)
    dt.sync()
    t2 = t()
    dt.execute(bound.stmts, None)
    dt.sync()
    t3 = t()
    outs = []
    for n in names:
        arr = _host_array(grids[n].data.shape, dt.np_dtype, True)
        dt.download(n, arr, sync=False)
        outs.append(arr)
    dt.sync()
    t4 = t()
    dt.close()
    t5 = t()
    log.append(dict(create=t1 - t0, h2d=t2 - t1, run=t3 - t2, d2h=t4 - t3, close=t5 - t4, total=t5 - t0))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    builder, shape, dtype, _, _ = bench.CONFIGS[cfg]
    bound, decls = corpus.config_target(builder, shape, 50, dtype)
    grids = bench.pinned_grids(decls, builder)
    names = list(decls)
    log = []
    for _ in range(3):
        once(bound, grids, names, log)
    for r in log:
        print({k: round(v * 1e3, 1) for k, v in r.items()})
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
