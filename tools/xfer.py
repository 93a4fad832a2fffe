"""Host<->device transfer rates of one grid through the C-ABI (development tool).

    python tools/xfer.py [n0 n1 n2]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04671_b200 import DeviceTarget  # noqa: E402
from paper_2309_04671_b200 import GridBuffer  # noqa: E402


def main():
    shape = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 1024, 1024)
    o = 4
    padded = tuple(e + 2 * o for e in shape)
    host = torch.empty(padded, dtype=torch.float32, pin_memory=True).numpy()
    host[...] = 1.0
    g = GridBuffer("f32", shape, o, host)
    dt = DeviceTarget({"u": g}, ["u"])
    for _ in range(2):
        dt.upload("u", host)
        dt.download("u", host)
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        dt.upload("u", host)
    up = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        dt.download("u", host)
    down = (time.perf_counter() - t0) / reps
    gb = host.nbytes / 1e9
    print(f"{gb:.2f} GB  H2D {gb / up:.1f} GB/s  D2H {gb / down:.1f} GB/s")
    dt.close()


if __name__ == "__main__":
    main()
