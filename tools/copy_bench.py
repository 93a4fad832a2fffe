"""H2D/D2H rates: contiguous pinned copies vs the pitched stkb_upload/download path."""

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04671_b200 import DeviceTarget  # noqa: E402
from paper_2309_04671_b200 import GridBuffer  # noqa: E402

shape, o = (1024, 1024, 1024), 4
padded = tuple(e + 2 * o for e in shape)
h = torch.zeros(padded, dtype=torch.float32, pin_memory=True)
d = torch.empty(padded, dtype=torch.float32, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print("torch contiguous H2D GB/s", h.numel() * 4 / (time.perf_counter() - t) / 1e9)
    t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print("torch contiguous D2H GB/s", h.numel() * 4 / (time.perf_counter() - t) / 1e9)
g = GridBuffer("f32", shape, o, h.numpy())
with DeviceTarget({"u": g}, ["u"]) as dt:
    for _ in range(2):
        t = time.perf_counter(); dt.upload("u", g.data); print("stkb_upload GB/s", g.data.nbytes / (time.perf_counter() - t) / 1e9)
        t = time.perf_counter(); dt.download("u", g.data); print("stkb_download GB/s", g.data.nbytes / (time.perf_counter() - t) / 1e9)
