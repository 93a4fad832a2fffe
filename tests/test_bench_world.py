"""Multi-GPU bench plumbing, checked on CPU.

* ``bench.py --gpus N`` outside torchrun launches N ranks itself
  (torch.distributed.run, 127.0.0.1) — never a silent one-GPU run — and under
  torchrun a world size other than --gpus is an error line and exit code 2.
* ``slabs.run_slab`` keeps its connected slab engine: the second call on the same
  program allocates nothing, exchanges no IPC handles and runs no peer probe, so the
  N>1 e2e timed call (``slabs.slab_e2e``) contains no setup.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import types

import numpy as np
import pytest

import bench
from conftest import ROOT
from paper_2309_04671_b200 import corpus, front, plan_gpu, slabs


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "3")
    assert "WORLD_SIZE=3" in bench.world_error(types.SimpleNamespace(gpus=2))
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.world_error(types.SimpleNamespace(gpus=2)) is None


def test_mismatched_world_is_an_error_line():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] is None and "WORLD_SIZE=3" in line["error"]


def test_gpus_n_without_torchrun_launches_n_ranks(monkeypatch):
    seen = {}

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return types.SimpleNamespace(returncode=0)

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    rc = bench.launch_world(types.SimpleNamespace(gpus=4), ["--gpus", "4", "--steps", "7"])
    cmd = seen["cmd"]
    assert rc == 0
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    assert cmd[-5].endswith("bench.py")


class _FakeDT:
    np_dtype = np.float32

    def __init__(self):
        self.names = ["u", "v"]
        self.uploads, self.zeros = [], []

    def upload(self, n, data, sync=True):
        self.uploads.append(n)

    def zero(self, n):
        self.zeros.append(n)

    def download(self, n, out, sync=True):
        out[...] = 1.0

    def sync(self):
        pass


class _FakeEngine:
    created = 0

    def __init__(self, body, decls, slab, device, precision):
        _FakeEngine.created += 1
        slabs.SETUP_COUNTS["engines_created"] += 1
        self.transport = "p2p"
        self.dt = _FakeDT()
        self.torch = types.SimpleNamespace(cuda=types.SimpleNamespace(synchronize=lambda *a: None))
        self.steps = 0
        self.closed = False

    def connect_ipc(self, dist):
        slabs.SETUP_COUNTS["ipc_connects"] += 1

    def run(self, n, dist=None):
        self.steps += n

    def finish(self, halo=True):
        pass

    def close(self):
        self.closed = True


def test_run_slab_reuses_its_connected_engine(monkeypatch):
    monkeypatch.setattr(slabs, "_new_engine", _FakeEngine)
    monkeypatch.setattr(slabs, "_SLAB_PARKED", {})
    barriers = []
    dist = types.SimpleNamespace(barrier=lambda: barriers.append(1))
    shape = (16, 12, 20)
    bound, decls = corpus.config_target("star3d4r_norm", shape, 5)
    slab = slabs.SlabPlan(shape[0], 2, 0, 4)
    GridBuffer = front.module("grids").GridBuffer
    local = {n: GridBuffer.zeros((slab.size,) + shape[1:], 4, "f32") for n in decls}
    local["u"].interior[...] = 2.0
    plan = plan_gpu(bound.stmts[0].body[0].info, {"template": "unroll"})
    before = dict(slabs.SETUP_COUNTS)
    slabs.run_slab(bound, plan, local, slab, dist, device=0)
    assert slabs.SETUP_COUNTS["engines_created"] == before["engines_created"] + 1
    assert slabs.SETUP_COUNTS["ipc_connects"] == before["ipc_connects"] + 1
    mid = dict(slabs.SETUP_COUNTS)
    out = slabs.run_slab(bound, plan, local, slab, dist, device=0)
    assert slabs.SETUP_COUNTS == mid  # the second call: no allocation, no IPC exchange
    (eng,) = slabs._SLAB_PARKED.values()
    assert eng.steps == 10 and not eng.closed
    assert eng.dt.zeros == ["v"]  # the dead input of a reused engine is cleared on the device
    assert out["u"].data.shape == local["u"].data.shape
    slabs.release_slab_engines()
    assert eng.closed and not slabs._SLAB_PARKED


def test_peer_probe_runs_once_per_device_pair(monkeypatch):
    from paper_2309_04671_b200 import peer_probe

    calls = []
    monkeypatch.setattr(peer_probe, "_VERDICTS", {})
    monkeypatch.setattr(peer_probe, "_probe", lambda a, b, t: calls.append((a, b)) or (True, ""))
    for _ in range(3):
        assert peer_probe.probe(0, 1) == (True, "")
    peer_probe.probe(1, 2)
    assert calls == [(0, 1), (1, 2)]


@pytest.mark.parametrize("name", ["slab_e2e"])
def test_e2e_reports_setup_of_its_timed_call(name):
    """slab_e2e's result carries the setup counters of the timed call (bench prints them)."""
    import inspect

    src = inspect.getsource(getattr(slabs, name))
    assert "setup_in_timed_call" in src and src.index("before = dict(SETUP_COUNTS") < src.index("t0 = time.perf_counter()")
