"""The multi-GPU transport probe never raises: without a usable GPU pair (this CPU
container) it reports failure with a reason, and connect_ipc then votes NCCL."""

from __future__ import annotations

import pytest

from paper_2309_04671_b200 import peer_probe


@pytest.mark.timeout(300)
def test_probe_reports_failure_without_gpus():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the GPU suite runs the probe for real")
    ok, why = peer_probe.probe(0, 1, timeout=240)
    assert ok is False
    assert isinstance(why, str) and why


def test_probe_timeout_is_a_failure(monkeypatch):
    import subprocess

    def boom(*a, **k):
        raise subprocess.TimeoutExpired(cmd="probe", timeout=1)

    monkeypatch.setattr(subprocess, "run", boom)
    monkeypatch.setattr(peer_probe, "_VERDICTS", {})  # verdicts are cached per device pair
    ok, why = peer_probe.probe(0, 1, timeout=1)
    assert ok is False and "did not finish" in why
