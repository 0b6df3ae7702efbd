"""Multi-GPU exchange parity (needs >= 2 GPUs on one node; skipped otherwise):
each mode of Tab. III plus the synchronous all-reduce, with and
without staleness and grouping, against the oracle's lockstep simulation."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(nproc, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    cmd += [str(a) for a in args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MGPU_OK" in out, out[-4000:]


@pytest.mark.parametrize("mode,group,stale,outer", [
    ("rma", 2, 0, 0), ("rma", 2, 1, 0), ("arar", 2, 0, 0), ("arar", 2, 1, 0), ("sync", 2, 0, 0), ("none", 2, 0, 0),
    ("rma-ag", 2, 1, 0)])
def test_two_gpu_exchange(mode, group, stale, outer):
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode, group, stale, 6, outer)


@pytest.mark.parametrize("mode,group,stale,outer", [
    ("rma", 4, 0, 0), ("rma", 2, 0, 2), ("arar-arar", 2, 1, 3), ("rma", 4, 1, 0), ("rma-ag", 4, 0, 0),
    ("rma-ag", 4, 1, 0), ("rma-ag", 2, 1, 2)])
def test_four_gpu_grouping(mode, group, stale, outer):
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, mode, group, stale, 6, outer)


@pytest.mark.parametrize("mode,group,stale,outer", [("rma", 2, 1, 0), ("sync", 2, 0, 0), ("arar", 2, 0, 0)])
def test_two_gpu_fused_bias_packet(mode, group, stale, outer):
    """Tensor fusion: the packet carries the bias
    gradients too and Adam(G) applies their reduction."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode, group, stale, 6, outer, 1)
