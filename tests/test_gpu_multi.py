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
    ("rma-ag", 2, 1, 0), ("rma-chunked", 2, 0, 0)])
def test_two_gpu_exchange(mode, group, stale, outer):
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode, group, stale, 6, outer)


@pytest.mark.parametrize("mode,group,stale,outer", [("rma-ag", 2, 1, 0), ("sync", 2, 0, 0), ("rma-chunked", 2, 0, 0),
                                                     ("rma", 2, 1, 0)])
def test_two_gpu_exchange_graph_steps(mode, group, stale, outer):
    """the same parity through CUDA-graph steps (SAGIPS_STEP_GRAPH): the push /
    wait / fold / Adam(G) kernels captured with the step and replayed"""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode, group, stale, 6, outer, 0, 1)


@pytest.mark.parametrize("mode,group,stale,outer", [
    ("rma", 4, 0, 0), ("rma", 2, 0, 2), ("arar-arar", 2, 1, 3), ("rma", 4, 1, 0), ("rma-ag", 4, 0, 0),
    ("rma-ag", 4, 1, 0), ("rma-ag", 2, 1, 2), ("rma-chunked", 4, 0, 0), ("rma-chunked", 2, 0, 2)])
def test_four_gpu_grouping(mode, group, stale, outer):
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, mode, group, stale, 6, outer)


@pytest.mark.parametrize("mode,group,stale,outer", [("rma-ag", 2, 1, 2), ("rma", 4, 1, 0), ("rma-chunked", 2, 0, 2)])
def test_four_gpu_grouping_graph_steps(mode, group, stale, outer):
    """grouping through CUDA-graph steps; the steps whose outer ring fires on
    a leader run eagerly (sagips.h SAGIPS_STEP_GRAPH) between graph steps"""
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, mode, group, stale, 6, outer, 0, 1)


@pytest.mark.parametrize("mode,group,stale,outer", [("rma", 2, 1, 0), ("sync", 2, 0, 0), ("arar", 2, 0, 0)])
def test_two_gpu_fused_bias_packet(mode, group, stale, outer):
    """Tensor fusion: the packet carries the bias
    gradients too and Adam(G) applies their reduction."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, mode, group, stale, 6, outer, 1)


def test_four_gpu_paper_size_staleness0_ring_completes():
    """Regression: at C2 sizes the fused pull (k_wait_fold_adam) puts a
    spinning CTA on every SM; the one-sided ring's forwarding agent must
    still fit beside them at g = 4, staleness 0 (it once needed a whole SM's
    register file and the ring timed out)."""
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "bench.py"),
           "--gpus", "4", "--mode", "rma", "--staleness", "0", "--steps", "10", "--warmup", "3",
           "--no-cpu-baseline", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and '"n_gpus": 4' in r.stdout, (r.stdout + r.stderr)[-4000:]
