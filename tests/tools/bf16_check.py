"""Diagnostic: the bf16 G step's dy on the GPU vs a numpy emulation of the
same bf16 roundings and vs the exact oracle, in units of the first-order
standard deviation of tests/bf16_bound.py.  python tests/tools/bf16_check.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import gan, mlp  # noqa: E402
from tests import bf16_bound as B  # noqa: E402
from tests.gpu_util import oracle_config, sync_params, unflat  # noqa: E402


def bf(x):
    x = np.asarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def main():
    from paper_2407_00051_b200 import _lib as L
    from paper_2407_00051_b200 import runtime
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cfg = L.config_init(1, seed=4, param_samples=64, events_per_sample=256, precision=L.PREC_BF16)
    ctx = runtime.make_context(cfg)
    ocfg = oracle_config(cfg)
    st = gan.RankState(ocfg, 0)
    sync_params(ctx, st)
    ctx.train_step(0, L.STEP_LOCAL_ONLY, sp)
    gan.local_step(ocfg, st, 0)
    Ws, bs = unflat(ctx.get(L.T_DISC_W), st.dW), unflat(ctx.get(L.T_DISC_B), st.db)
    y = ctx.get(L.T_EVENTS).reshape(-1, 2)[ocfg.n_events:].astype(np.float64)  # the GPU's own fake rows
    N, a = ocfg.n_events, ocfg.leaky_slope
    z, cache = mlp.forward(Ws, bs, y, a)
    dz = mlp.bce_grad(z[:, 0], np.ones(N))[:, None]
    _, _, dy = mlp.backward(Ws, cache, dz, a)
    h, cc = y, []
    for l in range(len(Ws)):
        zz = bf(h) @ bf(Ws[l]).T + bs[l] if 0 < l < len(Ws) - 1 else h @ Ws[l].T + bs[l]
        cc.append(zz)
        h = mlp.lrelu(zz, a) if l < len(Ws) - 1 else zz
    g = mlp.bce_grad(h[:, 0], np.ones(N))[:, None]
    for l in reversed(range(len(Ws))):
        d = g if l == len(Ws) - 1 else g * mlp.lrelu_grad(cc[l], a)
        g = bf(d) @ bf(Ws[l]) if 0 < l < len(Ws) - 1 else d @ Ws[l]
    emu = g
    gpu = ctx.get(L.T_DY).reshape(-1, 2).astype(np.float64)
    sig = np.sqrt(B.dy_variance(Ws, bs, y, a, 1.0 / N))
    for name, v in (("gpu", gpu), ("emu", emu)):
        r = np.abs(v - dy) / sig
        print(f"{name} vs exact: median {np.median(r):.3f} sigma, p99.9 {np.quantile(r, 0.999):.3f}, max {r.max():.3f}")
    r = np.abs(gpu - emu) / sig
    print(f"gpu vs emu: median {np.median(r):.3f} sigma, max {r.max():.3f}; rel {np.median(np.abs(gpu-emu)/np.abs(emu)):.3g}")
    zl = ctx.get(L.T_LOGITS_G).astype(np.float64)
    print("logit gpu-emu max", np.max(np.abs(zl - h[:, 0])), "gpu-exact max", np.max(np.abs(zl - z[:, 0])))


if __name__ == "__main__":
    main()
