"""Long-run drift of the fp32-class tensor-core discriminator against the
CUDA-core fp32 one at C2 (one GPU, same seed and inputs): two contexts, one
with disc_impl = tcgen05 (bf16x3 fused kernels, the product path) and one
with the CUDA-core fp32 kernels, trained side by side for --steps steps.
Every --every steps: both losses, the relative L2 distance between their
generator and discriminator weights, and the generator's mean constrained
parameters (the loop-closure estimate).  GAN training is chaotic, so
the trajectories separate eventually whatever the arithmetic; what this
shows is how fast, against the per-step parameter change (Adam moves a
weight by ~lr per step).  Diagnostic tool (not a parity test)."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_00051_b200 import _lib as L  # noqa: E402
from paper_2407_00051_b200 import runtime  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=600)
    p.add_argument("--every", type=int, default=50)
    p.add_argument("--out", default="gpurun_out/drift.json")
    a = p.parse_args()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ctxs = []
    for impl in (0, 1):
        cfg = L.config_init(L.PRESET_PAPER)
        cfg.disc_impl = impl
        ctxs.append(runtime.make_context(cfg))
    for which in (L.T_GEN_W, L.T_GEN_B, L.T_DISC_W, L.T_DISC_B):  # identical starting points
        ctxs[1].set(which, ctxs[0].get(which))
    rows = []
    w0 = ctxs[0].get(L.T_GEN_W).astype(np.float64)
    for t in range(a.steps):
        for c in ctxs:
            c.train_step(t, 0, sp)
        if (t + 1) % a.every == 0 or t == 0:
            s = [c.get(L.T_STATS) for c in ctxs]
            gw = [c.get(L.T_GEN_W).astype(np.float64) for c in ctxs]
            dw = [c.get(L.T_DISC_W).astype(np.float64) for c in ctxs]
            cm = [c.get(L.T_C).reshape(-1, 6).mean(axis=0) for c in ctxs]
            rows.append({"step": t + 1, "loss_d": [x.loss_d for x in s], "loss_g": [x.loss_g for x in s],
                         "gen_w_rel_l2": float(np.linalg.norm(gw[0] - gw[1]) / np.linalg.norm(gw[0])),
                         "gen_w_moved_rel_l2": float(np.linalg.norm(gw[0] - w0) / np.linalg.norm(w0)),
                         "disc_w_rel_l2": float(np.linalg.norm(dw[0] - dw[1]) / np.linalg.norm(dw[0])),
                         "c_mean": [cm[0].tolist(), cm[1].tolist()]})
            r = rows[-1]
            print(f"step {r['step']:5d}  loss_d {r['loss_d'][0]:.6f} / {r['loss_d'][1]:.6f}  "
                  f"loss_g {r['loss_g'][0]:.6f} / {r['loss_g'][1]:.6f}  "
                  f"|dG|/|G| {r['gen_w_rel_l2']:.2e} (moved {r['gen_w_moved_rel_l2']:.2e})  "
                  f"|dD|/|D| {r['disc_w_rel_l2']:.2e}", flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rows, f)
    for c in ctxs:
        runtime.close(c)


if __name__ == "__main__":
    main()
