"""Compare convergence.py outputs: mean-over-ranks loss curves and the
ensemble parameter residual (Eq. 6) per recorded step."""
import json
import sys

import numpy as np

runs = [json.load(open(p)) for p in sys.argv[1:]]
print("modes:", [(r["mode"], r["world"], r["group_size"], r["staleness"], r["outer_every"]) for r in runs])
print(f"{'step':>6s} " + " ".join(f"{r['mode']:>8s}:L_D  L_G   |r|  " for r in runs))
for i in range(len(runs[0]["records"])):
    row = []
    for r in runs:
        rec = r["records"][i]
        row.append(f"{np.mean(rec['loss_d']):.4f} {np.mean(rec['loss_g']):.4f} {np.mean(np.abs(rec['residual'])):.4f}")
    if i % 6 == 0 or i == len(runs[0]["records"]) - 1:
        print(f"{runs[0]['records'][i]['step']:6d} " + "   ".join(row))
base = runs[1] if len(runs) > 1 else runs[0]
for r in runs:
    dl = [abs(np.mean(a["loss_g"]) - np.mean(b["loss_g"])) / np.mean(b["loss_g"]) for a, b in zip(r["records"], base["records"])]
    print(f"{r['mode']}: max relative deviation of mean L_G from {base['mode']}: {max(dl):.3f}; wall {r['wall_s']:.1f} s")
