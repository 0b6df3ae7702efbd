"""Summarise an ncu launch list (gpu__time_duration.sum, --clock-control
none) of `bench.py --steps 2`: the kernels of the last full step (from the
last k_normals to the last k_adam before the standalone sampler runs), each
with its time and share of the step.  ncu serialises launches and flushes no
caches between them here, so absolute times are per-launch and only the
shares are compared with the bench line's CUDA-event times."""
import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10][1:]
    names = [re.sub(r"\(.*", "", r[4]).replace("sagips::", "").replace("void ", "") for r in rows]
    ns = [float(r[14]) for r in rows]
    starts = [i for i, n in enumerate(names) if n.startswith("k_gen_fwd")]
    ends = [i for i, n in enumerate(names) if n.startswith("k_fold_adam") or n.startswith("k_adam")]
    s = max(i for i in starts if any(j > i for j in ends))
    e = min(j for j in ends if j > s)
    tot = sum(ns[s:e + 1])
    print(f"one step (launches {s}-{e}, {e - s + 1} kernels): {tot / 1e3:.1f} us")
    for i in range(s, e + 1):
        print(f"  {names[i][:44]:44s} grid {rows[i][8]:>14s} {ns[i] / 1e3:9.1f} us  {ns[i] / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
