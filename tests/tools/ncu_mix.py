"""Executed-instruction mix of one kernel in an ncu report: per SASS opcode
and per CUDA source line (ncu --page source, cuda+sass view).
usage: ncu_mix.py REPORT [kernel-index] [top]"""
import collections
import csv
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, kidx=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    starts = [i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"] and "Address" in r]
    end = starts[kidx + 1] if kidx + 1 < len(starts) else len(rows)
    sec = rows[starts[kidx]:end]
    h = sec[0]
    ie = h.index("Instructions Executed")
    ops, lines, tot = collections.Counter(), [], 0.0
    for r in sec[1:]:
        if len(r) != len(h):
            continue
        if r[0] not in ("-", ""):
            lines.append((num(r[ie]), r[0], r[1].strip()[:90]))
        elif r[2] not in ("", "...") and r[3] not in ("", "..."):
            n = num(r[ie])
            tot += n
            toks = r[3].split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += n
    print(f"total warp instructions {tot / 1e6:.1f}M")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n / 1e6:8.2f}M {100 * n / tot:5.1f}%")
    lines.sort(reverse=True)
    for n, l, s in lines[:top]:
        print(f"{n / 1e6:8.2f}M L{l:>5s} {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
