"""Executed-instruction mix of one kernel launch in an ncu report: per SASS
opcode and per CUDA source line (ncu --page source, cuda+sass view; the page
has one section per (function, source file), repeated per launch).
usage: ncu_mix.py REPORT FUNCTION-REGEX [launch-index] [top] [--stalls]
(--stalls: source lines by warp-stall samples with their top reasons)"""
import collections
import csv
import re
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, fre, launch=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    func = path = None
    seen = collections.Counter()
    cur = None  # (function, launch) of the current section
    sections = collections.defaultdict(list)
    hdr = None
    for r in rows:
        if r[:1] == ["File Path"]:
            path = r[1]
            continue
        if r[:1] == ["Function Name"]:
            func = r[1]
            seen[(func, path)] += 1
            cur = (func, seen[(func, path)] - 1)
            continue
        if r[:3] == ["Line No", "Source", "Address"]:
            hdr = r
            continue
        if hdr and cur and len(r) == len(hdr):
            sections[cur].append((path, r))
    keys = [k for k in sections if re.search(fre, k[0]) and k[1] == launch]
    if not keys:
        print("no such kernel launch; functions:", sorted({k[0] for k in sections}))
        return
    ie = hdr.index("Instructions Executed")
    ops, lines, tot = collections.Counter(), [], 0.0
    for k in keys:
        for path, r in sections[k]:
            if r[0] not in ("-", ""):
                lines.append((num(r[ie]), path.split("/")[-1] + ":" + r[0], r[1].strip()[:80]))
            elif r[2] not in ("", "...") and r[3] not in ("", "..."):
                n = num(r[ie])
                tot += n
                toks = r[3].split()
                op = toks[1] if toks[0].startswith("@") else toks[0]
                ops[op.split(".")[0]] += n
    print(keys[0][0], "launch", launch, f": {tot / 1e6:.1f}M warp instructions")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n / 1e6:8.2f}M {100 * n / max(tot, 1):5.1f}%")
    lines.sort(reverse=True)
    for n, l, s in lines[:top]:
        print(f"{n / 1e6:8.2f}M {l:>22s} {s}")
    if "--stalls" in sys.argv:
        ks = hdr.index("Warp Stall Sampling (All Samples)")
        sc = [(i, c[6:]) for i, c in enumerate(hdr) if c.startswith("stall_") and "(Not Issued)" not in c]
        st = []
        for k in keys:
            for path, r in sections[k]:
                if r[0] not in ("-", ""):
                    v = num(r[ks])
                    why = sorted(((num(r[i]), c) for i, c in sc), reverse=True)[:3]
                    st.append((v, path.split("/")[-1] + ":" + r[0], r[1].strip()[:60], why))
        tot_s = sum(x[0] for x in st) or 1
        st.sort(key=lambda x: -x[0])
        print("--- stall samples by line")
        for v, l, s, why in st[:top]:
            print(f"{100 * v / tot_s:5.1f}% {l:>22s} {s:60s} " + " ".join(f"{c}:{100 * x / max(v, 1):.0f}%" for x, c in why if x > 0))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0,
         int(sys.argv[4]) if len(sys.argv) > 4 else 30)
