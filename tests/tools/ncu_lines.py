"""Top source lines of an ncu report by warp-stall samples, with the stall
reasons of each line (ncu --page source, CUDA source view)."""
import csv
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    data = []
    for r in rows:
        if "Warp Stall Sampling (All Samples)" in r:
            hdr = r
            continue
        # CUDA-line rows (the SASS rows under each line have "-" in the line column)
        if hdr and len(r) == len(hdr) and r[0] not in ("-", ""):
            d = dict(zip(hdr[2:], r[2:]))
            d["Line No"], d["Source"] = r[0], r[1]
            data.append(d)
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[key] or 0) for d in data) or 1
    stall_cols = [c for c in hdr if c.startswith("stall_")] if hdr else []
    data.sort(key=lambda d: -float(d[key] or 0))
    for d in data[:top]:
        v = float(d[key] or 0)
        if v <= 0:
            break
        st = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{100 * v / tot:5.1f}% L{d.get('Line No', d.get('#', '?')):>5s} {d['Source'][:70]:70s} "
              + " ".join(f"{n}:{100 * x / max(v, 1):.0f}%" for x, n in st if x > 0))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
