"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
per kernel: share of device time, launches, mean time, DRAM bytes, GB/s."""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def main(path, top=14):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    seen = set()
    for d in data:
        k = d["Kernel Name"].split("(")[0][:60]
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            agg[k]["n"] += 1
            agg[k]["ns"] += v
        elif m == "dram__bytes_read.sum":
            agg[k]["rd"] += v
        elif m == "dram__bytes_write.sum":
            agg[k]["wr"] += v
    tot = sum(a["ns"] for a in agg.values())
    print(f"total {tot / 1e6:.3f} ms over {sum(a['n'] for a in agg.values())} launches")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"])[:top]:
        gbs = (a["rd"] + a["wr"]) / a["ns"] if a["ns"] else 0
        print(f"{100 * a['ns'] / tot:5.1f}% n={a['n']:3d} {a['ns'] / a['n'] / 1e3:8.1f} us  rd {a['rd'] / a['n'] / 1e9:5.2f} GB "
              f"wr {a['wr'] / a['n'] / 1e9:5.2f} GB {gbs:7.0f} GB/s  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
