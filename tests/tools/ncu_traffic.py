"""Per-launch DRAM traffic of the discriminator kernels from an `ncu --set
full` capture, keyed by the kernel classes of sagips_kernel_times, for
bench.py's roofline "traffic" field.

Round 2 (fused kernels), one capture of the first step's five tcgen05
launches (`ncu --set full -k regex:"k_dfwd|k_gstep|k_bwd" -c 5`):
d_fwd_fused, d_bwd_last, d_bwd_mid, d_bwd_first, g_fused.

usage: ncu_traffic.py OUT.json step.ncu-rep
       ncu_traffic.py OUT.json tc_fwd.ncu-rep tc_bwd.ncu-rep   (round 1's per-layer passes)"""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"):
            i = hdr.index(k)
            d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        res.append((r[hdr.index("Kernel Name")], d))
    return res


def main(out, fwd, bwd=None):
    if bwd is None:
        classes = {fwd: ["d_fwd_fused", "d_bwd_last", "d_bwd_mid", "d_bwd_first", "g_fused"]}
    else:
        classes = {fwd: ["d_fwd_first", "d_fwd_mid", "d_fwd_head"], bwd: ["d_bwd_last", "d_bwd_mid", "d_bwd_first"]}
    res = {}
    for rep, names in classes.items():
        for name, (kern, d) in zip(names, launches(rep)):
            res[name] = {"kernel": kern, "duration_s": d["gpu__time_duration.sum"],
                         "dram_read_bytes": d["dram__bytes_read.sum"], "dram_write_bytes": d["dram__bytes_write.sum"],
                         "traffic_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                         "tensor_pipe_active_pct": d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]}
    doc = {"source": "ncu --set full --clock-control none, one launch per class; "
                     "per-launch DRAM bytes; durations are cold-cache and serialised",
           "workload": "C2 (bench.py default), fp32-class split precision", "rows_d": 2 ** 21, "split": True,
           "classes": res}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    for k, v in res.items():
        print(f"{k:12s} {v['traffic_bytes'] / 1e9:7.3f} GB  ({v['dram_read_bytes'] / 1e9:.3f} rd + "
              f"{v['dram_write_bytes'] / 1e9:.3f} wr)  {v['duration_s'] * 1e6:7.1f} us  {v['kernel'][:40]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
