"""One line per profiled kernel from an ncu report: duration, DRAM bytes and
throughput, top stall reasons, issue activity, tensor-pipe activity."""
import csv
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        f = lambda k: float((d.get(k) or "0").replace(",", "") or 0)
        stalls = sorted(((f(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in hdr
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        reverse=True)[:4]
        tot = sum(f(k) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")) or 1
        dur = f("gpu__time_duration.sum")
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        unit = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
        print(f"{d['Kernel Name'][:40]:40s} {dur:9.1f} {rows[1][hdr.index('gpu__time_duration.sum')]} "
              f"dram {f('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}% "
              f"({(rd * unit.get(rows[1][hdr.index('dram__bytes_read.sum')], 1) + wr * unit.get(rows[1][hdr.index('dram__bytes_write.sum')], 1)) / 1e9:.2f} GB) "
              f"issue {f('sm__inst_issued.avg.pct_of_peak_sustained_active'):5.1f}% "
              f"tensor {f('sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active') or f('sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active'):5.1f}% "
              f"l1 {f('l1tex__throughput.avg.pct_of_peak_sustained_active'):5.1f}% lts {f('lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}% | "
              + " ".join(f"{n}:{100 * v / tot:.0f}%" for v, n in stalls))


if __name__ == "__main__":
    main(sys.argv[1])
