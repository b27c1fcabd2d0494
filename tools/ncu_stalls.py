"""Summarise an ncu report: time, DRAM bytes/throughput, issue activity and the
top warp-stall reasons per kernel.   python tools/ncu_stalls.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread"]
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        print(r[idx["Kernel Name"]][:90])
        for k in keys:
            if k in idx:
                print(f"   {k} = {r[idx[k]]} {rows[1][idx[k]]}")
        st = []
        for h in stall:
            try:
                st.append((float(r[idx[h]]), h))
            except ValueError:
                pass
        for v, h in sorted(st, reverse=True)[:8]:
            print("   stall %-28s %.2f" % (h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], v))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
