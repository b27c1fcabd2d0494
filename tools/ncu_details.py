"""Condense an `ncu --page details --csv` export to the lines that matter.

    python tools/ncu_details.py gpurun_out/details_X.csv [--all]
"""

import csv
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Block Size",
        "Grid Size", "L2 Hit Rate", "L1/TEX Hit Rate", "Issue Slots Busy", "Executed Ipc Active",
        "No Eligible", "Dynamic Shared Memory Per Block", "Waves Per SM", "Warp Cycles Per Issued",
        "Mem Busy", "Max Bandwidth", "Elapsed Cycles", "SM Frequency", "DRAM Frequency")


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[0]
    sec, name, unit, val = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                                   "Metric Value"))
    kn = h.index("Kernel Name")
    print(rows[1][kn][:120])
    for r in rows[1:]:
        if "--all" in sys.argv or any(r[name].startswith(k) for k in KEEP):
            print(f"  {r[sec][:28]:28s} {r[name][:44]:44s} {r[val]:>14s} {r[unit]}")
    # rule messages
    if "Rule Name" in h:
        pass


if __name__ == "__main__":
    main()
