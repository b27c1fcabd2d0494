"""Summarize an ncu launch list (gpu__time_duration + dram bytes per launch) by kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [--top 40] [--json out.json]
"""

import argparse
import collections
import csv
import json
import re

_TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    k, m, v, u, i = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                           "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= max(k, m, v, u, i):
            continue
        per[int(r[i])][r[m]] = (r[k], float(r[v].replace(",", "")), r[u])
    out = []
    for _, d in sorted(per.items()):
        name, t, unit = d["gpu__time_duration.sum"]
        us = t * _TIME.get(unit, 1e-3)
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in d:
                b += d[key][1] * _BYTES.get(d[key][2], 1)
        out.append((re.sub(r"\(.*", "", name), us, b))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--json")
    a = ap.parse_args()
    launches = load(a.csv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for name, us, b in launches:
        g = agg[name[:100]]
        g[0] += 1
        g[1] += us
        g[2] += b
    tot = sum(us for _, us, _ in launches)
    print(f"launches {len(launches)}  total {tot:.1f} us (serialized, cold-cache ncu)")
    rows = sorted(agg.items(), key=lambda x: -x[1][1])
    for name, (n, us, b) in rows[:a.top]:
        print(f"{us:9.1f} us {100 * us / tot:5.1f}%  n={n:4d}  {b / 1e6:9.1f} MB  "
              f"{b / max(us, 1e-9) / 1e3:7.0f} GB/s  {name}")
    if a.json:
        json.dump({"total_us": tot, "launches": len(launches),
                   "kernels": [{"name": n, "count": c, "us": us, "dram_bytes": b}
                               for n, (c, us, b) in rows]}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
