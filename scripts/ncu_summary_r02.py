"""Summarise the round-2 ncu outputs of scripts/profile_r02.sh (run here, no GPU):
the launch lists (per-kernel share of the step) and the --set full captures (raw-page CSV
exports: DRAM bytes, duration, registers, grid, occupancy, issue activity).

  python scripts/ncu_summary_r02.py gpurun_out/prof > profiles/ncu_summary.json
"""
import collections
import csv
import json
import os
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", "ns"), 1e-9)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(v[1] for v in agg.values())
    return {k: {"launches": v[0], "total_ms": v[1] * 1e3, "share": v[1] / total if total else None}
            for k, v in agg.items()}


def raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d, u = dict(zip(hdr, row)), dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:140]}
        for m in METRICS:
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                rec[m] = v * SCALE.get(u.get(m, ""), 1)
        out.append(rec)
    return out


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
    res = {"round": 2, "source": "ncu (gpurun, 1x B200): scripts/profile_r02.sh", "launch_lists": {}, "captures": {}}
    for name in ("launches_7p5b", "launches_mlp"):
        p = os.path.join(d, name + ".csv")
        if os.path.exists(p):
            res["launch_lists"][name] = launches(p)
    for name in ("adam", "flatten", "rs", "copy"):
        p = os.path.join(d, name + ".raw.csv")
        if os.path.exists(p):
            res["captures"][name] = raw(p)
    json.dump(res, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
