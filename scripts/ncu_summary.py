"""Summarise ncu outputs (run here, no GPU): the launch list (per-kernel share of the
step) and the --set full captures (dram bytes, throughput, occupancy, stall mix)."""
import csv
import collections
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__shared_mem_per_block_dynamic",
           "sm__cycles_elapsed.avg.per_second", "lts__t_sectors_srcunit_tex_op_read.sum",
           "smsp__inst_executed.sum", "l1tex__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    return agg


def full(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append({"kernel": d.get("Kernel Name", "")[:120],
                    **{m: (d.get(m), u.get(m)) for m in METRICS if m in d}})
    return out


if __name__ == "__main__":
    res = {}
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        res["launch_list"] = {k: {"launches": v[0], "total_ms": v[1] / 1e6} for k, v in launches(lp).items()}
    for name in ("prof_adam", "prof_flatten"):
        p = os.path.join(OUT, name + ".ncu-rep")
        if os.path.exists(p):
            res[name] = full(p)
    json.dump(res, sys.stdout, indent=1)
