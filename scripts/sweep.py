"""Tuning sweep (GPU): run bench.py under each kernel variant and print the phase times."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--adam", default="0,1,11,21")
ap.add_argument("--flat", default="")          # e.g. "4x4,4x8"  (vecs x ctas)
ap.add_argument("--base", default="")          # fixed env for every run, e.g. "ZERO_ADAM_VARIANT=1"
ap.add_argument("--flat-tma", default="")      # e.g. "1,2,3,4"
ap.add_argument("--flat-streams", default="")  # e.g. "1,2,3,4"
ap.add_argument("--env", default="")           # free-form variants: "A=1,B=2|A=0" (one variant per '|')
args, extra = ap.parse_known_args()
base = dict(kv.split("=") for kv in args.base.split(",") if kv)
variants = []
for av in [x for x in args.adam.split(",") if x]:
    variants.append(dict(base, ZERO_ADAM_VARIANT=av))
for fv in [x for x in args.flat.split(",") if x]:
    v, c = fv.split("x")
    variants.append(dict(base, ZERO_FLAT_VECS=v, ZERO_FLAT_CTAS=c))
for fs in [x for x in args.flat_streams.split(",") if x]:
    variants.append(dict(base, ZERO_FLAT_STREAMS=fs))
for ft in [x for x in args.flat_tma.split(",") if x]:
    variants.append(dict(base, ZERO_FLAT_TMA=ft))
for ev in [x for x in args.env.split("|") if x]:
    variants.append(dict(base, **dict(kv.split("=") for kv in ev.split(",") if kv)))
for v in variants:
    env = dict(os.environ, **v)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "30", "--no-e2e",
                        "--no-cpu-baseline"] + extra, env=env, capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(json.dumps({"variant": v, "ms_per_step": round(d["ms_per_step"], 4),
                          "adam_ms": round(d["roofline"]["ms_per_launch"], 4),
                          "adam_frac": round(d["roofline"]["frac"], 4),
                          "reduce_ms": round(d["step_roofline"]["reduce_phase_ms"], 4),
                          "flatten_gbs": round(d["step_roofline"]["flatten_gbs"] or 0, 1),
                          "clocks": d["clocks"]}), flush=True)
    except Exception as e:
        print(json.dumps({"variant": v, "error": str(e), "stderr": r.stderr[-2000:]}), flush=True)
