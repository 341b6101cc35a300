"""Print one summary line per bench JSON in gpurun_out/q_*.json (dev loop)."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/q_*.json")):
    try:
        d = json.load(open(f))
        r = d["roofline"]
        print(f.split("/")[-1], "%.3e" % d["value"], round(d["ms_per_step"], 4),
              "e2e %.3e" % d["e2e"]["value"], r["kernel"], "frac %.3f" % r["frac"],
              round(r["avg_launch_ms"], 4),
              {k: round(v, 3) for k, v in r["kernel_time_share"].items() if v > 0.004})
    except Exception as e:  # noqa: BLE001
        print(f, e)
