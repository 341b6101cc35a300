"""Write profiles/<round>/SUMMARY.md from the bench lines and launch lists in it.

    python tools/summarize_profiles.py profiles/r1
"""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])


def line(name):
    p = d / f"bench_{name}.json"
    if not p.exists():
        return None
    return json.loads(p.read_text().strip().splitlines()[-1])


rows = []
for w in ("bed1m", "bed1m_mode8", "hero50k", "envs", "slab"):
    z = line(w)
    if not z:
        continue
    r, c = z.get("roofline") or {}, {**(z.get("config") or {}), **(z.get("run") or {})}
    cb = z.get("cpu_baseline") or {}
    rows.append(f"| {w} | {z['value']:.3e} | {z['ms_per_step']:.4f} | {z['e2e']['value']:.3e} | "
                f"{r.get('kernel')} | {r.get('frac', 0):.3f} | "
                f"{'-' if r.get('step_frac') is None else format(r['step_frac'], '.3f')} | "
                f"{cb.get('value', float('nan')):.3g} | {c.get('c_pp', 0):.2f} | {c.get('c_b', 0):.3f} | "
                f"{c.get('l2', '-')} |")
ref = line("reference")
clk = (line("bed1m") or line("hero50k") or {}).get("clocks", {})
out = [f"# {d.name} profiles (1x B200, sm_100a, SM clock {clk.get('sm_mhz')} MHz of "
       f"{clk.get('sm_max_mhz')}, throttle reasons {clk.get('reasons')})", "",
       "Bench lines: `bench_<workload>.json` (`python bench.py --workload <w>`; bed1m is the default "
       "workload (tools/gpu_round2.sh has the exact commands)).",
       "Launch lists: `launches_<workload>.csv` (ncu `gpu__time_duration.sum --clock-control none`, "
       "cold cache, serialised), summarised in `launches_summary.txt`.",
       "Full-set ncu captures of the top kernels: `ncu_full_summary.txt` (per kernel: duration, DRAM "
       "bytes, L1/L2 hit rates, occupancy, stall reasons); per-launch DRAM traffic in "
       "`../ncu_summary.json` (read by bench.py as `roofline.traffic`); per-SASS-instruction "
       "executions and stall samples in `sass_*.csv.gz` (attribute to source lines with "
       "`tools/sass_lines.py`).",
       "compute-sanitizer (memcheck, racecheck, synccheck, initcheck): `sanitizer/`.", "",
       "| workload | particle-steps/s | ms/step | e2e particle-steps/s | top kernel | HBM frac (kernel) | "
       "HBM frac (step model) | CPU oracle 1 core | c_pp | c_b | L2 |",
       "|---|---|---|---|---|---|---|---|---|---|---|", *rows, ""]
if ref:
    out.append(f"Reference arm (`bench.py --impl reference`, oracle port, "
               f"{ref['cpu_baseline']['cores']} core, {ref['cpu_baseline'].get('host_cores')} host cores): "
               f"{ref['value']:.3e} particle-steps/s on {ref['config']['workload']} "
               f"({ref['cpu_baseline']['sample']}).")
# where the time goes: kernel shares of each workload's step (bench roofline pass)
out += ["", "## Kernel time shares (device, per step)", ""]
for w in ("bed1m", "bed1m_mode8", "hero50k", "envs"):
    z = line(w)
    if not z:
        continue
    sh = (z.get("roofline") or {}).get("kernel_time_share", {})
    parts = ", ".join(f"{k} {v:.1%}" for k, v in sorted(sh.items(), key=lambda kv: -kv[1])
                      if v >= 0.01 and k != "k_solve")
    out.append(f"* {w}: {parts}")
# ncu full-set digest: one line per captured kernel (first capture of each name)
ncu = d / "ncu_full_summary.txt"
if ncu.exists():
    import re
    out += ["", "## ncu full-set digest (cold cache, one launch each)", "",
            "| capture | kernel | us | DRAM MB (r+w) | warps active | L1 hit | L2 hit | top stall (cycles per issue) |",
            "|---|---|---|---|---|---|---|---|"]
    cap, cur, seen = None, None, set()
    rows = {}
    for ln in ncu.read_text().splitlines():
        if ln.endswith(".ncu-rep"):
            cap = Path(ln.strip()).stem
            continue
        m = re.match(r"\s+--- (?:void )?([A-Za-z_][A-Za-z_0-9]*)(<[^>]*>)?\(", ln)
        if m:
            cur = (cap, m.group(1) + ("" if m.group(2) in (None, "<0>") else m.group(2)))
            if cur not in rows:
                rows[cur] = {}
            continue
        m = re.match(r"\s+(\S+)\s+([0-9.]+)\s*(\S*)", ln)
        if m and cur and m.group(1) not in rows[cur]:
            scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1e-6, "Kbyte": 1e-3,
                     "Mbyte": 1.0, "Gbyte": 1e3}.get(m.group(3), 1.0)
            rows[cur][m.group(1)] = float(m.group(2)) * scale
    for (c, k), r in rows.items():
        stalls = {n.split("stalled_")[1].split("_per_issue")[0]: v for n, v in r.items() if "stalled_" in n
                  and "selected" not in n}
        top = max(stalls.items(), key=lambda kv: kv[1]) if stalls else ("-", 0)
        out.append(f"| {c} | {k} | {r.get('gpu__time_duration.sum', 0):.1f} | "
                   f"{r.get('dram__bytes_read.sum', 0) + r.get('dram__bytes_write.sum', 0):.1f} | "
                   f"{r.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.0f}% | "
                   f"{r.get('l1tex__t_sector_hit_rate.pct', 0):.0f}% | {r.get('lts__t_sector_hit_rate.pct', 0):.0f}% | "
                   f"{top[0]} {top[1]:.1f} |")
(d / "SUMMARY.md").write_text("\n".join(out) + "\n")
print("\n".join(out))
