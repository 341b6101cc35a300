"""profiles/ncu_summary.json from .ncu-rep captures: per workload and kernel,
DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) and the
ncu duration.  The logical kernel k_solve (S x k_sweep + k_finish, one step)
is the sum of its parts.  bench.py reports these as roofline.traffic.

    python tools/ncu_traffic.py out.json hero50k=a.ncu-rep bed1m=b.ncu-rep ...
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, row, units)}


def val(d, key, scale=None):
    v, u = d[key]
    x = float(v.replace(",", ""))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
           "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
    return x * mul


def kname(raw):
    """'void gg::k_sweep_rm<false>(gg::Dev, int)' -> 'k_sweep_rm' (the names
    bench.py looks up; templated and plain kernels alike)"""
    n = raw.split("(")[0].replace("gg::", "").strip()
    if n.startswith("void "):
        n = n[5:]
    return n.split("<")[0].strip()


def add_solve(ent, S=10):
    """the logical k_solve of one step: S sweeps (record-major k_sweep_rm, or
    k_sweep) + k_finish (+ k_commit)"""
    sw = ent.get("k_sweep_rm") or ent.get("k_sweep")
    fi = ent.get("k_finish")
    if not sw or not fi:
        return
    co = ent.get("k_commit", {"dram_bytes_per_launch": 0.0, "ncu_us_per_launch": 0.0})
    ent["k_solve"] = {"dram_bytes_per_launch": S * sw["dram_bytes_per_launch"] + fi["dram_bytes_per_launch"]
                                               + co["dram_bytes_per_launch"],
                      "ncu_us_per_launch": S * sw["ncu_us_per_launch"] + fi["ncu_us_per_launch"]
                                           + co["ncu_us_per_launch"],
                      "launches": 1, "source": f"{S} x sweep + k_finish + k_commit (cold-cache ncu replays)"}


def renormalize(path):
    """re-key an existing summary by kname() and recompute k_solve"""
    summary = json.load(open(path))
    for wl, ent in summary.items():
        summary[wl] = {kname(k): v for k, v in ent.items() if k != "k_solve"}
        add_solve(summary[wl])
    json.dump(summary, open(path, "w"), indent=1, sort_keys=True)


def main():
    if sys.argv[1] == "--renormalize":
        for p in sys.argv[2:]:
            renormalize(p)
        return
    out_path = sys.argv[1]
    try:
        summary = json.load(open(out_path))
    except FileNotFoundError:
        summary = {}
    for arg in sys.argv[2:]:
        wl, rep = arg.split("=", 1)
        per = defaultdict(list)
        for d in rows(rep):
            name = kname(d["Kernel Name"][0])
            by = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
            per[name].append((by, val(d, "gpu__time_duration.sum")))
        ent = summary.setdefault(wl, {})
        for name, lst in per.items():
            ent[name] = {"dram_bytes_per_launch": sum(b for b, _ in lst) / len(lst),
                         "ncu_us_per_launch": sum(t for _, t in lst) / len(lst), "launches": len(lst),
                         "source": rep.split("/")[-1]}
        add_solve(ent)
    json.dump(summary, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(summary, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
