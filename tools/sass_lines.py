"""Attribute an ncu SASS source page (--page source --print-source sass --csv)
to CUDA source lines using nvdisasm --print-line-info of the same cubin.

usage: python tools/sass_lines.py <sass.csv.gz> <nvdisasm.dis> <mangled kernel> [N]
"""
import collections, csv, gzip, io, re, sys

csv_path, dis_path, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
# offset -> source line from the disassembly
txt = open(dis_path).read()
sec = re.search(r"\.text\.%s:(.*?)(?=\n\s*\.section|\Z)" % re.escape(fn), txt, re.S).group(1)
line_of, cur = {}, "?"
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and ";" in m.group(2):
        line_of[int(m.group(1), 16)] = (cur, m.group(2).split(";")[0].strip())
raw = gzip.open(csv_path, "rt").read() if csv_path.endswith(".gz") else open(csv_path).read()
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = []
for r in rows[hi + 1:]:  # first kernel block only
    if r and r[0] in ("Address", "Kernel Name"):
        break
    if len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
a0 = int(data[0]["Address"], 16)
inst = collections.Counter(); samp = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for d in data:
    off = int(d["Address"], 16) - a0
    src, sass = line_of.get(off, ("?", d["Source"].strip()))
    n = float(d["Instructions Executed"] or 0)
    inst[src] += n
    samp[src] += float(d["Warp Stall Sampling (All Samples)"] or 0)
    ops[src][sass.split()[0] if sass else "?"] += n
ti, ts = sum(inst.values()), sum(samp.values())
print(f"{fn}: {ti:.0f} warp instructions, {ts:.0f} stall samples")
for src, n in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    top_ops = ", ".join(f"{o}:{c/ max(n,1)*100:.0f}%" for o, c in ops[src].most_common(3))
    print(f"{n/ti*100:5.1f}% inst {samp[src]/ts*100:5.1f}% stall  {src:28s} {top_ops}")
