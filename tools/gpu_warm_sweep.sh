# ncu of the sweep kernels WITHOUT cache flushing (--cache-control none): the
# DRAM traffic of a sweep inside a step (records and w warm in L2 or not)
mkdir -p gpurun_out/ws
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:'k_sweep_rm|k_narrow|k_finish' -s 40 -c 13 --csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ws/warm.csv 2> gpurun_out/ws/warm.err
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/ws/warm.csv')))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]; ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value'); ii = hdr.index('ID')
cur = {}
for r in rows[hi + 1:]:
    if len(r) != len(hdr): continue
    cur.setdefault((r[ii], r[ki][:14]), {})[r[mi]] = r[vi]
for (i, k), m in cur.items():
    print(i, k, {a.split('__')[1][:18]: b for a, b in m.items()})
PY
