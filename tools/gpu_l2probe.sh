# DRAM bytes per sweep (ncu, caches not flushed) vs bed size: does the sweep's set stay in L2?
mkdir -p gpurun_out/l2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 250000 500000 700000 1000000; do
  timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:'k_sweep' -s 45 -c 6 --csv python tools/l2_probe.py $n 8 > gpurun_out/l2/n$n.csv 2> gpurun_out/l2/n$n.err
  python - $n <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f'gpurun_out/l2/n{sys.argv[1]}.csv')))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]; mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value')
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) == len(hdr): agg[r[mi]].append(float(r[vi].replace(',', '')))
print(sys.argv[1], {k.split('__')[1][:16]: round(sum(v) / len(v), 1) for k, v in agg.items()})
PY
done
