# source/SASS-level profile of one k_sweep and one k_narrow launch (bed1m, settled state cached in /tmp)

mkdir -p gpurun_out/src
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WL=${WL:-bed1m}

timeout 600 python bench.py --workload $WL --steps 200 --warmup 50 --no-cpu-baseline > gpurun_out/src/bench.json 2> gpurun_out/src/bench.err
for m in ${MODES:-}; do
  timeout 600 python bench.py --workload $WL --steps 200 --warmup 50 --no-cpu-baseline --solve-mode $m > gpurun_out/src/bench_mode$m.json 2>> gpurun_out/src/bench.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRX:-k_narrow|k_sweep}" -s ${SKIP:-120} -c ${CNT:-2} -o gpurun_out/src/$WL python bench.py --workload $WL --steps 20 --warmup 5 --no-cpu-baseline --profile-steps 1 > gpurun_out/src/run.log 2>&1
for k in ${KS:-k_sweep k_narrow}; do
  ncu -i gpurun_out/src/$WL.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/src/sass_${WL}_$k.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/src/$WL.ncu-rep > gpurun_out/src/summary.txt 2>&1
gzip -f gpurun_out/src/*.csv
rm -f gpurun_out/src/*.ncu-rep
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/src/bench*.json')):
    try:
        d = json.load(open(f)); r = d['roofline']
        print(f.split('/')[-1], '%.3e' % d['value'], round(d['ms_per_step'], 4), r['kernel'], '%.3f' % r['frac'],
              {k: round(v, 3) for k, v in r['kernel_time_share'].items() if v > 0.02})
    except Exception as e:
        print(f, e)
PY
