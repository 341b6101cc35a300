mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/phase_times.py hero50k 2>&1 | tail -3
timeout 600 python bench.py --steps 1000 --warmup 20 --cpu-seconds 5 > gpurun_out/bench_hero.json 2> gpurun_out/bench_hero.err; tail -3 gpurun_out/bench_hero.err
timeout 600 python bench.py --steps 200 --warmup 10 --workload bed1m --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; tail -3 gpurun_out/bench_1m.err
python - <<'PY'
import json
for f in ['gpurun_out/bench_hero.json','gpurun_out/bench_1m.json']:
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f, '%.3e'%d['value'], round(d['ms_per_step'],4), 'warm', round(d['config']['warm_ms_per_step'],4), 'e2e %.3e'%d['e2e']['value'], r['kernel'], '%.3f'%r['frac'], 'step_frac %.3f'%r['step_frac'], {k:round(v,3) for k,v in r['kernel_time_share'].items() if v>0.004})
    except Exception as e: print(f, e)
PY
