# quick perf check: 1M + envs bench lines (no cpu baseline) + per-kind breakdown
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in bed1m envs hero50k; do
timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --workload $w --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err; tail -2 gpurun_out/q_$w.err
done
python - <<'PY'
import json
for w in ['bed1m','envs','hero50k']:
    try:
        d=json.load(open(f'gpurun_out/q_{w}.json')); r=d['roofline']
        print(w, '%.3e'%d['value'], round(d['ms_per_step'],4), 'warm', d['config'].get('warm_ms_per_step'), 'e2e %.3e'%d['e2e']['value'], r['kernel'], '%.3f'%r['frac'], round(r['avg_launch_ms'],4), {k:round(v,3) for k,v in r['kernel_time_share'].items() if v>0.004})
    except Exception as e: print(w, e)
PY
