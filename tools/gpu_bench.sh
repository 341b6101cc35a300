# bench lines for all workloads + launch list per workload
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 1000 --warmup 20 --cpu-seconds 5 > gpurun_out/bench_hero.json 2> gpurun_out/bench_hero.err; tail -2 gpurun_out/bench_hero.err
timeout 900 python bench.py --steps 100 --warmup 5 --workload bed1m --cpu-seconds 5 > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; tail -2 gpurun_out/bench_1m.err
timeout 900 python bench.py --steps 200 --warmup 5 --workload envs --cpu-seconds 5 > gpurun_out/bench_envs.json 2> gpurun_out/bench_envs.err; tail -2 gpurun_out/bench_envs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_1m.csv python bench.py --workload bed1m --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_envs.csv python bench.py --workload envs --steps 10 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow' -s 3 -c 1 -o gpurun_out/full_narrow1m python bench.py --workload bed1m --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_narrow.log 2>&1; tail -1 gpurun_out/ncu_narrow.log
python tools/launches.py gpurun_out/launches_1m.csv gpurun_out/launches_envs.csv > gpurun_out/launches_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_narrow1m.ncu-rep > gpurun_out/ncu_narrow_summary.txt 2>&1
python - <<'PY'
import json
for f in ['gpurun_out/bench_hero.json','gpurun_out/bench_1m.json','gpurun_out/bench_envs.json']:
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f, '%.3e'%d['value'], round(d['ms_per_step'],4), 'e2e %.3e'%d['e2e']['value'], r['kernel'], '%.3f'%r['frac'], 'step_frac %.3f'%r['step_frac'], {k:round(v,3) for k,v in r['kernel_time_share'].items() if v>0.004})
    except Exception as e: print(f, e)
PY
cat gpurun_out/launches_summary.txt
