mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python tools/dbg_modes.py 2>&1 | grep -v "dx 0.0 dv 0.0 contacts True" | tail -5
for m in 0 4 7; do timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --solve-mode $m > gpurun_out/hero_m$m.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/hero_m$m.json')); print('mode $m', d['ms_per_step'], d['value'])"; done
python tools/phase_times.py hero50k 2>/dev/null
