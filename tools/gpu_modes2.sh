mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x -k "modes or determinism or single_step or physical" 2>&1 | tail -2
for m in 0 5 1 3; do
  timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --solve-mode $m --profile-steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', d['ms_per_step'], d['config']['warm_ms_per_step'], d['roofline']['avg_launch_ms'])"
done
