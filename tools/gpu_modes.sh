mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for m in 1 2 3; do
  timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --solve-mode $m --profile-steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', d['ms_per_step'], d['config']['warm_ms_per_step'])"
done
for r in 1 8 10000; do
  timeout 300 python bench.py --steps 300 --warmup 10 --workload bed1m --no-cpu-baseline --resort-every $r --profile-steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1m resort $r', d['ms_per_step'], d['config']['warm_ms_per_step'])"
done
