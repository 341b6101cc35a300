# A/B of the physical re-sort period on bed1m and hero50k (bench --resort-every)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for w in bed1m hero50k; do for re in 4 8 16 32; do
  st=200; [ $w = hero50k ] && st=800
  timeout 600 python bench.py --workload $w --steps $st --warmup 10 --no-cpu-baseline --resort-every $re --profile-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', 'resort_every=$re', round(d['ms_per_step'],4))"
done; done; done
