# A/B of the default contact slots per particle (GG_MAX_CONTACTS) on bed1m and envs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for K in 16 4; do for w in bed1m envs; do
GG_MAX_CONTACTS=$K timeout 600 python bench.py --steps 60 --warmup 5 --workload $w --no-cpu-baseline --profile-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K=$K', '$w', round(d['ms_per_step'],4))"
done; done; done
