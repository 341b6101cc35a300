# the paper's loop-structure comparison (Fig. 6) on B200: PipelineMode x workload
mkdir -p gpurun_out/pipe
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f /tmp/bed1m_settled.npz
for w in hero50k bed1m; do for p in two-loops-split two-loops-fused one-loop; do
  timeout 600 python bench.py --workload $w --pipeline $p --steps 200 --warmup 10 --no-cpu-baseline --profile-steps 3 > gpurun_out/pipe/${w}_$p.json 2> gpurun_out/pipe/${w}_$p.err || tail -2 gpurun_out/pipe/${w}_$p.err
done; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/pipe/*.json')):
    try:
        d=json.load(open(f)); print(f.split('/')[-1], '%.3e'%d['value'], round(d['ms_per_step'],4))
    except Exception as e: print(f, e)
PY
