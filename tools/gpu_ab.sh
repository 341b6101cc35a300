# interleaved A/B of build_variants/*.so: R rounds x workloads, one line per run
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq 1 ${R:-2}); do
  for lib in build_variants/*.so; do
    v=$(basename $lib .so)
    for w in ${WLS:-bed1m envs}; do
      GG_LIB=$PWD/$lib timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --workload $w --no-cpu-baseline --profile-steps 3 > gpurun_out/ab/${v}_${w}_$r.json 2> gpurun_out/ab/${v}_${w}_$r.err || tail -3 gpurun_out/ab/${v}_${w}_$r.err
    done
  done
done
python - <<'PY'
import json, glob, collections
res = collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/ab/*.json')):
    try:
        d = json.load(open(f)); v, w, r = f.split('/')[-1][:-5].rsplit('_', 2)
        sh = d['roofline']['kernel_time_share']
        res[(w, v)].append((d['ms_per_step'], {k: round(x * d['ms_per_step'], 4) for k, x in sh.items() if x > 0.02}))
    except Exception as e: print(f, e)
for (w, v), runs in sorted(res.items()):
    print(w, v, [round(m, 4) for m, _ in runs], runs[-1][1])
PY
