# A/B: bench each prebuilt library variant in build_variants/
mkdir -p gpurun_out
for lib in build_variants/*.so; do
  v=$(basename $lib .so)
  for w in ${WLS:-bed1m envs hero50k}; do
    GG_LIB=$PWD/$lib timeout 600 python bench.py --steps ${STEPS:-60} --warmup ${WARM:-5} --workload $w --no-cpu-baseline --profile-steps 3 --bed-state /tmp/bed1m_settled.npz > gpurun_out/v_${v}_$w.json 2> gpurun_out/v_${v}_$w.err || tail -3 gpurun_out/v_${v}_$w.err
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/v_*.json')):
    try:
        d=json.load(open(f)); r=d['roofline']
        print(f.split('/')[-1], '%.3e'%d['value'], round(d['ms_per_step'],4), r['kernel'], '%.3f'%r['frac'], {k:round(v,3) for k,v in r['kernel_time_share'].items() if v>0.02})
    except Exception as e: print(f, e)
PY
