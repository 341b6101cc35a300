# hero50k A/B of build_variants/*.so: bench ms/step + fused-kernel phase times (contact sub-phases)
mkdir -p gpurun_out/hab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in build_variants/*.so; do v=$(basename $lib .so)
  GG_LIB=$PWD/$lib timeout 300 python bench.py --workload hero50k --steps 400 --warmup 20 --no-cpu-baseline --profile-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4))"
done; done
for lib in build_variants/*.so; do v=$(basename $lib .so)
  echo "== $v"; GG_LIB=$PWD/$lib timeout 300 python tools/phase_times.py hero50k 2>&1 | grep -v "^resort=False" | head -3
done
