# dev loop on one GPU: build, a test subset ($TESTS), quick bench lines ($WLS)
mkdir -p gpurun_out
rm -f gpurun_out/q_*.json
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -m gpu -q -x ${PYARGS:-} 2>&1 | grep -v "^\.*$" | tail -${TAILN:-15}
fi
for w in ${WLS:-}; do
  timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --workload $w --no-cpu-baseline ${BENCHARGS:-} > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err; tail -2 gpurun_out/q_$w.err
done
python tools/quick_print.py
