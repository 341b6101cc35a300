# the whole -m gpu suite under compute-sanitizer memcheck (every kernel every
# test launches) -> gpurun_out/san/memcheck_tests.log
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 3300 compute-sanitizer --tool memcheck --print-limit 20 --target-processes all python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/san/memcheck_tests.log 2>&1
echo "rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/memcheck_tests.log | tail -5
