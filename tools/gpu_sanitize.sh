# compute-sanitizer over every schedule (tools/sanitize.py) and the two-rank
# peer-memory slab step (tools/sanitize_slab_p2p.py) -> gpurun_out/san/
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.log | tail -2 | tr '\n' ' ')"
done
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --target-processes all --tool $tool --print-limit 20 python tools/sanitize_slab_p2p.py > gpurun_out/san/slab_p2p_$tool.log 2>&1
  echo "slab p2p $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok' gpurun_out/san/slab_p2p_$tool.log | tail -4 | tr '\n' ' ')"
done
