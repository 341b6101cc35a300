mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep|k_narrow' -s 30 -c 3 -o gpurun_out/prof_1m python bench.py --steps 4 --warmup 2 --workload bed1m --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu2.log 2>&1
tail -5 gpurun_out/ncu2.log
