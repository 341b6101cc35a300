mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_solve' -s 4 -c 2 -o gpurun_out/prof3_1m python bench.py --steps 3 --warmup 1 --workload bed1m --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_solve' -s 10 -c 2 -o gpurun_out/prof3_hero python bench.py --steps 8 --warmup 2 --no-cpu-baseline --profile-steps 1 >> gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/ncu3.log
