# hero50k fused-kernel phase times + ncu full set of the bed1m sweep / commit kernels -> gpurun_out/hs/
mkdir -p gpurun_out/hs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/phase_times.py hero50k > gpurun_out/hs/phases_hero50k.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep_rm|k_commit|k_finish' -s 30 -c 12 -o gpurun_out/hs/full_sweep python bench.py --steps 6 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/hs/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/hs/full_sweep.ncu-rep > gpurun_out/hs/summary.txt 2>&1
ncu -i gpurun_out/hs/full_sweep.ncu-rep --page source --csv --print-source sass -k regex:k_sweep_rm > gpurun_out/hs/sass_sweep.csv 2>/dev/null
gzip -f gpurun_out/hs/sass_sweep.csv; rm -f gpurun_out/hs/full_sweep.ncu-rep
cat gpurun_out/hs/phases_hero50k.txt
