# GPU tests (E=1 regression after the env-segmented kernels), then ncu of k_narrow (1M) and the fused hero step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/phase_times.py hero50k > gpurun_out/phase_hero.txt 2>&1; tail -2 gpurun_out/phase_hero.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow' -s 3 -c 1 -o gpurun_out/full_narrow1m python bench.py --workload bed1m --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_narrow.log 2>&1; tail -1 gpurun_out/ncu_narrow.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_fused' -s 8 -c 1 -o gpurun_out/full_hero python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_hero.log 2>&1; tail -1 gpurun_out/ncu_hero.log
python tools/ncu_summary.py gpurun_out/full_narrow1m.ncu-rep gpurun_out/full_hero.ncu-rep > gpurun_out/ncu_full_summary2.txt 2>&1
