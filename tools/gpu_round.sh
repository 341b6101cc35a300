# one GPU session: smoke, gpu tests, bench (both workloads), launch lists, ncu full captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt
nproc > gpurun_out/nproc.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1000 --warmup 20 --cpu-seconds 10 > gpurun_out/bench_hero.json 2> gpurun_out/bench_hero.err; tail -2 gpurun_out/bench_hero.err
timeout 900 python bench.py --steps 100 --warmup 5 --workload bed1m --cpu-seconds 10 > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; tail -2 gpurun_out/bench_1m.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_hero.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_1m.csv python bench.py --workload bed1m --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_fused' -s 25 -c 1 -o gpurun_out/full_hero python bench.py --steps 5 --warmup 2 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_hero.log 2>&1; tail -2 gpurun_out/ncu_hero.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep|k_narrow|k_fill|k_count|k_bodies|k_finish' -s 40 -c 8 -o gpurun_out/full_1m python bench.py --workload bed1m --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_1m.log 2>&1; tail -2 gpurun_out/ncu_1m.log
python tools/launches.py gpurun_out/launches_hero.csv gpurun_out/launches_1m.csv > gpurun_out/launches_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_hero.ncu-rep gpurun_out/full_1m.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
cat gpurun_out/bench_hero.json gpurun_out/bench_1m.json gpurun_out/bench_ref.json | cut -c1-600
