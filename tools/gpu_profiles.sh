# round profiles: bench lines, launch lists, ncu --set full of the top kernels
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/prof/bench_hero50k.json 2> gpurun_out/prof/bench_hero50k.err; tail -1 gpurun_out/prof/bench_hero50k.err
timeout 900 python bench.py --workload bed1m --steps 200 --warmup 10 > gpurun_out/prof/bench_bed1m.json 2> gpurun_out/prof/bench_bed1m.err; tail -1 gpurun_out/prof/bench_bed1m.err
timeout 900 python bench.py --workload envs --steps 200 --warmup 5 > gpurun_out/prof/bench_envs.json 2> gpurun_out/prof/bench_envs.err; tail -1 gpurun_out/prof/bench_envs.err
timeout 900 python bench.py --workload slab --steps 30 --warmup 20 > gpurun_out/prof/bench_slab.json 2> gpurun_out/prof/bench_slab.err; tail -1 gpurun_out/prof/bench_slab.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/prof/bench_reference.json 2> gpurun_out/prof/bench_reference.err
# launch lists (the recipe's pass): per-launch duration, cold cache, serialised
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/prof/launches_hero50k.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_bed1m.csv python bench.py --workload bed1m --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 300 --csv --log-file gpurun_out/prof/launches_envs.csv python bench.py --workload envs --steps 20 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
# full sets of the top kernels (one launch each, after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_fused' -s 40 -c 1 -o gpurun_out/prof/full_hero50k python bench.py --steps 60 --warmup 5 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_sweep|k_finish|k_fill|k_count|k_scatter' -s 240 -c 16 -o gpurun_out/prof/full_bed1m python bench.py --workload bed1m --steps 40 --warmup 10 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_sweep|k_finish' -s 1300 -c 12 -o gpurun_out/prof/full_envs python bench.py --workload envs --steps 20 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/prof/launches_*.csv > gpurun_out/prof/launches_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof/full_*.ncu-rep > gpurun_out/prof/ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py gpurun_out/prof/ncu_summary.json hero50k=gpurun_out/prof/full_hero50k.ncu-rep bed1m=gpurun_out/prof/full_bed1m.ncu-rep envs=gpurun_out/prof/full_envs.ncu-rep > /dev/null 2>&1
# source-level exports (per-line stalls / instructions) instead of the big .ncu-rep files
ncu -i gpurun_out/prof/full_hero50k.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof/src_hero50k_fused.csv 2>/dev/null
ncu -i gpurun_out/prof/full_bed1m.ncu-rep --page source --csv --print-source cuda -k regex:k_narrow > gpurun_out/prof/src_bed1m_narrow.csv 2>/dev/null
gzip -f gpurun_out/prof/src_*.csv
rm -f gpurun_out/prof/*.ncu-rep
ls -la gpurun_out/prof
