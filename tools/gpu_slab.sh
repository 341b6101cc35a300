mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload slab --steps 20 --warmup 10 > gpurun_out/bench_slab.json 2> gpurun_out/bench_slab.err; tail -3 gpurun_out/bench_slab.err; cut -c1-400 gpurun_out/bench_slab.json
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --solve-mode 6 > gpurun_out/bench_hero_m6.json 2> gpurun_out/bench_hero_m6.err; tail -2 gpurun_out/bench_hero_m6.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_solve_cluster' -s 5 -c 1 -o gpurun_out/full_cluster python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 --solve-mode 6 > gpurun_out/ncu_cluster.log 2>&1; tail -1 gpurun_out/ncu_cluster.log
python tools/ncu_summary.py gpurun_out/full_cluster.ncu-rep > gpurun_out/ncu_cluster_summary.txt 2>&1
