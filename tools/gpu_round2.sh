# Round-2 evidence on one GPU: smoke, all GPU tests, bench lines (bed1m =
# default, hero50k, envs, slab, reference arm), ncu launch lists and full-set
# captures of the top kernels, summaries.  Output: gpurun_out/r2/
set -u
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/nvsmi.txt
nproc > $O/nproc.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 10 > $O/bench_bed1m.json 2> $O/bench_bed1m.err; tail -1 $O/bench_bed1m.err
timeout 900 python bench.py --workload hero50k --steps 1000 --warmup 20 > $O/bench_hero50k.json 2> $O/bench_hero50k.err; tail -1 $O/bench_hero50k.err
timeout 900 python bench.py --workload envs --steps 200 --warmup 5 > $O/bench_envs.json 2> $O/bench_envs.err; tail -1 $O/bench_envs.err
timeout 900 python bench.py --workload slab --steps 20 --warmup 3 > $O/bench_slab.json 2> $O/bench_slab.err; tail -1 $O/bench_slab.err
timeout 900 python bench.py --workload bed1m --solve-mode 8 --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_bed1m_mode8.json 2> $O/bench_bed1m_mode8.err; tail -1 $O/bench_bed1m_mode8.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err; tail -1 $O/bench_reference.err
# launch lists (cold cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bed1m.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_hero50k.csv python bench.py --workload hero50k --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_envs.csv python bench.py --workload envs --steps 10 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
python tools/launches.py $O/launches_bed1m.csv $O/launches_hero50k.csv $O/launches_envs.csv > $O/launches_summary.txt 2>&1
# full-set captures of the top kernels
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_sweep|k_finish|k_commit|k_fill|k_count|k_scatter|k_scan' -s 60 -c 18 -o $O/full_bed1m python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-steps 1 > $O/ncu_bed1m.log 2>&1; tail -1 $O/ncu_bed1m.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_fused' -s 3 -c 1 -o $O/full_hero50k python bench.py --workload hero50k --steps 5 --warmup 2 --no-cpu-baseline --profile-steps 1 > $O/ncu_hero.log 2>&1; tail -1 $O/ncu_hero.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_solve_staged' -s 3 -c 1 -o $O/full_bed1m_staged python bench.py --solve-mode 8 --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > $O/ncu_staged.log 2>&1; tail -1 $O/ncu_staged.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_sweep|k_finish' -s 30 -c 12 -o $O/full_envs python bench.py --workload envs --steps 10 --warmup 2 --no-cpu-baseline --profile-steps 1 > $O/ncu_envs.log 2>&1; tail -1 $O/ncu_envs.log
python tools/ncu_summary.py $O/full_bed1m.ncu-rep $O/full_hero50k.ncu-rep $O/full_bed1m_staged.ncu-rep $O/full_envs.ncu-rep > $O/ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py $O/ncu_summary.json bed1m=$O/full_bed1m.ncu-rep hero50k=$O/full_hero50k.ncu-rep envs=$O/full_envs.ncu-rep > /dev/null 2>&1
for k in k_narrow k_sweep; do
  ncu -i $O/full_bed1m.ncu-rep --page source --csv --print-source sass -k regex:$k > $O/sass_bed1m_$k.csv 2>/dev/null
done
gzip -f $O/sass_*.csv
rm -f $O/*.ncu-rep
python tools/summarize_profiles.py $O > /dev/null 2>&1
cat $O/launches_summary.txt | head -40
