set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --steps 300 --warmup 10 --workload bed1m --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; tail -2 gpurun_out/bench_1m.err; cat gpurun_out/bench_1m.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 400 -c 120 --csv --log-file gpurun_out/launches_hero.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 200 -c 60 --csv --log-file gpurun_out/launches_1m.csv python bench.py --steps 10 --warmup 2 --workload bed1m --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
ls -la gpurun_out
