# one build -> test -> bench -> launch-list iteration on the GPU box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 1000 --warmup 20 --cpu-seconds 5 > gpurun_out/bench_hero.json 2> gpurun_out/bench_hero.err; tail -3 gpurun_out/bench_hero.err; cat gpurun_out/bench_hero.json
timeout 600 python bench.py --steps 200 --warmup 10 --workload bed1m --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; tail -3 gpurun_out/bench_1m.err; cat gpurun_out/bench_1m.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 300 -c 60 --csv --log-file gpurun_out/launches_hero.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 100 -c 40 --csv --log-file gpurun_out/launches_1m.csv python bench.py --steps 10 --warmup 2 --workload bed1m --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
echo done
