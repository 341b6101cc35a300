mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/phase_times.py hero50k 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv --log-file gpurun_out/lt_fused.csv python tools/phase_times.py hero50k 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:'k_' --csv --log-file gpurun_out/lt_fused_nocc.csv python tools/phase_times.py hero50k 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 100 -c 60 --csv --log-file gpurun_out/lt_mode3.csv python bench.py --steps 10 --warmup 2 --no-cpu-baseline --profile-steps 1 --solve-mode 3 > /dev/null 2>&1
python tools/launches.py gpurun_out/lt_fused.csv gpurun_out/lt_fused_nocc.csv gpurun_out/lt_mode3.csv
