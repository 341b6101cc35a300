# ncu of the contact kernels on bed1m: launch list + full set + SASS of k_narrow_tiled -> gpurun_out/pt/
mkdir -p gpurun_out/pt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_narrow' -c 20 --csv --log-file gpurun_out/pt/launch.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow' -s 6 -c 2 -o gpurun_out/pt/full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/pt/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/pt/full.ncu-rep > gpurun_out/pt/summary.txt 2>&1
ncu -i gpurun_out/pt/full.ncu-rep --page source --csv --print-source sass -k regex:k_narrow_tiled > gpurun_out/pt/sass_tiled.csv 2>/dev/null
gzip -f gpurun_out/pt/sass_tiled.csv
rm -f gpurun_out/pt/full.ncu-rep
python tools/launches.py gpurun_out/pt/launch.csv
