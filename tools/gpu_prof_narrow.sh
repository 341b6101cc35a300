# ncu of the large-n contact kernel on bed1m: launch list, full set and the
# SASS source page of k_narrow -> gpurun_out/pn/ (attribute the SASS to
# source lines with tools/sass_lines.py and nvdisasm of the same build)
mkdir -p gpurun_out/pn
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_narrow' -c 20 --csv --log-file gpurun_out/pn/launch.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow' -s 6 -c 1 -o gpurun_out/pn/full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/pn/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/pn/full.ncu-rep > gpurun_out/pn/summary.txt 2>&1
ncu -i gpurun_out/pn/full.ncu-rep --page source --csv --print-source sass -k regex:k_narrow > gpurun_out/pn/sass_narrow.csv 2>/dev/null
gzip -f gpurun_out/pn/sass_narrow.csv
rm -f gpurun_out/pn/full.ncu-rep
python tools/launches.py gpurun_out/pn/launch.csv
