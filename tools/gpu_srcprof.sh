# source/SASS-level profile of one k_sweep and one k_narrow launch (bed1m)
mkdir -p gpurun_out/src
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WL=${WL:-bed1m}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_narrow|k_sweep' -s ${SKIP:-120} -c 2 -o gpurun_out/src/$WL python bench.py --workload $WL --steps 20 --warmup 5 --no-cpu-baseline --profile-steps 1 > gpurun_out/src/run.log 2>&1
for k in k_sweep k_narrow; do
  ncu -i gpurun_out/src/$WL.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/src/sass_${WL}_$k.csv 2>/dev/null
  ncu -i gpurun_out/src/$WL.ncu-rep --page source --csv --print-source cuda -k regex:$k > gpurun_out/src/cuda_${WL}_$k.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/src/$WL.ncu-rep > gpurun_out/src/summary.txt 2>&1
gzip -f gpurun_out/src/*.csv
rm -f gpurun_out/src/*.ncu-rep
ls -la gpurun_out/src
