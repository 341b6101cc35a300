mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_step_fused' -s 25 -c 1 -o gpurun_out/prof4_hero python bench.py --steps 5 --warmup 2 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu4.log
