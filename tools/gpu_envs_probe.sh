mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -k regex:'k_sweep|k_narrow|k_finish' -s 200 -c 40 --csv --log-file gpurun_out/envs_nocc.csv python bench.py --workload envs --steps 30 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -k regex:'k_sweep|k_narrow|k_finish' -s 200 -c 40 --csv --log-file gpurun_out/bed1m_nocc.csv python bench.py --workload bed1m --steps 30 --warmup 2 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
for f in ['gpurun_out/envs_nocc.csv','gpurun_out/bed1m_nocc.csv']:
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ui=hdr.index('Metric Unit'); idi=hdr.index('ID')
    d=collections.defaultdict(dict)
    for r in rows[1:]:
        d[(r[idi], r[ki].split('(')[0])][r[mi]]=(r[vi],r[ui])
    agg=collections.defaultdict(list)
    for (i,k),m in d.items(): agg[k].append(m)
    print(f)
    for k,ms in agg.items():
        t=[float(m['gpu__time_duration.sum'][0].replace(',','')) for m in ms]
        rd=[float(m['dram__bytes_read.sum'][0].replace(',','')) for m in ms]
        print(' ',k,len(ms),'avg time',sum(t)/len(t), ms[0]['gpu__time_duration.sum'][1], 'read', sum(rd)/len(rd), ms[0]['dram__bytes_read.sum'][1], 'L2hit', ms[0]['lts__t_sector_hit_rate.pct'][0])
PY
