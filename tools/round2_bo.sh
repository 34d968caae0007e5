# ncu --set full of the top-level column gather of a config-5 solve and of one panel-generator chunk
export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave_gather_kernel --launch-skip 23 --launch-count 1 -o gpurun_out/bo_gather -f python tools/eigh_prof.py 5 65536 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_panel_rows --launch-skip 5 --launch-count 1 -o gpurun_out/bo_genpanel -f python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu genpanel rc=$?"
python tools/ncu_keys.py gpurun_out/bo_gather.ncu-rep > gpurun_out/bo_gather_keys.csv
python tools/ncu_keys.py gpurun_out/bo_genpanel.ncu-rep > gpurun_out/bo_genpanel_keys.csv
for f in bo_gather bo_genpanel; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h,u,r=rows[0],rows[1],rows[2]
for k in ('dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','launch__occupancy_limit_registers','launch__registers_per_thread','dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum'):
    if k in h: print('$f', k, r[h.index(k)], u[h.index(k)])
"
done
ls -la gpurun_out/bo_*.ncu-rep
