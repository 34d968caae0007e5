# Round-2 evidence at the current head: GPU suite, smoke, default bench (both arms), the
# bench's launch list (ncu durations), one multiply DRAM capture, config-5 full-solve
# launch list and the column gather's DRAM traffic
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rf_tests.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/rf_tests.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/rf_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/rf_bench.log > gpurun_out/rf_bench.json
tail -1 gpurun_out/rf_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline','e2e','same_n','gpu_launches','clocks']: print(k, json.dumps(d.get(k)))
for k,v in d.get('eigh',{}).items(): print(k, {x: v.get(x) for x in ('wall_s','wall_s_e2e','ratio_to_reference','glue_hbm')})
print('cpu', json.dumps(d.get('cpu_baseline')))"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rf_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/rf_ref.log | head -c 400; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:hsseig --csv \
  --log-file gpurun_out/rf_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/rf_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:tma_gemm --launch-skip 33 --launch-count 17 --csv --log-file gpurun_out/rf_mult.csv \
  python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu mult rc=$?"
export HSSEIG_NOPROF=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv --log-file gpurun_out/rf_cfg5.csv python tools/eigh_prof.py 5 65536 > gpurun_out/rf_cfg5_ncu.log 2>&1; echo "ncu cfg5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:"wave_gather_kernel|gen_panel_rows" --csv --log-file gpurun_out/rf_cfg5_gather.csv python tools/eigh_prof.py 5 65536 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:gen_panel_rows --launch-count 8 --csv --log-file gpurun_out/rf_genpanel.csv python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu genpanel rc=$?"
python tools/host_trace.py 5 65536 > gpurun_out/rf_cfg5_host.txt 2>&1; head -1 gpurun_out/rf_cfg5_host.txt
