export PYTHONUNBUFFERED=1 HSSEIG_NOPROF=1
python tools/eigh_prof.py 5 65536 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv --log-file gpurun_out/aq_cfg5.csv python tools/eigh_prof.py 5 65536 > gpurun_out/aq_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_table.py gpurun_out/aq_cfg5.csv | head -30
python tools/wave_prof.py 5 65536 2>&1 | head -45
