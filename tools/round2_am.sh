export PYTHONUNBUFFERED=1
timeout 600 python tools/eigh_prof.py 5 65536 2>&1 | head -40
HSSEIG_NOPROF=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2_am_ncu5.csv python tools/eigh_prof.py 5 65536 > /dev/null 2>&1; echo "ncu rc=$?"
