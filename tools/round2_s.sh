# where the full solves spend time: host profile + device kernel list (configs 2 ADC2, 3)
export PYTHONUNBUFFERED=1
timeout 600 python tools/eigh_prof.py 2 10000 > gpurun_out/round2_s_prof2.log 2>&1; head -45 gpurun_out/round2_s_prof2.log
timeout 600 python tools/eigh_prof.py 3 20000 > gpurun_out/round2_s_prof3.log 2>&1; head -45 gpurun_out/round2_s_prof3.log
HSSEIG_NOPROF=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2_s_ncu2.csv python tools/eigh_prof.py 2 10000 > /dev/null 2>&1; echo "ncu rc=$?"
HSSEIG_NOPROF=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2_s_ncu3.csv python tools/eigh_prof.py 3 20000 > /dev/null 2>&1; echo "ncu rc=$?"
