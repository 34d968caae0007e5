export PYTHONUNBUFFERED=1
timeout 300 python tools/srrsc_prof.py 32768 128 2 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:srrsc --csv --log-file gpurun_out/round2_ai_levels.csv python tools/srrsc_prof.py 32768 128 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srrsc --launch-skip 0 --launch-count 1 -o gpurun_out/round2_srrsc_leaf python tools/srrsc_prof.py 32768 128 1 > /dev/null 2>&1; echo "ncu full rc=$?"
