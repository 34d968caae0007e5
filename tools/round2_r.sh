export PYTHONUNBUFFERED=1
for r in 2 4 6 8; do echo "LW_R $r"; HSSEIG_LW_R=$r timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1; done
timeout 300 python tools/sec_bench.py 2>&1 | tail -1
