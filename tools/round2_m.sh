export PYTHONUNBUFFERED=1
for r in 40 48 56 64 80; do echo "reserve $r"; HSSEIG_SPLIT_RESERVE=$r timeout 600 python tools/prof_merge.py 32768 6 2>&1 | tail -1; done
