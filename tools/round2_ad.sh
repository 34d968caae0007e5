export PYTHONUNBUFFERED=1
for v in 0 1 2 3 4 5; do HSSEIG_SEC_VARIANT=$v timeout 300 python tools/sec_bench.py 2>&1 | tail -1; done
