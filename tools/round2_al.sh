export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_al_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_al_tests.log | head
for r in 32 40 48; do echo "reserve $r"; HSSEIG_SPLIT_RESERVE=$r timeout 600 python tools/prof_merge.py 32768 5 2>&1 | tail -1; done
HSSEIG_NVCC_EXTRA=-DHSSEIG_ID_TIMING timeout 600 python -c "from paper_1510_04591_b200 import build as b; b.build(force=True)" 2>&1 | tail -2
timeout 300 python tools/id_timing.py 2>&1 | tail -7
