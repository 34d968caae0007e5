export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_t_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_t_tests.log | head -20
timeout 300 python -m pytest tests/test_distributed_cpu.py -q -p no:cacheprovider 2>&1 | tail -1
HSSEIG_NOPROF=1 timeout 600 python tools/eigh_prof.py 2 10000 2>&1 | head -1
HSSEIG_NOPROF=1 timeout 600 python tools/eigh_prof.py 3 20000 2>&1 | head -1
HSSEIG_NOPROF=1 timeout 600 python tools/eigh_prof.py 5 65536 2>&1 | head -1
HSSEIG_NOPROF=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rotate --csv --log-file gpurun_out/round2_t_rot.csv python tools/eigh_prof.py 3 20000 > /dev/null 2>&1; echo "ncu rc=$?"
