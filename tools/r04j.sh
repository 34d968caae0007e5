timeout 600 python tools/check_sample.py 32768 2>&1 | tail -2
timeout 600 python tools/check_sample.py 5000 2>&1 | tail -2
timeout 600 python tools/c4_ranks.py 2>&1 | tail -25
