timeout 600 python -m pytest tests/test_gpu_srrsc.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python tools/srrsc_c4.py 32768 check
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:srrsc --launch-skip 8 --launch-count 8 --csv --log-file gpurun_out/srrsc_lv.csv python tools/srrsc_c4.py 32768 > /dev/null 2>&1
