timeout 900 python tools/orth_bisect.py kac > gpurun_out/r04_bis_kac.log 2>&1; echo "kac rc=$?"; cat gpurun_out/r04_bis_kac.log | tail -12
timeout 1200 python tools/orth_bisect.py c4 8192 > gpurun_out/r04_bis_c4.log 2>&1; echo "c4 rc=$?"; cat gpurun_out/r04_bis_c4.log | tail -12
