# GPU suite + config-4 bench + multiply per-level launch times + the N > 1 bench path (gloo, 2 ranks on one GPU)
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_g_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_g_tests.log | head -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-eigh > gpurun_out/round2_g_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/round2_g_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','ms_per_step','phases_ms','roofline']: print(k, json.dumps(d.get(k)))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:tma_gemm --launch-skip 33 --launch-count 17 --csv \
  --log-file gpurun_out/round2_g_mult.csv python tools/prof_merge.py 32768 2 > /dev/null 2>&1; echo "ncu rc=$?"
HSSEIG_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 3 --warmup 3 --n 16384 > gpurun_out/round2_g_bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/round2_g_bench2.log | head -c 4000; echo
