export PYTHONUNBUFFERED=1
for i in 1 2 3 4; do timeout 300 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/round2_y_mr$i.log 2>&1; echo "multirank $i rc=$?"; grep -E "passed|failed|SIGSEGV" gpurun_out/round2_y_mr$i.log | tail -1; done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/round2_y_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/round2_y_tests.log | head
HSSEIG_BENCH_N=16384 HSSEIG_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/round2_y_bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/round2_y_bench2.log | head -c 1500; echo
