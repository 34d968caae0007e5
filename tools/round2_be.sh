# the N > 1 bench path end to end with two gloo ranks on the one GPU (reduced N), after the round's solver changes
export PYTHONUNBUFFERED=1
HSSEIG_BENCH_N=16384 HSSEIG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/be_bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/be_bench2.log | head -c 3000; echo
