# the N > 1 bench path on one GPU: two gloo ranks sharing the device (host-side collectives)
export PYTHONUNBUFFERED=1
HSSEIG_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 --steps 3 --warmup 3 --n 16384 > gpurun_out/round2_f_bench2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/round2_f_bench2.log | head -c 3000; echo
