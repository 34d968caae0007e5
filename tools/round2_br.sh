export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/br.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/br.txt
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-eigh 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms']['sample'], d['phases_ms']['total'])"; done
timeout 300 python tools/stress_det.py 2>&1 | tail -3
