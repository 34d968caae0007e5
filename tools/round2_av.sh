export PYTHONUNBUFFERED=1
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print({k: round(v.get('wall_s'),4) for k,v in d.get('eigh',{}).items()})"
done
python tools/host_trace.py 3 20000
