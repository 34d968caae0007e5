export PYTHONUNBUFFERED=1
for n in 0 1036 2072 8192 32768; do
  echo "== NARROW=$n"
  HSSEIG_PANEL_NARROW=$n timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-eigh 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms']['sample'])"
done
