# panel chunks >= 1 on a narrow grid (co-resident with the DMMA CTAs): sweep of the block count
export PYTHONUNBUFFERED=1
for n in 0 148 222 296 370 592; do
  echo "== HSSEIG_PANEL_NARROW=$n"
  HSSEIG_PANEL_NARROW=$n timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-eigh 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['phases_ms']))"
done
