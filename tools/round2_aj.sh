export PYTHONUNBUFFERED=1
for ns in 8 16 32; do echo "streams $ns"; HSSEIG_HSS_STREAMS=$ns timeout 600 python tools/adc1_bench.py 2>&1 | head -2 | cut -c1-60; done
for ns in 8 32; do HSSEIG_HSS_STREAMS=$ns timeout 600 python tools/eigh_bench.py 3 2>&1 | tail -1 | cut -c1-80; done
