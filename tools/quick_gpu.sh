timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for kb in 32 64; do timeout 300 python bench.py --key-bits $kb --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"u$kb\", round(d[\"value\"]/1e9,3), round(d[\"ms_per_step\"],3)); [print(k[\"kernel\"], round(k[\"avg_ms\"],3)) for k in d[\"kernels\"][:10]]"; done
timeout 300 python bench.py --k 16 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 | tail -1 | cut -c1-200
