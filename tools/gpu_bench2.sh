# raster timing only, twice (variance check)
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --lm-steps 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'raster', round(d['breakdown_ms']['raster'],4), 'tan', round(d['breakdown_ms']['tangents'],4), 'chain', round(d['breakdown_ms']['chain'],4))"
done
