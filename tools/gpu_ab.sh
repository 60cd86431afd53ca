# A/B raster timing of library variants exp/*.so with optional smem pads
mkdir -p gpurun_out
run() { SLM_RASTER_PAD=$2 SLM_LIB=$PWD/$1 timeout 300 python bench.py --no-cpu-baseline --lm-steps 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 pad $2', 'value', round(d['value'],1), 'raster', round(d['breakdown_ms']['raster'],4))"; }
for cfg in ${AB_CFGS:-"exp/vA.so:0"}; do run ${cfg%%:*} ${cfg##*:}; done
