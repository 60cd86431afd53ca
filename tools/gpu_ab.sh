# A/B raster timing of library variants: AB_CFGS="lib.so:ENV=VAL,ENV2=VAL ..."
mkdir -p gpurun_out
run() { env $(echo $2 | tr ',' ' ') SLM_LIB=$PWD/$1 timeout 300 python bench.py --no-cpu-baseline --lm-steps 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', 'value', round(d['value'],1), 'raster', round(d['breakdown_ms']['raster'],4))"; }
for cfg in ${AB_CFGS:-"exp/w2.so:X=0"}; do run ${cfg%%:*} ${cfg#*:}; done
