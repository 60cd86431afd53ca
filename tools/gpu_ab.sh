# A/B product timing of library variants: AB_CFGS="lib.so:ENV=VAL,ENV2=VAL ..."
mkdir -p gpurun_out
run() { env $(echo $2 | tr ',' ' ') SLM_LIB=$PWD/$1 timeout 300 python bench.py --no-cpu-baseline --no-psnr --lm-steps ${LM:-0} --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('$1 $2', 'value', round(d['value'],1), 'tan', round(b['tangents'],4), 'raster', round(b['raster'],4), 'chain', round(b['chain'],4), 'lm', d['lm'] and round(d['lm']['ms_per_lm_step'],2))"; }
for cfg in ${AB_CFGS:-"exp/w2.so:X=0"}; do run ${cfg%%:*} ${cfg#*:}; done
