# configs[0] time-to-PSNR per library / env: AB_CFGS="lib.so:ENV=V ..."
for rep in 1 2; do for cfg in $AB_CFGS; do
  env $(echo ${cfg#*:} | tr ',' ' ') SLM_LIB=$PWD/${cfg%%:*} timeout 300 python bench.py --steps 3 --warmup 3 --lm-steps 0 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['time_to_psnr']; print('$cfg', 'time_to_psnr_s', round(p['time_to_psnr_s'],4), 'value', round(d['value'],1))"
done; done
