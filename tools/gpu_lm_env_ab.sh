# LM-step A/B by env: AB_CFGS="lib.so:ENV=V,..." -> per-stage timings of tools/lm_steps.py
for rep in 1 2; do for cfg in $AB_CFGS; do
  echo "== $cfg"; env $(echo ${cfg#*:} | tr ',' ' ') SLM_LIB=$PWD/${cfg%%:*} timeout 300 python tools/lm_steps.py 4 2>&1 | tail -1 | cut -c1-330
done; done
