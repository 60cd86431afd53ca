# bench at the other BASELINE configs' shapes (1 GPU): configs[1], configs[3] (N sweep), configs[4]
for a in "--gaussians 100000 --views 64 --width 800 --height 800 --spt 64" \
         "--gaussians 500000 --views 64 --width 800 --height 800 --spt 32" \
         "--gaussians 500000 --views 64 --width 800 --height 800 --spt 128" \
         "--gaussians 3000000 --views 300 --width 1600 --height 1066 --spt 32"; do
  echo "== $a"
  timeout 600 python bench.py --no-cpu-baseline --no-psnr --lm-steps 2 --steps 10 $a 2>&1 | grep -E "^\{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('matvec/s', round(d['value'],1), 'frac', round(d['matvec_roofline']['frac'],3), 'raster', round(d['breakdown_ms']['raster'],3), 'lm it/s', round(d['lm']['lm_iters_per_s'],2), 'E', d['matvec_roofline']['E_v_sum'])"
done
