# bench at the other BASELINE configs' shapes (1 GPU): configs[1], configs[4], and the configs[3]
# sampling sweep (tools/spt_sweep.py); full JSON lines into gpurun_out/
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for a in "configs[1]|--gaussians 100000 --views 64 --width 800 --height 800 --spt 64" \
         "configs[4]|--gaussians 3000000 --views 300 --width 1600 --height 1066 --spt 32"; do
  name=${a%%|*}; args=${a#*|}
  echo "== $name $args"
  timeout 900 python bench.py --no-cpu-baseline --no-psnr --lm-steps 3 --steps 10 $args 2> gpurun_out/configs_err.log | grep -E "^\{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['config']['workload']='$name: '+'$args'; print(json.dumps(d))" | tee -a gpurun_out/configs.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('matvec/s', round(d['value'],1), 'frac', round(d['matvec_roofline']['frac'],3), 'raster', round(d['breakdown_ms']['raster'],3), 'lm it/s', round(d['lm']['lm_iters_per_s'],2))"
done
timeout 1500 python tools/spt_sweep.py > gpurun_out/spt_sweep.jsonl 2> gpurun_out/spt_err.log; tail -5 gpurun_out/spt_sweep.jsonl | cut -c1-300
