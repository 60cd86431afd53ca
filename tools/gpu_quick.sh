# bench without the CPU baseline (quick GPU check)
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG:-q}_bench.json 2> gpurun_out/${TAG:-q}_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${TAG:-q}_bench.json'));print(d['value'],d['breakdown_ms'],d['lm']['ms_per_lm_step'],d['lm']['roofline']['frac'],d['time_to_psnr']['time_to_psnr_s'], d['e2e']['value'])"
grep "lm_step:" gpurun_out/${TAG:-q}_bench.err
