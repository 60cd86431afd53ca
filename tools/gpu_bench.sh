# full default bench (both arms) as the driver runs it
set -x
timeout 900 python bench.py > gpurun_out/${TAG:-r2}_bench.json 2> gpurun_out/${TAG:-r2}_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/${TAG:-r2}_bench.err
if [ -n "$REF" ]; then timeout 1750 python bench.py --impl reference > gpurun_out/${TAG:-r2}_bench_ref.json 2> gpurun_out/${TAG:-r2}_bench_ref.err; echo "ref rc=$?"; fi
