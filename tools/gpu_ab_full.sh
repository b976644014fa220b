# A/B of the builds in vlibs/, then the whole GPU suite + smoke + bench with the product library
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for l in vlibs/*.so; do timeout 300 python tools/time_variants.py $l >> gpurun_out/ab.txt 2>&1; done
cat gpurun_out/ab.txt
bash tools/gpu_suite.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -3 gpurun_out/bench.err
