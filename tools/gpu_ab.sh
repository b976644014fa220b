# A/B timing of the library builds in vlibs/ (tools/time_variants.py)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for l in vlibs/*.so; do timeout 300 python tools/time_variants.py $l >> gpurun_out/ab.txt 2>&1; done
cat gpurun_out/ab.txt
