# A/B timing of the library builds in vlibs/ (tools/time_variants.py)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
python tools/time_variants.py vlibs/*.so > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
