# A/B of the TMA pass kernel builds in vlibs/ + parity of the k = 8 large-transform tests
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for l in vlibs/*.so; do timeout 300 python tools/time_variants.py $l >> gpurun_out/ab.txt 2>&1; done
cat gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or c2 or c4 or C4 or batch or sharded or fourstep or shapes or poly" > gpurun_out/pytest_tma.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_tma.log
