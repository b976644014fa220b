# A/B of the builds in vlibs/ + the k = 16 / 32 parity tests with the product library
bash tools/gpu_ab.sh
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c5 or shapes or extreme or small_fft or linearity" > gpurun_out/pytest_k16.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_k16.log
