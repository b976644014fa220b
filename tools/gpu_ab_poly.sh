# A/B of the builds in vlibs/ + the poly-multiply parity tests with the product library
bash tools/gpu_ab.sh
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_profile.py tests/test_cli.py -m gpu -x -q -k "poly or c1 or c2 or C2 or ragged or host or profile or tma or shapes or linearity or extreme" > gpurun_out/pytest_poly.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_poly.log
