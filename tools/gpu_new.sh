# new GPU tests of this session + the checked-build run (evidence file)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_checked_build.py tests/test_refbridge.py tests/test_gpu_profile.py -m gpu -q -k "staged or mul_host or odd_offsets or checked or refbridge or reference_bench or profile or pass_times" > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_new.log
GFPFFT_LIB=$PWD/paper_1811_01490_b200/libgfpfft_checked.so timeout 900 python tools/checked_cases.py > gpurun_out/checked_cases.txt 2>&1; echo "checked exit $?"
grep -c GFP_CHECK gpurun_out/checked_cases.txt; tail -3 gpurun_out/checked_cases.txt
