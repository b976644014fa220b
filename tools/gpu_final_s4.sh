# Final session-4 verification on one B200: GPU parity suite, smoke, default
# bench line and the reference arm.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; echo "pytest exit $?" > gpurun_out/fin.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/fin.log
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench exit $?" >> gpurun_out/fin.log
timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref exit $?" >> gpurun_out/fin.log
