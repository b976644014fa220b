# GPU suite, smoke, default bench line on one B200 (outputs under gpurun_out/)
bash tools/gpu_suite.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -3 gpurun_out/bench.err
