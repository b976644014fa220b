# Round-2 final: GPU suite, smoke, bench line, reference arm + flow smoke, launch list, ncu captures
bash tools/gpu_suite.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -3 gpurun_out/bench.err
bash tools/gpu_evidence_r2b.sh > gpurun_out/evidence.log 2>&1
tail -5 gpurun_out/evidence.log
