# Session-4 round-end pass on one B200: GPU parity suite, smoke, default
# bench line, reference arm, the ncu launch list of the default bench command,
# ncu --set full of the C2 passes (traffic) and of the sharded-C4 exchange
# kernels (fused XCH last pass + standalone k_exchange).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu1 exit $?"
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_prof.sh c2 8 8 c2 k_pass 786432
python tools/ncu_traffic.py /tmp/prof_c2_raw.csv > gpurun_out/traffic_c2.txt 2>&1
timeout 300 python tools/run_case.py c4s 2 > gpurun_out/plain_c4s.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:true>|k_exchange' -c 3 -o /tmp/prof_c4s python tools/run_case.py c4s 2 > gpurun_out/ncu_c4s.log 2>&1
echo "ncu c4s exit $?"
ncu -i /tmp/prof_c4s.ncu-rep --page raw --csv > /tmp/prof_c4s_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/prof_c4s_raw.csv > gpurun_out/prof_c4s_metrics.txt 2>&1
cp /tmp/prof_c2_raw.csv /tmp/prof_c4s_raw.csv gpurun_out/ 2>/dev/null; echo round2 done
