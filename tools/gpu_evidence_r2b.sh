# Round-2 evidence after the TMA pass kernel: multi-rank flow smoke, reference arm, launch list
# of the default bench command, ncu --set full of the C4 passes and the C2 pass launches
bash tools/gpu_flow.sh
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "launches exit $?"
python tools/ncu_summary.py launches gpurun_out/launches_bench.csv > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_ncu_r2b.sh > gpurun_out/ncu_r2b.log 2>&1
python tools/ncu_traffic.py /tmp/prof_r02b_c2_raw.csv > gpurun_out/ncu_traffic.log 2>&1 && cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
ls gpurun_out
