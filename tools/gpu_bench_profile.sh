# Launch list of the default bench command and an ncu --set full capture of
# the eight pass launches of one C2 poly-multiply (tools/run_case.py c2,
# second repetition), reduced to CSV on the box.
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "launches exit $?"
timeout 300 python tools/run_case.py c2 2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_pass -s 8 -c 8 \
    -o /tmp/prof_c2 python tools/run_case.py c2 2 > gpurun_out/ncu_c2.log 2>&1
echo "c2 exit $?"
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2_raw.csv 2>/dev/null
ncu -i /tmp/prof_c2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_c2_src.csv 2>/dev/null
