# Round-2 ncu evidence: launch list of the default bench command, --set full
# of the C2 pass launches, the C4 passes and the C3 passes (8 transforms).
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "launches exit $?"
python tools/ncu_summary.py launches gpurun_out/launches_bench.csv > gpurun_out/launches_summary.txt 2>&1
prof() {  # tag case reps skip count regex nel [B]
  TAG=$1; CASE=$2; REPS=$3; SKIP=$4; CNT=$5; REGEX=$6; NEL=$7; B=$8
  timeout 600 python tools/run_case.py $CASE $REPS $B > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain $TAG failed"; return; }
  timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:$REGEX -s $SKIP -c $CNT \
      -o /tmp/prof_$TAG python tools/run_case.py $CASE $REPS $B > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu $TAG exit $?"
  ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > /tmp/prof_${TAG}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_${TAG}_src.csv 2>/dev/null
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source sass > /tmp/prof_${TAG}_sass.csv 2>/dev/null
  python tools/ncu_summary.py full /tmp/prof_${TAG}_raw.csv > gpurun_out/prof_${TAG}_metrics.txt 2>&1
  python tools/ncu_sass_ops.py /tmp/prof_${TAG}_sass.csv $NEL > gpurun_out/prof_${TAG}_ops.txt 2>&1
  python tools/ncu_src_lines.py /tmp/prof_${TAG}_src.csv 0.8 $NEL > gpurun_out/prof_${TAG}_lines.txt 2>&1
}
prof r02_c2 c2 2 8 8 k_pass 786432
prof r02_c4 c4 2 6 6 k_pass 16777216
prof r02_c3 c3 2 4 4 k_pass 8388608 8
ls -la gpurun_out/
