# Round-2 (TMA pass kernel) ncu evidence: --set full of the C4 passes and the C2 pass launches
set -x
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
  python tools/ncu_src_lines.py /tmp/prof_${TAG}_src.csv 0.5 $NEL > gpurun_out/prof_${TAG}_lines.txt 2>&1
}
prof r02b_c4 c4 2 6 6 "k_pass|k_first|k_pmid" 16777216
python tools/passes_table_r2.py gpurun_out/prof_r02b_c4_metrics.txt 16777216 "C4 forward, 2^24 k=8 (6 passes, k_pass44t)" > gpurun_out/r02b_ncu_c4_passes.md
prof r02b_c2 c2 2 7 7 "k_pass|k_first|k_pmid" 786432
python tools/passes_table_r2.py gpurun_out/prof_r02b_c2_metrics.txt 65536 "C2 poly-mul, 2^16 k=8 (7 launches: forward passes 0-2 on both operands, the fused forward-last + pointwise + inverse-first kernel, inverse passes 1-3)" > gpurun_out/r02b_ncu_c2_passes.md
prof r02b_c3 c3 2 4 4 "k_pass|k_first" 8388608 8
python tools/passes_table_r2.py gpurun_out/prof_r02b_c3_metrics.txt 8388608 "C3 forward, 8 x 2^20 k=16 (4 passes; pass 0 = k_first16t)" > gpurun_out/r02b_ncu_c3_passes.md
ls -la gpurun_out/
