# ncu --set full of the pass kernels of one case (after a plain run exits 0):
#   bash tools/gpu_prof.sh <case> <skip> <count> <tag> [kernel-regex] [n_elements]
# summaries (metrics per launch, SASS opcode mix, per-line hot spots) land in
# gpurun_out/prof_<tag>_*.txt; the big CSVs stay in /tmp on the box
CASE=$1; SKIP=$2; CNT=$3; TAG=$4; REGEX=${5:-k_pass}; NEL=${6:-0}
timeout 300 python tools/run_case.py $CASE 2 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain $TAG failed"; exit 1; }
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:$REGEX -s $SKIP -c $CNT \
    -o /tmp/prof_$TAG python tools/run_case.py $CASE 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG exit $?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > /tmp/prof_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_${TAG}_src.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source sass > /tmp/prof_${TAG}_sass.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/prof_${TAG}_raw.csv > gpurun_out/prof_${TAG}_metrics.txt 2>&1
python tools/ncu_sass_ops.py /tmp/prof_${TAG}_sass.csv $NEL > gpurun_out/prof_${TAG}_ops.txt 2>&1
python tools/ncu_src_lines.py /tmp/prof_${TAG}_src.csv 0.8 $NEL > gpurun_out/prof_${TAG}_lines.txt 2>&1
head -c 200000 /tmp/prof_${TAG}_sass.csv > gpurun_out/prof_${TAG}_sass_head.csv
ls -la gpurun_out/prof_${TAG}_*
