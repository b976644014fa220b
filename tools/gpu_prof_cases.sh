# ncu --set full of the pass kernel at C4 (k=8, N=2^24), C3 (k=16, 8 x 2^20) and
# the C5 multiply (k=32); each case first runs plain and must exit 0.  The
# reports are reduced to CSV on the box (raw + source pages) to stay small.
set -x
cases=${CASES:-"c4 c3 c5"}
for n in $cases; do
  args="$n 1"; [ $n = c3 ] && args="c3 1 8"
  pat=${PAT:-'regex:k_pass'}; [ $n = c5 ] && pat='regex:k_mul_fast'
  timeout 300 python tools/run_case.py $args > gpurun_out/plain_$n.log 2>&1 && \
  timeout 900 ncu -f --set full --clock-control none --import-source on -k $pat -s 1 -c 1 \
      -o /tmp/prof_$n python tools/run_case.py $args > gpurun_out/ncu_$n.log 2>&1
  echo "$n exit $?"
  ncu -i /tmp/prof_$n.ncu-rep --page raw --csv > gpurun_out/prof_${n}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${n}_src.csv 2>/dev/null
  ncu -i /tmp/prof_$n.ncu-rep --page details --csv > gpurun_out/prof_${n}_details.csv 2>/dev/null
  ls -la /tmp/prof_$n.ncu-rep
done
