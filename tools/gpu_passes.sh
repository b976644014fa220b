# Per-pass duration / DRAM bytes / pipe use of one forward transform of a case
# (tools/run_case.py <case> 2 [batch]); usage: CASE=c3 BATCH=8 NP=4 PAT=k_pass bash tools/gpu_passes.sh
CASE=${CASE:-c4}; NP=${NP:-6}; PAT=${PAT:-k_pass}
timeout 300 python tools/run_case.py $CASE 2 $BATCH > gpurun_out/plain_${CASE}p.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:$PAT -s $NP -c $NP --csv --log-file gpurun_out/${CASE}_passes.csv \
    python tools/run_case.py $CASE 2 $BATCH > gpurun_out/ncu_${CASE}p.log 2>&1
echo "exit $?"
