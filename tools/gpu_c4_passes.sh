# Per-pass duration and DRAM bytes of the C4 forward (6 radix-16 passes, k=8,
# N=2^24): pass 0 has no twiddle multiplies (pure butterflies), passes 1-5
# carry the general multiplies.
timeout 300 python tools/run_case.py c4 2 > gpurun_out/plain_c4p.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_pass44 -s 6 -c 6 --csv --log-file gpurun_out/c4_passes.csv \
    python tools/run_case.py c4 2 > gpurun_out/ncu_c4p.log 2>&1
echo "exit $?"
