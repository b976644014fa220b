timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" > gpurun_out/g3_nw.log
timeout 300 python tools/run_case.py c4s 2 > gpurun_out/plain_c4s.log 2>&1 && \
timeout 900 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:bool.1>' -c 2 -o /tmp/prof_xch python tools/run_case.py c4s 2 > gpurun_out/ncu_xch.log 2>&1
echo "ncu xch exit $?" >> gpurun_out/g3_nw.log
ncu -i /tmp/prof_xch.ncu-rep --page raw --csv > gpurun_out/prof_xch_raw.csv 2>/dev/null
python tools/ncu_summary.py full gpurun_out/prof_xch_raw.csv > gpurun_out/prof_xch_metrics.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4s.csv python tools/run_case.py c4s 2 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4s.csv > gpurun_out/launches_c4s.txt 2>&1
