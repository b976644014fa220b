# checked-build cases (evidence file) + ncu of the word-prime NTT passes
GFPFFT_LIB=paper_1811_01490_b200/libgfpfft_checked.so timeout 900 python tools/checked_cases.py > gpurun_out/checked_cases.txt 2>&1; echo "checked exit $?"
tail -3 gpurun_out/checked_cases.txt
timeout 300 python tools/word_time.py > gpurun_out/word_time.txt 2>&1; cat gpurun_out/word_time.txt
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_word_pass -s 10 -c 5 -o /tmp/prof_word python tools/word_time.py > gpurun_out/ncu_word.log 2>&1
ncu -i /tmp/prof_word.ncu-rep --page raw --csv > /tmp/prof_word_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/prof_word_raw.csv > gpurun_out/prof_word_metrics.txt 2>&1
head -60 gpurun_out/prof_word_metrics.txt
