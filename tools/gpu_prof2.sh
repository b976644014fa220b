bash tools/gpu_prof.sh c4 7 1 c4 k_pass 16777216
bash tools/gpu_prof.sh c2 8 8 c2 k_pass 786432
