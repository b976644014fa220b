# multi-rank flow smoke of bench.py on ONE GPU (2 ranks share it over gloo;
# timings meaningless) + the reference arm
GFP_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --cpu-budget 2 \
  > gpurun_out/flow2.json 2> gpurun_out/flow2.err; echo "flow exit $?"
tail -3 gpurun_out/flow2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref exit $?"
