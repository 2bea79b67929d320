# the N>1 bench path on one GPU (SPX_BENCH_SHARED_GPU=1: two ranks share cuda:0 over gloo)
SPX_BENCH_SHARED_GPU=1 timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/at_bench2.json 2> gpurun_out/at_bench2.err; echo "rc=$?"
tail -c 1500 gpurun_out/at_bench2.json; tail -5 gpurun_out/at_bench2.err
