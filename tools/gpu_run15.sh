SPX_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r1_n2.json 2> gpurun_out/r1_n2.err
cat gpurun_out/r1_n2.json; tail -5 gpurun_out/r1_n2.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r1_n1.json 2> gpurun_out/r1_n1.err; cat gpurun_out/r1_n1.json; tail -3 gpurun_out/r1_n1.err
