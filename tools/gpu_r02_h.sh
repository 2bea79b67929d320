for v in "t384:-DSPX_MQ_THREADS=384" "mb1:-DSPX_MQ_MINB=1" "t256m3:-DSPX_MQ_THREADS=256 -DSPX_MQ_MINB=4"; do
  python -c "from paper_2001_00532_b200 import build as b; b.build_variant('${v%%:*}', 'spx_csf.cu', '${v#*:}'.split())" ; done
timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_irpath.py -q -x -k "mttkrp or stats" 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 2>&1 | tail -1 | cut -c1-250
for v in t384 mb1 t256m3; do echo "variant $v"; SPX_LIB=tools/variants/libspx_$v.so timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200; done
SPX_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/h_bench2.json 2> gpurun_out/h_bench2.err; tail -c 1500 gpurun_out/h_bench2.json; tail -3 gpurun_out/h_bench2.err
