# MTTKRP quarter kernel: parity, cfg4 timing, variant sweep, ncu.
for v in "t512:-DSPX_MQ_THREADS=512" "r4:-DSPX_MQ_RING=4" "t256:-DSPX_MQ_THREADS=256 -DSPX_MQ_MINB=3"; do
  python -c "from paper_2001_00532_b200 import build as b; b.build_variant('${v%%:*}', 'spx_csf.cu', '${v#*:}'.split())" ; done
timeout 900 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_edge.py -q -x -k "mttkrp" 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 2>&1 | tail -1 | cut -c1-300
for w in 128 512; do timeout 300 python tools/bench_configs.py --cfg 4 --only A6 --no-parity --params NNZ_PER_TB=$((w*8)),NNZ_PER_WARP=$w 2>&1 | tail -1 | cut -c1-200; done
for v in t512 r4 t256; do echo "variant $v"; SPX_LIB=tools/variants/libspx_$v.so timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -s 2 -c 1 -o gpurun_out/mq_full3 -f python tools/prof_mttkrp.py > gpurun_out/mq_ncu.log 2>&1; tail -2 gpurun_out/mq_ncu.log
