python -c "from paper_2001_00532_b200 import build as b; b.build_variant('v1', 'spx_csf.cu', ['-DSPX_MQ_V2=0']); b.build_variant('v2t384', 'spx_csf.cu', ['-DSPX_MQ_THREADS=384']); b.build_variant('v2r3', 'spx_csf.cu', ['-DSPX_MQ_RING=3'])"
timeout 600 python -m pytest tests/test_gpu_mttkrp_quarter.py tests/test_gpu_shards.py -q -x 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --cfg 4 --only A6 2>&1 | tail -1 | cut -c1-250
for v in v1 v2t384 v2r3; do echo "variant $v"; SPX_LIB=tools/variants/libspx_$v.so timeout 600 python tools/bench_configs.py --cfg 4 --only A6 --no-parity 2>&1 | tail -1 | cut -c1-200; done
for w in 128 512; do timeout 300 python tools/bench_configs.py --cfg 4 --only A6 --no-parity --params NNZ_PER_TB=$((w*8)),NNZ_PER_WARP=$w 2>&1 | tail -1 | cut -c1-200; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_quarter -c 1 -o gpurun_out/j_k8 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 4 --only A6 > gpurun_out/j_k8.log 2>&1
echo done
