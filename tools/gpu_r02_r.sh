python -c "
from paper_2001_00532_b200 import build as b
b.build_variant('r0', 'spx_sddmm.cu', ['-DSPX_SDDMM_RING_ON=0'])
b.build_variant('r4', 'spx_sddmm.cu', ['-DSPX_SDDMM_RING=4'])
b.build_variant('r16', 'spx_sddmm.cu', ['-DSPX_SDDMM_RING=16'])"
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_fullscale.py tests/test_gpu_acceptance.py -q -x -k "sddmm or K6 or cfg3" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py --cfg 3 --only K6 2>&1 | tail -1 | cut -c1-250
for v in r0 r4 r16; do echo "variant $v"; SPX_LIB=tools/variants/libspx_$v.so timeout 600 python tools/bench_configs.py --cfg 3 --only K6 --no-parity 2>&1 | tail -1 | cut -c1-200; done
timeout 600 ncu --set full --clock-control none -k regex:sddmm_ring -c 1 -o gpurun_out/r_k6 -f python tools/bench_configs.py --reps 1 --warm 1 --no-parity --cfg 3 --only K6 > gpurun_out/r_k6.log 2>&1
echo done
