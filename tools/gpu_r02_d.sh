timeout 600 python -m pytest tests/test_gpu_coo.py tests/test_gpu_generic.py tests/test_gpu_irpath.py tests/test_gpu_pack.py -q -x 2>&1 | tail -25
