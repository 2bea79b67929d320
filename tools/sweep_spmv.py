"""A2 SpMV on cfg5 and K6 SDDMM on cfg3 across schedule constants (tooling)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np, torch
from bench_configs import time_launch
from paper_2001_00532_b200 import corpus, lower, synth
from paper_2001_00532_b200.execution import Executor
from paper_2001_00532_b200.formats import DeviceTensor

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
A = synth.config_matrix(5)
Ad = DeviceTensor.from_arrays((A.M, A.N), "ds", {1: A.pos}, {1: A.crd}, A.vals, device=dev)
x = DeviceTensor.dense(synth.dense((A.N,), seed=105), device=dev)
y = torch.empty(A.M, dtype=torch.float64, device=dev)
for tb, w, t in [(2048, 256, 8), (1024, 128, 4), (2048, 128, 4), (4096, 512, 16), (8192, 512, 16), (1024, 256, 8), (4096, 256, 8)]:
    ex = Executor(lower(corpus.build("A2", NNZ_PER_TB=tb, NNZ_PER_WARP=w, NNZ_PER_THREAD=t)), {"A": Ad, "x": x}, y, dtype="f64")
    print("spmv", tb, w, t, round(statistics.median(time_launch(ex, flush, 9, 3)), 4), flush=True)
del Ad, A
torch.cuda.empty_cache()
B = synth.config_matrix(3)
Bd = DeviceTensor.from_arrays((B.M, B.N), "ds", {1: B.pos}, {1: B.crd}, B.vals.astype(np.float32), device=dev, dtype="f32")
C = DeviceTensor.dense(synth.dense((B.M, 256), seed=303, dtype=np.float32), device=dev)
D = DeviceTensor.dense(synth.dense((B.N, 256), seed=304, dtype=np.float32), device=dev)
o = torch.empty(B.nnz, dtype=torch.float32, device=dev)
for tb, w in [(2048, 256), (4096, 512), (1024, 128), (2048, 128), (4096, 256), (8192, 1024)]:
    ex = Executor(lower(corpus.build("K6", NNZ_PER_TB=tb, NNZ_PER_WARP=w, BOUND=8)), {"B": Bd, "C": C, "D": D}, o, dtype="f32", dense_out=False)
    print("sddmm", tb, w, round(statistics.median(time_launch(ex, flush, 9, 3)), 4), flush=True)
