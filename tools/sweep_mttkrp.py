"""A6 MTTKRP on cfg4 across schedule constants (tooling)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2001_00532_b200 import corpus, lower, synth
from paper_2001_00532_b200.execution import Executor
from paper_2001_00532_b200.formats import DeviceTensor
sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_configs import time_launch

T = synth.config_matrix(4)
dev = torch.device("cuda")
B = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, T.vals.astype(np.float32), device=dev, dtype="f32")
C = DeviceTensor.dense(synth.dense((2048, 32), seed=401, dtype=np.float32), device=dev)
D = DeviceTensor.dense(synth.dense((2048, 32), seed=402, dtype=np.float32), device=dev)
out = torch.empty(2048 * 32, dtype=torch.float32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for tb, w in [(2048, 256), (4096, 512), (8192, 1024), (16384, 2048), (16384, 4096), (8192, 8192)]:
    prog = lower(corpus.build("A6", NNZ_PER_TB=tb, NNZ_PER_WARP=w))
    ex = Executor(prog, {"B": B, "C": C, "D": D}, out, dtype="f32")
    ts = time_launch(ex, flush, 8, 3)
    print(tb, w, round(float(np.median(ts)), 4), flush=True)
