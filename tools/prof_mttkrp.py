"""ncu driver: three A.6 MTTKRP launches on cfg4 (2048^3, 100M nnz, R=32 fp32).
    python tools/prof_mttkrp.py [NNZ_PER_TB NNZ_PER_WARP]"""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2001_00532_b200 import corpus, lower, synth
from paper_2001_00532_b200.execution import Executor
from paper_2001_00532_b200.formats import DeviceTensor
T = synth.config_matrix(4)
v = T.vals.astype(np.float32)
B = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, v, device="cuda", dtype="f32")
C = DeviceTensor.dense(synth.dense((T.dims[1], 32), seed=401, dtype=np.float32), device="cuda")
D = DeviceTensor.dense(synth.dense((T.dims[2], 32), seed=402, dtype=np.float32), device="cuda")
out = torch.empty(T.dims[0] * 32, dtype=torch.float32, device="cuda")
p = [int(x) for x in sys.argv[1:3]] if len(sys.argv) > 2 else [2048, 256]
ex = Executor(lower(corpus.build("A6", NNZ_PER_TB=p[0], NNZ_PER_WARP=p[1], BOUND=1)), {"B": B, "C": C, "D": D}, out, dtype="f32")
for _ in range(3): ex.launch()
torch.cuda.synchronize()
