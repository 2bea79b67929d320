import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2001_00532_b200 import corpus, lower, synth
from paper_2001_00532_b200.execution import Executor
from paper_2001_00532_b200.formats import DeviceTensor
T = synth.config_matrix(4)
v = T.vals.astype(np.float32)
B = DeviceTensor.from_arrays(T.dims, "sss", T.pos, T.crd, v, device="cuda", dtype="f32")
c = DeviceTensor.dense(synth.dense((T.dims[2],), seed=403, dtype=np.float32), device="cuda")
out = torch.empty(T.dims[0]*T.dims[1], dtype=torch.float32, device="cuda")
p = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else [2048, 256, 8]
ex = Executor(lower(corpus.build("K11", NNZ_PER_TB=p[0], NNZ_PER_WARP=p[1], NNZ_PER_THREAD=p[2])), {"B": B, "c": c}, out, dtype="f32")
for _ in range(3): ex.launch()
torch.cuda.synchronize()
