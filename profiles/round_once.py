import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_06532_b200 as T
comm = T.default_comm()
y = T.DistTTTensor.random(comm, (8000,)*10, (1,)+(30,)*9+(1,), 0)
x = T.add(y, y)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    out = T.round_tt(x, T.RoundingOptions(1e-10))
torch.cuda.synchronize()
print(out.ranks)
