"""Run one landmark eigendecomposition (config given as argv[1]) -- ncu target."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_04094_b200 import nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = W.CONFIGS[cid]
g = W.grid(W.scaled(c, n=min(c.n, 1 << 16)))
lm = W.equidistant_landmarks(g, c.m)
for _ in range(2):
    fm = N.build_feature_map(RbfKernel(c.sigma2), lm)
torch.cuda.synchronize()
print("m_eff", fm.m_eff, "sweeps", fm._host["sweeps"])
