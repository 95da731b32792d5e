"""One config-4-shaped fused Gram (kernel-space path) at n = argv[1] rows (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if os.environ.get("NYS_PROBE_LIB"):
    from paper_2510_04094_b200 import _lib
    _lib.load(os.environ["NYS_PROBE_LIB"])
from paper_2510_04094_b200 import linear as L, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 18)
cfg = W.scaled(W.CONFIGS[4], n=n)
bt = W.linear_batch(cfg, 0, 1)
fm = N.build_feature_map(RbfKernel(cfg.sigma2), bt.landmarks)
pts = torch.as_tensor(bt.pts, device="cuda")
coef = torch.as_tensor(bt.coef[0], device="cuda")
forc = torch.as_tensor(bt.forcing[0], device="cuda")
for _ in range(2):
    E = L.gram_ext_device(fm, 2, pts, coef, forc)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(3):
    E = L.gram_ext_device(fm, 2, pts, coef, forc)
ev[1].record()
torch.cuda.synchronize()
print("ok", float(E[0, 0]), "ms/gram", ev[0].elapsed_time(ev[1]) / 3)
