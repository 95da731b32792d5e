"""Time the config-2 batched Gram launch alone (optionally with a probe build
of the library, NYS_PROBE_LIB) -- CUDA events over 10 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2510_04094_b200 import _lib

if os.environ.get("NYS_PROBE_LIB"):
    _lib.load(os.environ["NYS_PROBE_LIB"])
from paper_2510_04094_b200 import batch as BT, workloads as W
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[2]
bt = W.linear_batch(cfg, 0, cfg.batch)
cond = ivp(bt.instances[0].conditions())
pipe = BT.SharedGridPipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond,
                             cfg.batch)
coef = torch.as_tensor(bt.coef, device="cuda")
forc = torch.as_tensor(bt.forcing, device="cuda")
vals = torch.as_tensor(bt.cond_values, device="cuda")
x, info = pipe.run_device(coef, forc, vals)
torch.cuda.synchronize()
s = pipe.solver
fm = s.fmap
lib = _lib.load()
wsb = lib.nys_batch_gram_workspace_bytes(s.n_c, fm.m_eff, s.order, cfg.batch)


def gram():
    _lib.call("nys_batch_gram_f64", _lib.ptr(fm.d_landmarks), fm.m, _lib.ptr(fm.d_W), fm.m,
              fm.m_eff, float(cfg.sigma2), s.order, _lib.ptr(s.pts), s.n_c, _lib.ptr(coef),
              _lib.ptr(forc), cfg.batch, None, _lib.ptr(s.ws), wsb, _lib.stream_ptr())


for _ in range(3):
    gram()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    gram()
e1.record()
torch.cuda.synchronize()
print(f"gram+psi: {e0.elapsed_time(e1) / 10:.3f} ms   info ok: {int((info == 0).sum())}/{cfg.batch}")
