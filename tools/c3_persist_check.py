"""Device-resident Newton (NYS_NEWTON_PERSIST=1) vs the host-orchestrated loop
on the config-3 batch: outcomes, traces, y_hat and step time."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W, linear as L
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = W.CONFIGS[3]
g = W.grid(cfg); lm = W.equidistant_landmarks(g, cfg.m); pts = g[1:]
insts = [W.instance(3, 0, i) for i in range(B)]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]), np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
res = {}
for mode in ("0", "1"):
    os.environ["NYS_NEWTON_PERSIST"] = mode
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
        eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
        st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    Y = L.predict_batch(fm, X[:, :eng.me + 1], 0, g).cpu().numpy()
    res[mode] = (st, X, tr, rung, Y, dt)
    print(f"persist={mode}: {dt*1e3:.1f} ms  status {np.bincount(st, minlength=4).tolist()} "
          f"rungs {np.bincount(rung, minlength=6).tolist()} its {sum(len(t)-1 for t in tr)}", flush=True)
a, b = res["0"], res["1"]
same_st = int((a[0] == b[0]).sum())
same_tr = sum(1 for x, y in zip(a[2], b[2]) if len(x) == len(y) and np.array_equal(np.array(x), np.array(y)))
conv = (a[0] == 0) & (b[0] == 0)
d = max((np.linalg.norm(a[4][i] - b[4][i]) / np.linalg.norm(a[4][i]) for i in np.flatnonzero(conv)), default=0)
print(f"same status {same_st}/{B}; bit-identical traces {same_tr}/{B}; max y_hat rel diff (both converged) {d:.3e}")

# phase clocks per instance of one persistent rung (rung 3 start: linearized, undamped; and a damped rung)
os.environ["NYS_NEWTON_PERSIST"] = "1"
from paper_2510_04094_b200 import _lib
lib = _lib.load()
fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), vals, cfg.gamma, family=fam)
prof = torch.zeros((B, 8), dtype=torch.int64, device="cuda")
lib.nys_newton_persist_profile(prof.data_ptr())
ids = list(range(B))
for name, x0fn, damp in [("const undamped", lambda: eng.const_state(ids), False),
                         ("const damped", lambda: eng.const_state(ids), True),
                         ("lin undamped", lambda: eng.linearized_state(ids)[0], False),
                         ("lin damped", lambda: eng.linearized_state(ids)[0], True)]:
    x0 = x0fn()
    prof.zero_()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st, Xn, tr = eng.solve_once(ids, x0, cfg.gamma, 1e-10 * (1 + cfg.gamma), damp, cfg.newton_max_iters)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    p = prof.cpu().numpy().astype(float)
    its = np.array([len(t) - 1 for t in tr])
    j = int(np.argmax(p[:, :4].sum(1)))
    print(f"{name}: {dt*1e3:.1f} ms; its max {its.max()} sum {its.sum()}; slowest instance {j}: "
          f"its {its[j]} trials {int(p[j,5])} clocks resid/trials {p[j,0]:.3g} reduce {p[j,1]:.3g} "
          f"LU {p[j,2]:.3g} step {p[j,3]:.3g} -> per it reduce {p[j,1]/max(its[j],1):.3g} "
          f"LU {p[j,2]/max(its[j],1):.3g} step {p[j,3]/max(its[j],1):.3g} resid/trial "
          f"{p[j,0]/max(p[j,5]+its[j],1):.3g}", flush=True)
lib.nys_newton_persist_profile(None)
