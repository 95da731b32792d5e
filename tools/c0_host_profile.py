import cProfile, pstats, sys, os, time
sys.path.insert(0, ".")
if os.environ.get("NYS_PROBE_LIB"):
    from paper_2510_04094_b200 import _lib
    _lib.load(os.environ["NYS_PROBE_LIB"])
import torch
from paper_2510_04094_b200 import linear as L, workloads as W
from paper_2510_04094_b200.problems import ivp
cfg = W.CONFIGS[int(os.environ.get("CFG", "0"))]
bt = W.linear_batch(cfg, 0, 1)
cond = ivp(bt.instances[0].conditions())
pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond, device="cuda")
p = torch.as_tensor(bt.pts, device="cuda"); c = torch.as_tensor(bt.coef[0], device="cuda"); f = torch.as_tensor(bt.forcing[0], device="cuda")
for _ in range(20):
    pipe.run_device(p, c, f)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    pipe.run_device(p, c, f)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host {1e6*(t1-t0)/500:.1f} us/call, wall {1e6*(t2-t0)/500:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    pipe.run_device(p, c, f)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# graph replay alone (host time of the launch)
g = next(iter(pipe._graph.values()))[0]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    g.replay()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"graph replay host {1e6*(t1-t0)/500:.1f} us, wall {1e6*(t2-t0)/500:.1f} us per replay")
from paper_2510_04094_b200 import nystrom as N
buf = pipe._eigbufs[0]
es = torch.cuda.Stream()
t0 = time.perf_counter()
for _ in range(500):
    N.launch_eig_async(pipe.kernel, buf, pipe.drop_tol, es)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"eig launch host {1e6*(t1-t0)/500:.1f} us, wall {1e6*(t2-t0)/500:.1f} us per eig")

# warm per-kernel durations of the replayed post graph
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = {}
for e in ev:
    agg.setdefault(e.name[:60], []).append(e.time_range.end - e.time_range.start)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v) / len(v):8.1f} us x{len(v)}  {k}")
