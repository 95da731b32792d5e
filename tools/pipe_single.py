"""single_timeline.py plug-in: the SingleSolvePipeline path."""
from paper_2510_04094_b200 import linear as L


def make(cfg, bt, cond, pts, coef, forc):
    pipe = L.SingleSolvePipeline(bt.landmarks, cfg.sigma2, bt.grid, cfg.gamma, cfg.order, cond)
    return lambda: pipe.run_device(pts, coef, forc)
