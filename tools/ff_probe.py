import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
from test_gpu_full_feature import _problem, _rel
from conftest import load_golden
from paper_2510_04094_b200 import baselines as BL
g = load_golden("full_feature")
for pid in (1, 7, 8, 12, 16):
    key = f"p{pid}"; prob = _problem(g, key); n = int(g[f"{key}_n"])
    model, secs = BL.full_feature_baseline(prob, float(g[f"{key}_gamma"]), float(g[f"{key}_sigma2"]), n)
    y = model.predict(0, BL.grid_for(prob, n)); ref = g[f"{key}_yhat"]
    print(pid, "err %.2e yard %.2e m_eff %d/%d" % (_rel(y, ref), _rel(g[f"{key}_yhat_dsyev"], ref), model.feature_map.m_eff, int(g[f"{key}_m_eff"])))
