"""Probe: device vs LAPACK spectrum of the P3 landmark matrix (noise-floor tail)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "baseline", "_ref"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from nysode import nystrom as N0, harness
from nysode.kernel import RbfKernel as K0
from nysode.problems import get_problem, grid_for
from paper_2510_04094_b200 import nystrom as N1
from paper_2510_04094_b200.kernel import RbfKernel as K1

for pid in (3, 12, 4):
    p = get_problem(pid); d = p.defaults
    g = grid_for(p, d.n)
    lm = N0.select_landmarks(N0.Equidistant(), g, d.m)
    f0 = N0.build_feature_map(K0(d.sigma2), lm)
    f1 = N1.build_feature_map(K1(d.sigma2), lm)
    from nysode import kernel as kern
    om = kern.kernel_matrix(K0(d.sigma2), 0, lm, lm)
    allv = np.linalg.eigvalsh((om + om.T) / 2)[::-1]
    print(f"P{pid} m={lm.size} m_eff ref {f0.m_eff} dev {f1.m_eff} s0 {allv[0]:.3e} thr {1e-16*allv[0]:.3e}")
    print("  ref all :", " ".join(f"{v:.2e}" for v in allv[15:]))
    print("  dev kept:", " ".join(f"{v:.2e}" for v in f1.eigenvalues[15:]))
    print("  dev _host keys", list(f1._host.keys()))
