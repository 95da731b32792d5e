"""Helpers shared by the -m gpu parity tests (golden fixtures only: the GPU box
has no /root/reference)."""
import numpy as np

from paper_2510_04094_b200 import linear as L
from paper_2510_04094_b200 import nystrom as N
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import BoundaryCondition, Conditions


def fmap_from_golden(g):
    return N.build_feature_map(RbfKernel(float(g["sigma2"])), g["landmarks"])


def conditions(g, b=0):
    ents = tuple(BoundaryCondition(float(t), int(o), float(v)) for t, o, v in
                 zip(g["cond_points"], g["cond_orders"], g["cond_values"][b]))
    return Conditions(str(g["kind"]), ents)


class ArraySpec:
    """A LinearOdeSpec whose callables replay sampled golden arrays."""

    def __init__(self, order, coef, forcing, pts):
        self.order = order
        self._pts = pts
        self.coeffs = tuple((lambda t, c=c: self._at(t, c)) for c in coef)
        self.forcing = lambda t: self._at(t, forcing)
        self.domain = (float(pts[0]), float(pts[-1]))

    def _at(self, t, arr):
        t = np.asarray(t, dtype=float)
        assert t.shape == self._pts.shape and np.array_equal(t, self._pts)
        return arr


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def solve_golden_instance(g, fmap, b):
    spec = ArraySpec(int(g["order"]), g["coef"][b], g["forcing"][b], g["pts"])
    sy = L.assemble(spec, conditions(g, b), fmap, g["grid"], float(g["gamma"]))
    return sy, L.solve(sy, fmap)
