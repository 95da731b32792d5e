"""ctypes binding of the in-tree C-ABI library ``libnysb200.so`` (include/nysb200.h).

There is no CPU fallback: importing the solver API works anywhere (so the host
logic can be unit-tested), but every numeric entry point calls
:func:`require_device`, which raises :class:`NativeUnavailable` when the
library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NYS_LIB_PATH") or os.path.join(HERE, "libnysb200.so")   # override: A/B builds (tools/)

NYS_OK, NYS_EINVAL, NYS_ECUDA, NYS_EWORKSPACE, NYS_EUNSUPPORTED = range(5)
INFO_OK, INFO_SINGULAR, INFO_NONFINITE, INFO_DIVERGED, INFO_MAXITERS, INFO_DEGENERATE = range(6)

_vp, _i, _d, _sz = C.c_void_p, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); keep in sync with include/nysb200.h
SIGNATURES = {
    "nys_abi_version": (_i, []),
    "nys_status_string": (C.c_char_p, [_i]),
    "nys_last_cuda_error": (C.c_char_p, []),
    "nys_launch_count": (C.c_ulonglong, []),
    "nys_replay_pair": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "nys_stage_upload": (_i, [_vp, _vp, _sz, _vp, _vp, _vp, _vp]),
    "nys_stage_download": (_i, [_vp, _vp, _sz, _vp, _vp]),
    "nys_landmark_eig_workspace_bytes": (_sz, [_i]),
    "nys_landmark_eig_f64": (_i, [_vp, _i, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nys_feature_matrix_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _i, _vp, _i, _vp, _i, _vp]),
    "nys_predict_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _i, _vp, _i, _vp, _i, _i, _vp, _i, _vp]),
    "nys_fused_gram_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "nys_fused_gram_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _i, _vp, _vp, _vp, _i, _i, _i, _vp,
                                _vp, _sz, _vp]),
    "nys_batch_gram_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "nys_batch_gram_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _i, _vp, _i, _vp, _vp, _i, _vp, _vp,
                                _sz, _vp]),
    "nys_kkt_workspace_bytes": (_sz, [_i, _i, _i]),
    "nys_kkt_solve_f64": (_i, [_vp, _i, _i, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp, _sz,
                               _vp]),
    "nys_batch_kkt_solve_f64": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _d, _i, _vp, _vp, _vp]),
    "nys_ode_residual_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _i, _vp, _vp, _vp, _i, _vp, _vp]),
    "nys_transpose_f64": (_i, [_vp, _i, _i, _vp, _vp]),
    "nys_newton_pack_doubles": (_sz, [_i, _i]),
    "nys_newton_pack_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _vp, _i, _vp, _vp]),
    "nys_newton_residual_f64": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _i, _vp, _vp, _i, _vp, _i, _vp, _vp, _vp, _vp,
                                     _vp]),
    "nys_newton_trial_scratch_bytes": (C.c_size_t, [_i, _i, _i, _i]),
    "nys_newton_trial_norms_f64": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _i, _vp, _vp, _vp, _i, _vp, _i, _vp, _i, _vp, _vp,
                                        C.c_size_t, _vp]),
    "nys_newton_reduced_f64": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _i, _vp,
                                    _vp, _vp]),
    "nys_newton_reduced_workspace_bytes": (_sz, [_i, _i, _i]),
    "nys_newton_reduced_ws_f64": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _i,
                                       _vp, _vp, _vp, _sz, _vp]),
    "nys_lu_solve_f64": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp]),
    "nys_newton2_workspace_bytes": (_sz, [_i, _i, _i]),
    "nys_newton2_pack_doubles": (_sz, [_i, _i]),
    "nys_newton2_pack_f64": (_i, [_vp, _i, _vp, _i, _i, _d, _vp, _i, _vp, _vp]),
    "nys_newton2_residual_f64": (_i, [_vp, _vp, _vp, _i, _i, _vp, _i, _vp, _vp, _vp, _i, _vp,
                                      _vp, _i, _vp, _i, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nys_newton2_reduced_f64": (_i, [_vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _i,
                                     _vp, _vp, _vp, _sz, _vp]),
    "nys_newton2_step_f64": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _i, _vp, _i, _vp]),
    "nys_leverage_workspace_bytes": (_sz, [_i]),
    "nys_leverage_scores_f64": (_i, [_vp, _i, _d, _d, _vp, _vp, _vp, _sz, _vp]),
    "nys_pchol_rbf_f64": (_i, [_vp, _i, _d, _d, _i, _vp, _vp, _vp]),
    "nys_leverage_sketch_workspace_bytes": (_sz, [_i, _i, _i]),
    "nys_leverage_sketch_f64": (_i, [_vp, _i, _vp, _i, _d, _d, _vp, _i, _vp, _vp, _vp, _sz, _vp]),
    "nys_sym_eig_workspace_bytes": (_sz, [_i]),
    "nys_landmark_eig_compressed_workspace_bytes": (_sz, [_i]),
    "nys_landmark_eig_compressed_f64": (_i, [_vp, _i, _i, _d, _vp, _vp, _vp, _i, _vp, _vp, _vp,
                                             _sz, _vp]),
    "nys_explicit_gram_workspace_bytes": (_sz, [_i, _i]),
    "nys_kspace_gram_workspace_bytes": (_sz, [_i, _i, _i]),
    "nys_kspace_gram_f64": (_i, [_vp, _i, _d, _i, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _sz,
                                 _vp]),
    "nys_kspace_project_workspace_bytes": (_sz, [_i, _i]),
    "nys_kspace_project_f64": (_i, [_vp, _i, _vp, _i, _i, _vp, _vp, _sz, _vp]),
    "nys_explicit_gram_f64": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nys_sym_eig_f64": (_i, [_vp, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "nys_newton_step_f64": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _i, _vp, _i, _i, _vp]),
    "nys_newton_solve_once_work_doubles": (_sz, [_i, _i, _i]),
    "nys_newton_persist_profile": (None, [_vp]),
    "nys_newton_ladder_f64": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _i, _d, _i, _i, _vp,
                                   _sz, _vp, _vp, _vp, _vp, _vp]),
    "nys_newton_solve_once_f64": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _i, _vp, _vp, _vp, _i, _vp, _i, _i, _d, _i, _i, _vp,
                                       _sz, _vp, _vp, _vp, _vp]),
}


class NativeUnavailable(RuntimeError):
    """The CUDA extension or a CUDA device is missing (no CPU fallback exists)."""


class NativeError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str = ""):
        super().__init__(f"{fn} failed: status {status} ({detail})")
        self.status = status


_lib: Optional[C.CDLL] = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libnysb200.so and attach the prototypes (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_GRAPH_LAUNCHES = 0


def note_graph_launches(n: int) -> None:
    """Kernels replayed from a CUDA graph (the C-side counter only sees the
    launches made while the graph was captured)."""
    global _GRAPH_LAUNCHES
    _GRAPH_LAUNCHES += int(n)


def launch_count() -> int:
    """nys_launch_count() plus kernels replayed from captured graphs."""
    return int(load().nys_launch_count()) + _GRAPH_LAUNCHES


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def require_device():
    """Return (lib, torch) or raise: the product path has no CPU fallback."""
    import torch

    lib = load()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the nysb200 solver path runs on the GPU only")
    return lib, torch


def check(status: int, fn: str):
    if status != NYS_OK:
        lib = load()
        detail = lib.nys_status_string(status).decode()
        if status == NYS_ECUDA:
            detail += ": " + lib.nys_last_cuda_error().decode()
        raise NativeError(fn, status, detail)


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def call(name: str, *args):
    lib = load()
    check(getattr(lib, name)(*args), name)


class Workspace:
    """Grow-only device scratch buffer (one per device), reused across calls."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes: int, device):
        import torch

        key = str(device)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            self._buf[key] = buf
        return buf


WORKSPACE = Workspace()


def as_f64(x, device):
    """numpy / list / tensor -> contiguous float64 tensor on device."""
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).contiguous()
    a = np.ascontiguousarray(x, dtype=np.float64)
    if not a.flags.writeable:
        a = a.copy()
    return torch.as_tensor(a, device=device)
