"""Exception identity with the reference package, when it is importable.

The reference's callers catch its own classes: ``harness._run_nls`` catches
``nysode.newton.MaxItersExceeded`` (pkg/src/nysode/harness.py:173), tests catch
``nysode.linear.SingularSystemError`` etc.  For the monkeypatch drop-in
 to keep those handlers working, every error this package
raises on the reference's behalf is a SUBCLASS of the reference's class when
``nysode`` can be imported, and of the reference's own base (ValueError,
LinAlgError, RuntimeError) otherwise.

Only the exception classes are taken from ``nysode`` -- no reference code runs.
Set ``NYSB200_NO_NYSODE=1`` to never import it.
"""
from __future__ import annotations

import importlib
import os

_CACHE: dict = {}


def _nysode_module(name: str):
    if os.environ.get("NYSB200_NO_NYSODE"):
        return None
    if name in _CACHE:
        return _CACHE[name]
    try:
        mod = importlib.import_module(f"nysode.{name}")
    except Exception:    # not installed / not on sys.path: plain bases
        mod = None
    _CACHE[name] = mod
    return mod


def ref_base(module: str, cls: str, fallback: type) -> tuple:
    """Bases for a mirror of ``nysode.<module>.<cls>`` (fallback when absent)."""
    mod = _nysode_module(module)
    ref = getattr(mod, cls, None) if mod is not None else None
    if isinstance(ref, type) and issubclass(ref, BaseException):
        return (ref,)
    return (fallback,)


def nysode_available() -> bool:
    return _nysode_module("newton") is not None
