"""Module swap: make ``import modpa`` resolve to this package.

The reference's callers import ``modpa.pa``, ``modpa.bignum``,
``modpa.bench`` and ``modpa.security`` (pkg/src/modpa/__init__.py:10-35,
pkg/src/modpa/bench.py).  ``install()`` registers this package's modules
under those names, so a caller -- or the reference's own hash-path tests --
runs unchanged on the B200 path:

    import paper_1910_04429_b200.compat as c; c.install()
    from modpa import pa          # -> paper_1910_04429_b200.pa (CUDA)

Only the hash path is provided.  ``modpa.bench`` carries the
batch/bench callers of that path (RunConfig, run_pa, run_bench, bench_input,
measure_ratio_spread); the CLI, reports and the universality auditor are out
of scope and are not registered.
"""
from __future__ import annotations

import sys
import types

from . import benchrun, bignum, pa, runpa, security

_NAMES = ("modpa", "modpa.pa", "modpa.bignum", "modpa.bench", "modpa.security")


def _bench_module() -> types.ModuleType:
    m = types.ModuleType("modpa.bench")
    m.__doc__ = "B200 drop-in for pkg/src/modpa/bench.py (batch and benchmark callers)."
    for src in (runpa, benchrun):
        for k, v in vars(src).items():
            if not k.startswith("__"):
                setattr(m, k, v)
    m.TIMING_PIPELINE, m.TIMING_MULTIPLY = "pipeline", "multiply"
    return m


def install() -> types.ModuleType:
    """Register the swap in sys.modules; returns the ``modpa`` package module.

    Refuses to shadow a different ``modpa`` that is already imported.
    """
    cur = sys.modules.get("modpa")
    if cur is not None and getattr(cur, "__b200_dropin__", False):
        return cur
    if cur is not None:
        raise RuntimeError("another modpa is already imported; install() must run first")
    import paper_1910_04429_b200 as pkg

    top = types.ModuleType("modpa")
    top.__doc__ = pkg.__doc__
    top.__path__ = []  # a package, so `import modpa.pa` works
    top.__b200_dropin__ = True
    for k in pkg.__all__:
        setattr(top, k, getattr(pkg, k))
    bench = _bench_module()
    for name, mod in (("pa", pa), ("bignum", bignum), ("bench", bench), ("security", security)):
        setattr(top, name, mod)
        sys.modules["modpa." + name] = mod
    sys.modules["modpa"] = top
    return top


def uninstall() -> None:
    for name in _NAMES:
        mod = sys.modules.get(name)
        if name == "modpa" and not getattr(mod, "__b200_dropin__", False):
            return
        sys.modules.pop(name, None)
