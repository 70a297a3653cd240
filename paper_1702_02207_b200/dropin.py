"""Switch the reference package ``oscbench`` over to the B200 path.

``install(oscbench)`` rebinds the hot-path functions of the reference --
``integrate`` (oscillator.py:234-263), ``rk4_step`` (:194-231),
``derivative`` (:184-191) and ``energy`` (:266-276) -- to this package's
GPU implementations, in every ``oscbench`` module that imported them by name
(``oscbench/__init__.py:9-23``, ``harness.py:33-42``, ``cli.py:34``, ...).
Everything else (types, validation, modal analysis, harness, CLI, the CPU
thread engine ``run_parallel``) stays the reference's own code, so after the
call a reference user -- or the reference's own test suite -- runs unchanged
on the B200.  The GPU functions return the caller's types (the reference's
``PhaseState``/``Trajectory``) and raise exceptions that are instances of the
reference's classes (``oscillator._family``).

``python -m pytest -p paper_1702_02207_b200.dropin <reference tests>``
does the rebinding before the reference's tests are imported (pytest plugin
hooks below) and, with ``OSC_DROPIN_REPORT=<path>``, writes how many calls
each rebound function served on the GPU -- the evidence that the suite ran
through ``libosc_b200.so`` rather than the reference's Python loop.
"""

from __future__ import annotations

import functools
import json
import os
import sys
import types

REBOUND = ("integrate", "rk4_step", "derivative", "energy")

CALLS: dict = {name: 0 for name in REBOUND}


def _gpu_functions() -> dict:
    from . import oscillator

    out = {}
    for name in REBOUND:
        fn = getattr(oscillator, name)

        @functools.wraps(fn)
        def counted(*args, _fn=fn, _name=name, **kw):
            CALLS[_name] += 1
            return _fn(*args, **kw)

        counted.__osc_b200__ = True
        out[name] = counted
    return out


def install(oscbench: types.ModuleType | None = None, names=REBOUND):
    """Rebind ``names`` throughout the ``oscbench`` package; returns an
    ``uninstall`` callable that restores every rebound attribute.

    A module attribute is rebound only where it IS the reference's function
    (``from .oscillator import integrate`` copies), so helpers of the same
    name elsewhere are left alone."""
    from . import _native

    _native.lib()  # fail here, loudly, when there is no device or library
    if oscbench is None:
        import oscbench  # noqa: F811
    import importlib
    import pkgutil

    for info in pkgutil.iter_modules(oscbench.__path__):
        importlib.import_module(f"{oscbench.__name__}.{info.name}")
    originals = {name: getattr(oscbench.oscillator, name) for name in names}
    gpu = _gpu_functions()
    rebound = []
    for modname, mod in list(sys.modules.items()):
        if mod is None or not (modname == oscbench.__name__
                               or modname.startswith(oscbench.__name__ + ".")):
            continue
        for name in names:
            if getattr(mod, name, None) is originals[name]:
                rebound.append((mod, name, originals[name]))
                setattr(mod, name, gpu[name])

    def uninstall():
        for mod, name, fn in rebound:
            setattr(mod, name, fn)

    uninstall.rebound = [(m.__name__, n) for m, n, _ in rebound]
    return uninstall


# -- pytest plugin: `-p paper_1702_02207_b200.dropin` ------------------------

_STATE: dict = {}


def pytest_configure(config):
    _STATE["uninstall"] = install()
    config.addinivalue_line("markers", "gpu: (no-op in the reference suite)")


def pytest_report_header(config):
    where = sorted({m for m, _ in _STATE["uninstall"].rebound})
    return [f"osc_b200 drop-in: {', '.join(REBOUND)} rebound to the B200 path in {where}"]


def pytest_unconfigure(config):
    uninstall = _STATE.pop("uninstall", None)
    if uninstall is not None:
        uninstall()
    path = os.environ.get("OSC_DROPIN_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"calls": CALLS,
                       "rebound": uninstall.rebound if uninstall else []}, f, indent=1)
