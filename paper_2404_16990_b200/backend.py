"""The reference package's own host code on the GPU engine.

Everything in the reference `multispin` that is not the sweep -- the CLI
(pkg/src/multispin/cli.py), the equilibration statistics
(observables.py:64-153), the record/replay harness (reference.py:179-208)
and its test suite -- reaches the engine through two names:
``multispin.engine.Engine`` and ``multispin.engine.run_simulations``
(re-bound by ``from .engine import ...`` in ``multispin/__init__.py:26`` and
``cli.py:23``).  ``install()`` re-binds those names, in every loaded
``multispin`` module, to this package's ``Engine`` / ``run_simulations``, so
the unmodified reference code runs on libmsb200:

    from paper_2404_16990_b200 import backend
    with backend.gpu_backend():
        multispin.cli.main(["simulate", ...])       # CSV byte-identical to the CPU run

The reference itself must be importable: pip-installed next to this
package, or in this checkout's ``baseline/_ref`` (tools/install_reference.sh).
Nothing here is on the hot path; it only decides which engine class the
reference's host code constructs.
"""

from __future__ import annotations

import contextlib
import importlib
import sys
from pathlib import Path

from .engine import Engine, run_simulations

__all__ = ["import_reference", "BackendEngine", "install", "gpu_backend"]

_LOCAL_REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
_PRISTINE_ADD4 = [None]  # the reference's own multispin.engine.bitwise_add4, captured at install()


def import_reference():
    """The reference package module (``multispin``)."""
    try:
        return importlib.import_module("multispin")
    except ImportError:
        if (_LOCAL_REF / "multispin").is_dir() and str(_LOCAL_REF) not in sys.path:
            sys.path.append(str(_LOCAL_REF))
            return importlib.import_module("multispin")
        raise ImportError("the reference package `multispin` is not importable: pip-install it, or run "
                          "tools/install_reference.sh to place it under baseline/_ref") from None


class BackendEngine(Engine):
    """``Engine`` that also honours the reference's adder fault seam.

    The reference selftest corrupts the word adder by replacing
    ``multispin.engine.bitwise_add4`` and expects the engine to diverge
    from the plain oracle (cli.py:460-473).  The GPU kernels never call
    that Python function, so while it is replaced this engine switches on
    its own adder corruption (``Engine.fault``, the kernels' ``fault`` flag).
    """

    @property
    def fault(self):
        mod = sys.modules.get("multispin.engine")
        pristine = _PRISTINE_ADD4[0]
        seam = mod is not None and pristine is not None and getattr(mod, "bitwise_add4", None) is not pristine
        return int(bool(self._fault) or seam)

    @fault.setter
    def fault(self, value):
        self._fault = value


def _multispin_modules():
    for name in ("multispin.engine", "multispin.observables", "multispin.reference", "multispin.cli"):
        try:
            importlib.import_module(name)
        except ImportError:
            pass
    return [m for k, m in list(sys.modules.items()) if m is not None and (k == "multispin" or k.startswith("multispin."))]


def install():
    """Re-bind ``Engine`` and ``run_simulations`` in every ``multispin``
    module to the GPU engine; returns a function that restores them."""
    import_reference()
    ref_engine = importlib.import_module("multispin.engine")
    originals = {"Engine": ref_engine.Engine, "run_simulations": ref_engine.run_simulations}
    if getattr(ref_engine.Engine, "__module__", "").startswith(__package__):
        return lambda: None  # already installed
    _PRISTINE_ADD4[0] = getattr(ref_engine, "bitwise_add4", None)
    swaps = {"Engine": BackendEngine, "run_simulations": run_simulations}
    done = []
    for mod in _multispin_modules():
        for attr, new in swaps.items():
            if getattr(mod, attr, None) is originals[attr]:
                setattr(mod, attr, new)
                done.append((mod, attr, originals[attr]))

    def restore():
        for mod, attr, old in done:
            setattr(mod, attr, old)
    return restore


@contextlib.contextmanager
def gpu_backend():
    """``install()`` for the duration of a ``with`` block."""
    restore = install()
    try:
        yield
    finally:
        restore()
