"""Reroute an imported ``kronblur`` (the reference package) to the B200 hot path.

kronblur binds its hot-path functions by name in several modules: ``pipeline`` does
``from .solvers import sfista, estimate_lipschitz`` (pipeline.py:27-35) and ``from .kron import
kron_apply, kron_apply_adjoint`` (pipeline.py:25); ``solvers`` does the same for kron_apply
(solvers.py:37). Replacing ``kronblur.solvers.sfista`` alone would leave ``restore()`` and
``run_case()`` on the CPU path, so every binding is patched. Results are returned as kronblur's
own ``SolveRun`` / ``IterationRecord`` types.
"""

from __future__ import annotations

import importlib

from . import blur as _blur
from . import kron as _kron
from . import solvers as _solvers

PATCH_SITES = {
    "sfista": ("", "solvers", "pipeline"),
    "kron_apply": ("", "kron", "solvers", "pipeline"),
    "kron_apply_adjoint": ("", "kron", "solvers", "pipeline"),
    "estimate_lipschitz": ("", "solvers", "pipeline"),
    # exact blur (psf.py:170-193): by-name imports in pipeline.py:26 and imaging.py:26
    "blur_direct": ("", "psf", "pipeline", "imaging"),
    # lambda selection (solvers.py:255-306): by-name import in pipeline.py:33
    "select_lambda": ("", "solvers", "pipeline"),
}


def _wrap_sfista(ref_solvers, options):
    def sfista(op, B, cfg, X0=None, truth=None, exact_apply=None):
        run = _solvers.sfista(op, B, cfg, X0=X0, truth=truth, exact_apply=exact_apply, options=options)
        hist = [ref_solvers.IterationRecord(k=h.k, t=h.t, objective=h.objective, eta=h.eta,
                                            gamma=h.gamma, ms=h.ms) for h in run.history]
        return ref_solvers.SolveRun(x=run.x, iterations=run.iterations, solve_ms=run.solve_ms,
                                    history=hist, iterates=run.iterates)

    sfista.__doc__ = "B200 sfista (kronblur signature); see paper_1901_00913_b200.solvers.sfista"
    return sfista


def install(kronblur_module=None, options: _solvers.SolveOptions | None = None):
    """Patch kronblur's hot-path bindings; returns a callable that restores the originals."""
    kb = kronblur_module or importlib.import_module("kronblur")
    ref_solvers = importlib.import_module(kb.__name__ + ".solvers")
    repl = {
        "sfista": _wrap_sfista(ref_solvers, options),
        "kron_apply": _kron.kron_apply,
        "kron_apply_adjoint": _kron.kron_apply_adjoint,
        "estimate_lipschitz": _solvers.estimate_lipschitz,
        "blur_direct": _blur.blur_direct,
        "select_lambda": _solvers.select_lambda,
    }
    saved = []
    for name, mods in PATCH_SITES.items():
        for sub in mods:
            mod = kb if not sub else importlib.import_module(f"{kb.__name__}.{sub}")
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, repl[name])

    def uninstall():
        for mod, name, orig in reversed(saved):
            setattr(mod, name, orig)

    return uninstall
