"""Integration hook: rebind the reference package's hot-path functions to this package's CUDA adapters.

The reference's "operator API" for the hot path is a handful of plain module functions:

    selector.cumulative_products / select_tetris / expected_accepted          (selector.py:95-176, :286-306)
    accept_model.verify_token / residual_distribution / sample_emitted_token  (accept_model.py:291-327, :357-368)
    sim_engine.apply_verification                                             (sim_engine.py:374-404)

and the modules that import them by name (sim_engine.py:27-35, cli.py:21-29, the package __init__.py).  A caller that
already uses `tetris_sched` switches the hot path to the GPU with

    import tetris_sched, tetris_sched.selector as S, tetris_sched.accept_model as A, tetris_sched.sim_engine as E
    import tetris_sched.cli as CLI
    from paper_2502_15197_b200.dropin import install
    handle = install(S, A, E, CLI, tetris_sched)      # ... handle.uninstall() restores the CPU functions

`install` replaces every module attribute that IS one of the reference's original function objects (so re-exports
and `from .selector import select_tetris` bindings are all covered) and points the adapters' output types at the
reference's own classes (Candidate, Selection, PolicyStats, TokenDistribution, DegenerateResidualError, see
_types.py), so what the rebound reference code gets back compares equal to what it would have computed itself.
This package never imports `tetris_sched`: the caller hands the modules in.
"""
from __future__ import annotations

import functools
import threading
from collections import Counter
from types import ModuleType

from . import _types

# (defining module role, function name) -> adapter, resolved lazily so importing this module needs no GPU
HOT_PATH = {
    "selector": ("cumulative_products", "select_tetris", "expected_accepted"),
    "accept_model": ("verify_token", "residual_distribution", "sample_emitted_token"),
    "sim_engine": ("apply_verification",),
}
CLASSES = {
    "selector": ("Candidate", "Selection", "PolicyStats"),
    "accept_model": ("AcceptanceMatrix", "TokenDistribution", "DegenerateResidualError"),
}

_lock = threading.Lock()
_active = []


def _adapter(role: str, name: str):
    if role == "selector":
        from . import selector as m
    elif role == "accept_model":
        from . import accept_model as m
    else:
        from . import sim_engine as m
    return getattr(m, name)


class Installation:
    """What `install` changed; `calls` counts adapter invocations (proof that the rebound path ran)."""

    def __init__(self):
        self.patched = []      # (module, attribute, original)
        self.calls = Counter()
        self.prev_types = None
        self.active = True

    def uninstall(self) -> None:
        with _lock:
            if not self.active:
                return
            for mod, attr, orig in reversed(self.patched):
                setattr(mod, attr, orig)
            _types.restore(self.prev_types)
            self.active = False
            _active.remove(self)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()


def install(selector_mod: ModuleType, accept_model_mod: ModuleType, sim_engine_mod: ModuleType = None,
            *importers: ModuleType) -> Installation:
    """Rebind the hot-path functions of the given reference modules (and of every module in `importers` that holds
    them under the same name) to the CUDA adapters; returns an Installation (context manager / `.uninstall()`)."""
    roles = {"selector": selector_mod, "accept_model": accept_model_mod}
    if sim_engine_mod is not None:
        roles["sim_engine"] = sim_engine_mod
    for role, mod in roles.items():
        for name in HOT_PATH[role]:
            if not callable(getattr(mod, name, None)):
                raise TypeError(f"{mod.__name__} has no function {name!r}; is it the reference's {role} module?")
    with _lock:
        if _active:
            raise RuntimeError("the drop-in is already installed; uninstall() it first")
        inst = Installation()
        types = {}
        for role, names in CLASSES.items():
            for n in names:
                cls = getattr(roles[role], n, None)
                if cls is None:
                    raise TypeError(f"{roles[role].__name__} has no class {n!r}")
                types[n] = cls
        modules = list(dict.fromkeys([*roles.values(), *importers]))
        for role, mod in roles.items():
            for name in HOT_PATH[role]:
                orig = getattr(mod, name)
                wrapped = _counting(_adapter(role, name), inst.calls, name)
                for m in modules:
                    if getattr(m, name, None) is orig:
                        inst.patched.append((m, name, orig))
                        setattr(m, name, wrapped)
        inst.prev_types = _types.override(types)
        _active.append(inst)
        return inst


def _counting(fn, counter: Counter, name: str):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        counter[name] += 1
        return fn(*args, **kwargs)

    call.__tetris_b200_adapter__ = True
    return call


def installed() -> bool:
    return bool(_active)
