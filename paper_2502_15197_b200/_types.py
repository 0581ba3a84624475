"""The container classes and exceptions the drop-in adapters construct / raise.

By default these are this package's mirrors of the reference's dataclasses (selector.py / accept_model.py below).
`dropin.install()` points them at the reference's own classes (tetris_sched.selector.Selection, PolicyStats,
Candidate, accept_model.TokenDistribution, DegenerateResidualError, ...), so that every object the rebound reference
code receives from an adapter is an instance of the reference's class and compares equal to what the reference
itself would have built (tetris_sched tests/test_selector.py:121, :217; tests/test_accept_model.py:179-195).
Adapters read their inputs by duck typing (`.rows`, `.probs`, `.windows`, `.cum`), so either family is accepted.
"""
from __future__ import annotations

_DEFAULTS: dict = {}
_current: dict = {}

NAMES = ("Candidate", "Selection", "PolicyStats", "AcceptanceMatrix", "TokenDistribution", "DegenerateResidualError")


def set_default(name: str, cls) -> None:
    _DEFAULTS[name] = cls
    _current.setdefault(name, cls)


def get(name: str):
    return _current[name]


def override(mapping: dict) -> dict:
    """Install `mapping` (name -> class); returns the previous bindings for `restore`."""
    prev = dict(_current)
    for name, cls in mapping.items():
        if name not in NAMES:
            raise KeyError(f"unknown container name {name!r}")
        _current[name] = cls
    return prev


def restore(prev: dict) -> None:
    _current.clear()
    _current.update(prev)


def defaults() -> dict:
    return dict(_DEFAULTS)
