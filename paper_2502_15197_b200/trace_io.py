"""StepOutcome wire format: the reference's JSONL step trace (trace_io.py:119-206) for outcomes
produced on the GPU (sim_engine.GpuSimulator), byte-compatible with tetris_sched's write_trace / read_trace so a GPU
run feeds metrics.build_report (metrics.py:166-228) unchanged.  Host-side I/O; nothing here touches the device.
"""
from __future__ import annotations

import json
from pathlib import Path
from typing import Sequence

from .sim_engine import GpuStepOutcome

TRACE_SCHEMA = "tetris-sched-trace"  # trace_io.py:21-22
TRACE_VERSION = 1


class TraceSchemaError(ValueError):
    """A trace file does not match the expected schema (trace_io.py:33-34)."""


def outcome_to_json(o) -> dict:
    """trace_io.py:119-139: same keys in the same order (json.dumps keeps insertion order)."""
    st = o.stats
    return {
        "step": o.step,
        "windows": list(o.windows),
        "accepted": list(o.accepted),
        "credited": list(o.credited),
        "bonus": o.bonus,
        "sent": sum(o.windows),
        "tau": o.tau,
        "expected_accepted": o.expected_accepted,
        "stats": None if st is None else {"extracts": st.extracts, "inserts": st.inserts,
                                          "peak_queue": st.peak_queue, "comparisons": st.comparisons},
        "completions": [list(c) for c in o.completions],
    }


def write_trace(outcomes: Sequence, path) -> None:
    """One header line, then one line per step (trace_io.py:166-173)."""
    path = Path(path)
    header = {"schema": TRACE_SCHEMA, "version": TRACE_VERSION, "steps": len(outcomes)}
    with path.open("w") as fh:
        fh.write(json.dumps(header) + "\n")
        for o in outcomes:
            fh.write(json.dumps(outcome_to_json(o)) + "\n")


def read_trace(path) -> list:
    """Read a trace back into GpuStepOutcome records; schema problems name the offending line (trace_io.py:176-206)."""
    from .selector import PolicyStats

    path = Path(path)
    lines = path.read_text().splitlines()
    if not lines:
        raise TraceSchemaError(f"{path}: line 1: empty file, header expected")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as exc:
        raise TraceSchemaError(f"{path}: line 1: {exc.msg}") from None
    if not isinstance(header, dict) or header.get("schema") != TRACE_SCHEMA:
        raise TraceSchemaError(f"{path}: line 1: not a {TRACE_SCHEMA} header")
    if header.get("version") != TRACE_VERSION:
        raise TraceSchemaError(f"{path}: line 1: unsupported trace version {header.get('version')!r}")
    out = []
    for lineno, raw in enumerate(lines[1:], start=2):
        try:
            obj = json.loads(raw)
            st = obj["stats"]
            o = GpuStepOutcome(
                step=int(obj["step"]), windows=tuple(int(w) for w in obj["windows"]),
                accepted=tuple(int(a) for a in obj["accepted"]), credited=tuple(int(c) for c in obj["credited"]),
                bonus=int(obj["bonus"]), expected_accepted=float(obj["expected_accepted"]),
                stats=None if st is None else PolicyStats(int(st["extracts"]), int(st["inserts"]),
                                                          int(st["peak_queue"]), int(st["comparisons"])),
                completions=tuple((int(i), int(s)) for i, s in obj["completions"]), alpha_hat=float("nan"),
                tau=float(obj["tau"]))
            if int(obj["sent"]) != o.sent:
                raise ValueError(f"sent={obj['sent']} disagrees with windows {obj['windows']}")
            out.append(o)
        except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
            raise TraceSchemaError(f"{path}: line {lineno}: {exc}") from None
    steps = header.get("steps")
    if steps is not None and steps != len(out):
        raise TraceSchemaError(f"{path}: line {len(lines)}: header promises {steps} steps, found {len(out)} "
                               f"(file truncated?)")
    return out
