"""CPU: the GPU-outcome trace writer/reader (paper_2502_15197_b200.trace_io) round-trips the reference's own JSONL
traces byte for byte (tests/golden/sim_trace_*.jsonl, written by tetris_sched.trace_io.write_trace) and rejects
malformed files the way trace_io.py:176-206 does."""
import pytest

from _sim_golden import PATH
from paper_2502_15197_b200.trace_io import TraceSchemaError, read_trace, write_trace

TRACES = sorted(PATH.parent.glob("sim_trace_*.jsonl"))


@pytest.mark.parametrize("path", TRACES, ids=[p.stem for p in TRACES])
def test_round_trip_is_byte_identical(path, tmp_path):
    outs = read_trace(path)
    assert len(outs) > 0
    write_trace(outs, tmp_path / "t.jsonl")
    assert (tmp_path / "t.jsonl").read_bytes() == path.read_bytes()


def test_schema_errors(tmp_path):
    bad = tmp_path / "b.jsonl"
    bad.write_text("")
    with pytest.raises(TraceSchemaError, match="line 1"):
        read_trace(bad)
    bad.write_text('{"schema": "other", "version": 1}\n')
    with pytest.raises(TraceSchemaError, match="line 1"):
        read_trace(bad)
    good = TRACES[0].read_text().splitlines()
    bad.write_text("\n".join(good[:-1]) + "\n")  # truncated
    with pytest.raises(TraceSchemaError, match="truncated"):
        read_trace(bad)
    lines = list(good)
    lines[2] = lines[2].replace('"sent": ', '"sent": 1')
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(TraceSchemaError, match="line 3"):
        read_trace(bad)
