"""CSV traces (trace_io.hpp): byte-identical to the reference's CsvTraceWriter
on a fixture it wrote (tests/golden/trace_ref.csv, from
tests/golden/make_trace_ref.cpp), lossless round trip, parser errors."""
import io
import os

import pytest

import paper_2203_08680_b200 as G

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "trace_ref.csv")


def test_writer_matches_reference_bytes():
    ref = open(GOLDEN).read()
    rows = G.parse_trace(io.StringIO(ref))
    out = io.StringIO()
    w = G.CsvTraceWriter(out, 0.5)
    for r in rows[:19]:                      # improvements: always written
        w.improvement(r)
    for i in range(6):                       # boundaries: 0.5 s heartbeat
        w.boundary(G.TraceRecord(10.0 + 0.2 * i, 50.0 + i, 100 + i, 1, 9.0))
    assert out.getvalue() == ref


@pytest.mark.parametrize("x,s", [(0.0, "0"), (1110.0, "1110"), (1e-05, "1e-05"), (1e16, "1e+16"),
                                 (123456.0, "123456"), (1e15, "1e+15"), (0.1, "0.1"), (-3.5, "-3.5"),
                                 (1428571428571428.5, "1428571428571428.5"), (2.5e-300, "2.5e-300")])
def test_format_double_like_to_chars(x, s):
    assert G.format_double(x) == s
    assert float(s) == x


def test_parse_errors_and_monotone():
    with pytest.raises(ValueError):
        G.parse_trace(io.StringIO("bad header\n"))
    with pytest.raises(ValueError):
        G.parse_trace(io.StringIO(G.TRACE_HEADER + "\n1,2,3,4\n"))
    with pytest.raises(ValueError):
        G.parse_trace(io.StringIO(G.TRACE_HEADER + "\n1,2,x,4,5\n"))
    rows = G.parse_trace(io.StringIO(G.TRACE_HEADER + "\n\n0.5,1,0,1,10\n1,2,1,1,12\n"))
    assert len(rows) == 2 and G.trace_monotone(rows)
    assert not G.trace_monotone(rows[::-1])
