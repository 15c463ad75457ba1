"""Edge-list loader (maxcut.hpp:149-226) against the reference's own KATs:
parse errors carry the line they were detected on (test_maxcut.cpp:182-201),
comments/blank lines are skipped, and save -> load is canonical
(test_maxcut.cpp:203-215).  Host-only: the loader needs no GPU, the torus
generator runs in libgomix_b200.so's host code."""
import io

import numpy as np
import pytest

import paper_2203_08680_b200 as G

# test_maxcut.cpp:182-201, verbatim inputs and expected line numbers
KATS = [
    ("nonsense\n", 1),
    ("3\n", 1),
    ("3 2\n1 2 1\n1 2 2\n", 3),      # duplicate edge
    ("3 2\n1 1 1\n2 3 1\n", 2),      # self loop
    ("3 2\n1 4 1\n2 3 1\n", 2),      # vertex out of range
    ("3 2\n0 2 1\n2 3 1\n", 2),      # 1-based indices required
    ("3 3\n1 2 1\n2 3 1\n", 3),      # fewer edges than declared
    ("3 1\n1 2 1\n2 3 1\n", 3),      # more edges than declared
    ("3 2\n1 2\n2 3 1\n", 2),        # missing weight
]


@pytest.mark.parametrize("text,line", KATS)
def test_parse_errors_carry_line_numbers(text, line):
    with pytest.raises(G.ParseError) as e:
        G.load_edge_list(io.StringIO(text))
    assert e.value.line == line
    assert str(e.value).startswith(f"line {line}: ")


# beyond the KATs: outcomes checked against the reference's own loader
# (oracle/_ref/ref_driver color --edges FILE) when the fixtures were written
@pytest.mark.parametrize("text,line,what", [
    ("", 0, "missing header"),
    ("# only a comment\n\n", 2, "missing header"),
    ("0 0\n", 1, "malformed header"),
    ("3 -1\n", 1, "malformed header"),
    ("3 2 7\n", 1, "malformed header"),
    ("3 1\n1 2 nan\n", 2, "malformed edge line"),   # libstdc++ >> double reads no nan / inf
    ("3 1\n1 2 inf\n", 2, "malformed edge line"),
    ("3 1\n1 2 1e400\n", 2, "malformed edge line"),
    ("3 1\n1.0 2 1\n", 2, "malformed edge line"),
    ("3 1\n2 1 1\n# trailing comment\n\n", None, None),
    ("3 2\n1 2 1\n\n# gap\n3 2 5\n", None, None),
    ("3 2\n1 2 1\n2 1 5\n", 3, "duplicate edge"),     # (2,1) is (1,2) reversed
])
def test_parse_edge_cases(text, line, what):
    if what is None:
        inst = G.load_edge_list(io.StringIO(text))
        assert (np.diff(inst.edge_u.astype(np.int64)) >= 0).all()
        return
    with pytest.raises(G.ParseError) as e:
        G.load_edge_list(io.StringIO(text))
    assert e.value.line == line and what in str(e.value)


def test_float_weights_and_sorting():
    inst = G.load_edge_list(io.StringIO("# c\n3 2\n\n3 1 0.5\n1 2 -2\n"))
    assert inst.num_vertices == 3
    assert inst.edge_u.tolist() == [0, 0] and inst.edge_v.tolist() == [1, 2]
    assert inst.edge_w.tolist() == [-2.0, 0.5]


def test_save_load_round_trip_is_canonical(tmp_path):
    inst = G.generate_torus(4, 5, ("int", -9, 9), 77)
    p = tmp_path / "t.txt"
    G.save_edge_list(str(p), inst)
    back = G.load_edge_list(str(p))
    assert back.num_vertices == inst.num_vertices
    assert (back.edge_u == inst.edge_u).all() and (back.edge_v == inst.edge_v).all()
    assert (back.edge_w == inst.edge_w).all()
    p2 = tmp_path / "t2.txt"
    G.save_edge_list(str(p2), back)
    assert p.read_text() == p2.read_text()
