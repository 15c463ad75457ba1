"""The forced-improvement restatement (oracle/fi_oracle.py) pinned to the
unmodified reference: with singleton groups (complete graph, univariate FOS)
and one flagged solution it must reproduce forced_improvement
(engine_serial.hpp:98-128) run by oracle/_ref/ref_driver's fi mode with the
set order that driver draws.  CPU only."""
import os
import tempfile

import numpy as np
import pytest

import paper_2203_08680_b200 as G
from oracle import fi_oracle as FO
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not os.path.exists(O.REF_DRIVER), reason="oracle/_ref not built")


@pytest.mark.parametrize("seed", range(1, 9))
def test_restatement_equals_reference_forced_improvement(seed):
    rs = np.random.RandomState(seed)
    m, n = 11, 8
    u, v = np.triu_indices(m, 1)
    w = rs.randint(-5, 10, len(u)).astype(np.float64)
    inst = G.MaxCutInstance(m, u.astype(np.uint32), v.astype(np.uint32), w)
    fos = G.univariate_fos(m)
    g = rs.randint(0, 2, (n, m)).astype(np.uint8)
    f = inst.cut_values(g)
    e = int(np.argmax(f))
    o = (e + 1 + seed) % n
    with tempfile.TemporaryDirectory() as d:
        edges, pop, out = (os.path.join(d, x) for x in ("g.txt", "pop.bin", "fi.bin"))
        G.save_edge_list(edges, inst)
        with open(pop, "wb") as fh:
            fh.write(np.array([n, m, o, e], np.int64).tobytes())
            fh.write(g.tobytes())
        ref = O.run_ref("fi", "--edges", edges, "--fos", "univariate", "--seed", str(seed), "--pop", pop, out=out)
    groups = [np.array([s], np.uint64) for s in range(m)]  # every set its own colour
    order = ref["set_order"].astype(np.int64)
    flags = np.zeros(n, np.uint8)
    flags[o] = 1
    rg, rf, _, _, calls, _ = FO.fi_pass(inst.edge_u, inst.edge_v, inst.edge_w, fos.set_offset, fos.set_vars,
                                        groups, order, g, f, e, f[e], flags)
    assert (rg[o] == ref["genotype"]).all()
    assert rf[o] == ref["fitness"][0]
    assert calls == int(ref["evaluator_calls"][0])
