"""The fixed linkage model (bounded) FLT built without the n x n similarity
matrix (csrc/linkage.cu) against the reference's learn_tree_upgma over
vig_similarity (linkage.hpp:133-264, model.hpp:31-52): identical sets in
identical order on every golden fixture the unmodified reference produced,
plus structural properties at BASELINE sizes where the dense reference
cannot run (10^6 variables)."""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from tests import golden_util as GU

CASES = [("bflt10_40x40", 10), ("bflt4_8x8", 4), ("col_torus40_bflt10", 10), ("col_torus10_bflt3", 3),
         ("col_torus10_bflt7", 7), ("col_reg64_bflt6", 6), ("col_reg50_bflt2", 2), ("col_torus7x5_flt", None),
         ("col_torus12x9_bflt16", 16)]


@pytest.mark.parametrize("name,bound", CASES)
def test_sparse_flt_equals_reference_upgma(name, bound):
    d = GU.load(name)
    nv, eu, ev, ew = GU.instance(d)
    inst = G.MaxCutInstance(nv, eu, ev, ew)
    fos = G.bounded_flt_fos(inst, bound)
    off, vars_ = GU.fos(d)
    assert fos.num_sets == len(off) - 1
    assert (fos.set_offset == off).all()
    assert (fos.set_vars == vars_).all()


def test_flt_at_c3_size():
    """10^6 variables (the dense reference needs 8 TB here): sizes within the
    bound, every variable in its singleton and in at least one merged set."""
    inst = G.generate_torus(1000, 1000, "unit", 1)
    fos = G.bounded_flt_fos(inst, 8)
    nv = inst.num_vertices
    sizes = np.diff(fos.set_offset.astype(np.int64))
    assert (sizes[:nv] == 1).all() and sizes.max() <= 8 and fos.num_sets < 2 * nv
    assert np.bincount(fos.set_vars[fos.set_offset[nv]:].astype(np.int64), minlength=nv).min() >= 1


def test_flt_structure():
    """300x300 torus, bound 8: a laminar family (every merged set is the
    union of two earlier sets), sets sorted, sizes within the bound, the full
    set never emitted."""
    inst = G.generate_torus(300, 300, "unit", 1)
    fos = G.bounded_flt_fos(inst, 8)
    nv = inst.num_vertices
    sizes = np.diff(fos.set_offset.astype(np.int64))
    assert (sizes[:nv] == 1).all() and (fos.set_vars[:nv] == np.arange(nv)).all()
    assert sizes.max() <= 8 and sizes.min() >= 1
    assert fos.num_sets < 2 * nv
    # laminar, built by merges: every merged set is the disjoint union of
    # exactly two earlier clusters (the latest sets holding its variables)
    latest = np.arange(nv, dtype=np.int64)  # singleton v is set v
    for i in range(nv, fos.num_sets):
        s = fos.set(i).astype(np.int64)
        assert (np.diff(s) > 0).all()
        parts = np.unique(latest[s])
        assert len(parts) == 2, i
        assert sizes[parts].sum() == len(s)
        latest[s] = i


def test_unbounded_flt_and_validation():
    inst = G.generate_torus(6, 6, "unit", 1)
    fos = G.bounded_flt_fos(inst)  # full tree: n singletons + n - 2 merges (root dropped)
    assert fos.num_sets == 2 * 36 - 2
    with pytest.raises(ValueError):
        G.bounded_flt_fos(inst, 0)


@pytest.mark.gpu
def test_bflt_model_runs_on_the_gpu_engine():
    """A bounded-FLT FOS on C2's torus through the GPU colouring and engine."""
    inst = G.generate_torus(100, 100, ("int", 1, 10), 1)
    fos = G.bounded_flt_fos(inst, 6)
    P = G.GpuProblem(inst, fos)
    E = G.GpuParallelEngine(P, 64, 1, mode="philox")
    for _ in range(3):
        E.run_generation()
    g, f = E.population()
    assert (inst.cut_values(g) == f).all()
