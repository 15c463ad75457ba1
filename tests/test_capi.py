"""CPU-side checks of the drop-in boundary: libgomix_b200.so loads, exports every
symbol include/gomix_gpu.h declares, validates inputs like the reference
(std::invalid_argument -> GOMIX_E_INVALID) and fails loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

import paper_2203_08680_b200 as G
from paper_2203_08680_b200 import _capi
from tests import golden_util as GU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gomix_gpu.h")).read()
    return sorted(set(re.findall(r"^GOMIX_API\s+[\w\s\*]+?\b(gomix_\w+)\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    assert "gomix_gpu_run_generation" in syms and "gomix_gpu_problem_create" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_capi.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_capi._SIGNATURES) >= set(declared_symbols())


def test_abi_version():
    assert _capi.lib().gomix_gpu_abi_version() == 1


def test_torus_generator_equals_reference_instance():
    for name, w in (("c1_int", ("int", 1, 10)), ("c1_pm5", ("int", -5, 5))):
        d = GU.load(name)
        t = G.generate_torus(10, 10, w, 1)
        assert (t.edge_u == d["edge_u"]).all() and (t.edge_v == d["edge_v"]).all()
        assert (t.edge_w == d["edge_w"]).all()
    d = GU.load("bflt10_40x40")
    t = G.generate_torus(40, 40, "unit", 1)
    assert (t.edge_u == d["edge_u"]).all() and (t.edge_w == 1.0).all()


def test_regular_generator_is_simple_and_regular():
    for nv, deg in ((100, 3), (1000, 4), (500, 8), (64, 5)):
        g = G.generate_regular(nv, deg, ("real",), seed=nv + deg)
        assert g.num_edges == nv * deg // 2
        assert (g.edge_u < g.edge_v).all()
        key = g.edge_u.astype(np.int64) * nv + g.edge_v
        assert (np.diff(key) > 0).all()  # sorted, unique
        d = np.bincount(np.concatenate([g.edge_u, g.edge_v]), minlength=nv)
        assert (d == deg).all()
        assert ((g.edge_w >= 0) & (g.edge_w < 1)).all()


def test_neighbourhood_fos():
    t = G.generate_torus(5, 4, "unit", 1)
    f = G.neighbourhood_fos(t)
    assert f.num_sets == 20
    assert f.set(0).tolist() == [0, 1, 4, 5, 15]
    for i in range(20):
        s = f.set(i)
        assert (np.diff(s.astype(np.int64)) > 0).all() and i in s and len(s) == 5


def test_edge_list_roundtrip(tmp_path):
    g = G.generate_regular(40, 3, ("real",), seed=5)
    p = tmp_path / "g.txt"
    G.save_edge_list(str(p), g)
    h = G.load_edge_list(str(p))
    assert (h.edge_u == g.edge_u).all() and (h.edge_v == g.edge_v).all() and (h.edge_w == g.edge_w).all()


def _problem_status(inst, fos):
    h = C.c_void_p()
    return _capi.lib().gomix_gpu_problem_create(C.byref(inst._struct()), C.byref(fos._struct()), None, -1,
                                                C.byref(h))


@pytest.mark.parametrize("case", ["unsorted", "loop", "range", "nan", "emptyset", "bigset", "unsortedset"])
def test_invalid_inputs_are_rejected_before_any_device_work(case):
    t = G.generate_torus(4, 4, "unit", 1)
    fos = G.univariate_fos(16)
    if case == "unsorted":
        t.edge_u, t.edge_v = t.edge_u[::-1].copy(), t.edge_v[::-1].copy()
    elif case == "loop":
        t.edge_v = t.edge_v.copy()
        t.edge_v[0] = t.edge_u[0]
    elif case == "range":
        t.num_vertices = 10
    elif case == "nan":
        t.edge_w = t.edge_w.copy()
        t.edge_w[3] = np.nan
    elif case == "emptyset":
        fos = G.Fos(16, np.array([0, 0] + list(range(1, 17)), np.uint64), np.arange(16, dtype=np.uint32))
    elif case == "bigset":
        t = G.generate_torus(10, 10, "unit", 1)
        fos = G.Fos.from_sets(100, [list(range(65))] + [[v] for v in range(65, 100)])
    elif case == "unsortedset":
        fos = G.Fos.from_sets(16, [[1, 0]] + [[v] for v in range(2, 16)])
    assert _problem_status(t, fos) == _capi.GOMIX_E_INVALID
    assert _capi.lib().gomix_gpu_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    t = G.generate_torus(4, 4, "unit", 1)
    with pytest.raises(_capi.GomixError) as e:
        G.GpuProblem(t, G.univariate_fos(16))
    assert e.value.status in (_capi.GOMIX_E_CUDA, _capi.GOMIX_E_OOM)


def test_null_arguments():
    L = _capi.lib()
    assert L.gomix_gpu_engine_destroy(None) == 0  # delete nullptr is a no-op
    assert L.gomix_gpu_run_generation(None, None, None) == _capi.GOMIX_E_INVALID
    assert L.gomix_gpu_problem_info(None, None) == _capi.GOMIX_E_INVALID


def test_flag_constants_match_the_header():
    """The Python mirror's engine flags are the header's GOMIX_FLAG_* values."""
    import re

    hdr = open(os.path.join(ROOT, "include", "gomix_gpu.h")).read()
    vals = {m.group(1): 1 << int(m.group(2)) for m in re.finditer(r"GOMIX_FLAG_(\w+)\s*=\s*1u\s*<<\s*(\d+)", hdr)}
    from paper_2203_08680_b200 import _capi as K
    for name, v in vals.items():
        assert getattr(K, "FLAG_" + name) == v, name
    assert "FORCED_IMPROVEMENT" in vals and "NO_TRUTH_TABLE" in vals
