"""Helpers to load the committed golden fixtures (tests/golden/*.npz)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def colour_from_groups(d: dict) -> np.ndarray:
    """ColorGroups (groups indexed by colour) -> per-set colour array."""
    m = len(d["set_off"]) - 1
    col = np.full(m, -1, np.int32)
    goff = d["group_off"]
    for c in range(len(goff) - 1):
        col[d["group_sets"][goff[c]:goff[c + 1]]] = c
    assert (col >= 0).all()
    return col


def instance(d: dict):
    return (int(d["num_vertices"][0]), d["edge_u"].astype(np.uint32), d["edge_v"].astype(np.uint32),
            d["edge_w"].astype(np.float64))


def fos(d: dict):
    return d["set_off"].astype(np.uint64), d["set_vars"].astype(np.uint32)
