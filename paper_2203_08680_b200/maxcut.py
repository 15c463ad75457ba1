"""Max-Cut instances and linkage models (inputs of the GOM path).

Mirrors the reference's MaxCutInstance (maxcut.hpp:21-37), generate_torus
(maxcut.hpp:121-147), the edge-list format (maxcut.hpp:160-248) and the Fos
type (linkage.hpp:124-131).  Generators run in the product library's host code
(gomix_generate_*), so a torus equals the reference's for the same seed.
"""
from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass

import ctypes as C
from typing import Optional

import numpy as np

from . import _capi


@dataclass
class MaxCutInstance:
    num_vertices: int
    edge_u: np.ndarray  # uint32, u < v, sorted by (u, v), unique
    edge_v: np.ndarray
    edge_w: np.ndarray  # float64

    @property
    def num_edges(self) -> int:
        return len(self.edge_u)

    def integer_weights(self) -> bool:  # maxcut.hpp:32-36
        w = self.edge_w
        return bool(np.all(w == np.floor(w)) and np.all(np.abs(w) <= 9e15))

    def cut_value(self, genotype) -> float:  # maxcut.hpp:57-64 (left to right)
        g = np.asarray(genotype)
        cut = g[self.edge_u] != g[self.edge_v]
        total = 0.0
        for x in self.edge_w[cut]:
            total += float(x)
        return total

    def cut_values(self, genotypes: np.ndarray, chunk: int = 256) -> np.ndarray:
        """Vectorised cut values (exact for integer weights), chunk rows at a time."""
        g = np.asarray(genotypes)
        out = np.empty(g.shape[0], np.float64)
        for a in range(0, g.shape[0], chunk):
            cut = g[a:a + chunk, self.edge_u] != g[a:a + chunk, self.edge_v]
            out[a:a + chunk] = cut.astype(np.float64) @ self.edge_w
        return out

    def adjacency(self):
        """VIG adjacency (graybox.hpp:305-323) as a list of sorted arrays."""
        nbrs = [[] for _ in range(self.num_vertices)]
        for a, b in zip(self.edge_u.tolist(), self.edge_v.tolist()):
            nbrs[a].append(b)
            nbrs[b].append(a)
        return [np.array(sorted(x), np.uint32) for x in nbrs]

    def _struct(self):
        self._keep = (np.ascontiguousarray(self.edge_u, np.uint32), np.ascontiguousarray(self.edge_v, np.uint32),
                      np.ascontiguousarray(self.edge_w, np.float64))
        return _capi.Maxcut(self.num_vertices, len(self.edge_u), *(a.ctypes.data for a in self._keep))


def _weights(weights):
    if weights in ("unit", None) or weights[0] == "unit":
        return 0, 1, 1
    if weights[0] == "int":
        return 1, int(weights[1]), int(weights[2])
    if weights[0] == "real":
        return 2, 0, 0
    raise ValueError("weights: 'unit' | ('int', lo, hi) | ('real',)")


def generate_torus(width: int, height: int, weights=("int", 1, 10), seed: int = 1) -> MaxCutInstance:
    """maxcut.hpp:121-147: 2-D wrap-around grid, 2*width*height edges."""
    kind, lo, hi = _weights(weights)
    q = 2 * width * height
    eu, ev, ew = np.zeros(q, np.uint32), np.zeros(q, np.uint32), np.zeros(q, np.float64)
    _capi.check(_capi.lib().gomix_generate_torus(width, height, kind, lo, hi, seed, eu.ctypes.data,
                                                  ev.ctypes.data, ew.ctypes.data))
    return MaxCutInstance(width * height, eu, ev, ew)


def generate_regular(num_vertices: int, degree: int, weights=("real",), seed: int = 1) -> MaxCutInstance:
    """Random simple d-regular graph (BASELINE config C4)."""
    kind, lo, hi = _weights(weights)
    q = num_vertices * degree // 2
    eu, ev, ew = np.zeros(q, np.uint32), np.zeros(q, np.uint32), np.zeros(q, np.float64)
    _capi.check(_capi.lib().gomix_generate_regular(num_vertices, degree, kind, lo, hi, seed, eu.ctypes.data,
                                                    ev.ctypes.data, ew.ctypes.data))
    return MaxCutInstance(num_vertices, eu, ev, ew)


def save_edge_list(path: str, inst: MaxCutInstance) -> None:
    """maxcut.hpp:240-248: header, then 1-based "u v w"; integral weights as integers."""
    with open(path, "w") as fh:
        fh.write(f"{inst.num_vertices} {inst.num_edges}\n")
        for a, b, w in zip(inst.edge_u.tolist(), inst.edge_v.tolist(), inst.edge_w.tolist()):
            ws = str(int(w)) if w == math.floor(w) and abs(w) <= 9e15 else repr(float(w))
            fh.write(f"{a + 1} {b + 1} {ws}\n")


class ParseError(ValueError):
    """maxcut.hpp:149-158: a malformed edge list; `line` is the 1-based line
    the error was detected on (the message starts with "line N: ")."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


def _int_token(t: str) -> int:
    """A whole token read by istream >> long long: optional sign, digits."""
    if not re.fullmatch(r"[+-]?[0-9]+", t):
        raise ValueError(t)
    return int(t)


def load_edge_list(source) -> MaxCutInstance:
    """load_edge_list (maxcut.hpp:160-226): a "<num_vertices> <num_edges>"
    header, then one "<u> <v> <w>" line per edge, 1-based endpoints; blank
    lines and lines starting with '#' skipped.  Errors raise ParseError with
    the reference's line numbers (KATs: test_maxcut.cpp:182-201).  `source`
    is a path or a text stream."""
    fh = open(source) if isinstance(source, (str, bytes, os.PathLike)) else source
    try:
        lines = iter(fh)
        line_no = 0

        def next_payload():
            nonlocal line_no
            for line in lines:
                line_no += 1
                s = line.strip()
                if not s or s.startswith("#"):
                    continue
                return s
            return None

        head = next_payload()
        if head is None:
            raise ParseError(line_no, "missing header")
        parts = head.split()
        try:
            if len(parts) != 2:
                raise ValueError(head)
            nv, ne = _int_token(parts[0]), _int_token(parts[1])
            if nv < 1 or ne < 0:
                raise ValueError(head)
        except ValueError:
            raise ParseError(line_no, "malformed header, expected '<num_vertices> <num_edges>'") from None
        rows = []
        seen = set()
        while len(rows) < ne:
            s = next_payload()
            if s is None:
                raise ParseError(line_no, "fewer edge lines than the header declares")
            parts = s.split()
            try:
                if len(parts) != 3:
                    raise ValueError(s)
                u, v, w = _int_token(parts[0]), _int_token(parts[1]), float(parts[2])
                if not math.isfinite(w):  # istream >> double reads no inf / nan / overflow
                    raise ValueError(s)
            except ValueError:
                raise ParseError(line_no, "malformed edge line, expected '<u> <v> <w>'") from None
            if u < 1 or v < 1 or u > nv or v > nv:
                raise ParseError(line_no, "vertex index out of range")
            if u == v:
                raise ParseError(line_no, "self-loop")
            if not math.isfinite(w):
                raise ParseError(line_no, "non-finite weight")
            a, b = min(u, v) - 1, max(u, v) - 1
            if (a, b) in seen:
                raise ParseError(line_no, "duplicate edge")
            seen.add((a, b))
            rows.append((a, b, w))
        if next_payload() is not None:
            raise ParseError(line_no, "more edge lines than the header declares")
    finally:
        if fh is not source:
            fh.close()
    rows.sort(key=lambda r: (r[0], r[1]))
    u = np.array([r[0] for r in rows], np.uint32)
    v = np.array([r[1] for r in rows], np.uint32)
    return MaxCutInstance(nv, u, v, np.array([r[2] for r in rows], np.float64))


@dataclass
class Fos:
    """Family of linkage sets (linkage.hpp:124-131) in CSR form."""
    num_variables: int
    set_offset: np.ndarray  # uint64, num_sets + 1
    set_vars: np.ndarray    # uint32

    @property
    def num_sets(self) -> int:
        return len(self.set_offset) - 1

    def set(self, i: int) -> np.ndarray:
        return self.set_vars[self.set_offset[i]:self.set_offset[i + 1]]

    @staticmethod
    def from_sets(num_variables: int, sets) -> "Fos":
        off = np.zeros(len(sets) + 1, np.uint64)
        off[1:] = np.cumsum([len(s) for s in sets])
        vars_ = np.concatenate([np.asarray(s, np.uint32) for s in sets]) if sets else np.zeros(0, np.uint32)
        return Fos(num_variables, off, vars_)

    def _struct(self):
        self._keep = (np.ascontiguousarray(self.set_offset, np.uint64), np.ascontiguousarray(self.set_vars, np.uint32))
        return _capi.Fos(self.num_sets, self._keep[0].ctypes.data, self._keep[1].ctypes.data)


def univariate_fos(num_variables: int) -> Fos:
    """Singletons in variable order (the CLI's `univariate` = bound 1)."""
    return Fos(num_variables, np.arange(num_variables + 1, dtype=np.uint64),
               np.arange(num_variables, dtype=np.uint32))


def bounded_flt_fos(inst: MaxCutInstance, bound: Optional[int] = None, weighted: bool = False) -> Fos:
    """The reference's fixed linkage tree (build_fixed_model, model.hpp:31-52):
    UPGMA over the VIG similarity (or |w| with weighted=True), merged sets of
    at most `bound` variables (None: unbounded FLT).  Computed on sparse
    similarities (no n x n matrix), same sets in the same order."""
    if bound is not None and bound <= 0:
        raise ValueError("linkage: size bound must be positive")
    L = _capi.lib()
    eu = np.ascontiguousarray(inst.edge_u, np.uint32)
    ev = np.ascontiguousarray(inst.edge_v, np.uint32)
    ew = np.ascontiguousarray(inst.edge_w, np.float64)
    m, tv = C.c_uint64(), C.c_uint64()
    args = (inst.num_vertices, inst.num_edges, eu.ctypes.data, ev.ctypes.data, ew.ctypes.data, bound or 0,
            int(weighted))
    _capi.check(L.gomix_fos_bounded_flt(*args, C.byref(m), C.byref(tv), None, None))
    off = np.zeros(m.value + 1, np.uint64)
    vars_ = np.zeros(tv.value, np.uint32)
    _capi.check(L.gomix_fos_bounded_flt(*args, C.byref(m), C.byref(tv), off.ctypes.data, vars_.ctypes.data))
    return Fos(inst.num_vertices, off, vars_)


def neighbourhood_fos(inst: MaxCutInstance) -> Fos:
    """Set v = {v} U N(v), sorted (BASELINE config C2's 'neighbourhood FOS')."""
    nv = inst.num_vertices
    u = np.concatenate([inst.edge_u, inst.edge_v, np.arange(nv, dtype=np.uint32)])
    v = np.concatenate([inst.edge_v, inst.edge_u, np.arange(nv, dtype=np.uint32)])
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    off = np.zeros(nv + 1, np.uint64)
    np.add.at(off, u.astype(np.int64) + 1, 1)
    return Fos(nv, np.cumsum(off).astype(np.uint64), v.astype(np.uint32))
