"""ctypes view of the oracle restatement (oracle/gomix_oracle.c) and a reader for
oracle/_ref/ref_driver's named-array dumps.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu-baseline / --impl reference legs of bench.py — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mt_state_size.restype = C.c_size_t
        L.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_stream_init.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_mt_next.restype = C.c_uint64
        L.orc_mt_next.argtypes = [C.c_void_p]
        L.orc_uniform_index.restype = C.c_uint64
        L.orc_uniform_index.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_permutation.argtypes = [C.c_void_p, _u64p, C.c_uint64]
        L.orc_generate_torus.restype = C.c_int
        L.orc_generate_torus.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int64, C.c_int64,
                                         C.c_uint64, _u32p, _u32p, _f64p]
        L.orc_color_sets.restype = C.c_int64
        L.orc_color_sets.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p, C.c_uint64,
                                     _u64p, _u32p, _i32p, C.POINTER(C.c_uint64)]
        L.orc_engine_create.restype = C.c_void_p
        L.orc_engine_create.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p, C.c_uint64,
                                        _u64p, _u32p, C.c_void_p, C.c_uint64, C.c_uint64,
                                        C.c_void_p]
        L.orc_engine_set_termination.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int,
                                                 C.c_double, C.c_int, C.c_int64]
        L.orc_engine_run_generation.restype = C.c_int
        L.orc_engine_run_generation.argtypes = [C.c_void_p]
        L.orc_engine_offer_elitist.argtypes = [C.c_void_p, _u8p, C.c_double]
        for name, rt in (("orc_engine_num_groups", C.c_uint64), ("orc_engine_generation", C.c_int64),
                         ("orc_engine_stop_reason", C.c_int), ("orc_engine_evaluator_calls", C.c_uint64),
                         ("orc_engine_exact", C.c_int)):
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p]
        L.orc_engine_population.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_engine_elitist.restype = C.c_double
        L.orc_engine_elitist.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_engine_group.restype = C.c_uint64
        L.orc_engine_group.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_engine_group_fp.restype = C.c_uint64
        L.orc_engine_group_fp.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_engine_counters.argtypes = [C.c_void_p, _u64p, _u64p]
        L.orc_engine_last_groups.restype = C.c_uint64
        L.orc_engine_last_groups.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_engine_last_batch.argtypes = [C.c_void_p, C.c_uint64, _i32p, _f64p, _u8p, _u8p]
        L.orc_engine_trace.restype = C.c_uint64
        L.orc_engine_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_engine_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def mix64(x: int) -> int:
    return lib().orc_mix64(x)


class MT64:
    """std::mt19937_64 (raw seed) or RngStream (seed passed through mix64)."""

    def __init__(self, seed: int, stream: bool = True):
        self._buf = C.create_string_buffer(lib().orc_mt_state_size())
        (lib().orc_stream_init if stream else lib().orc_mt_seed)(self._buf, seed)

    def next_u64(self) -> int:
        return lib().orc_mt_next(self._buf)

    def uniform_index(self, n: int) -> int:
        return lib().orc_uniform_index(self._buf, n)

    def permutation(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        lib().orc_permutation(self._buf, out, n)
        return out


def generate_torus(width: int, height: int, weights=("int", 1, 10), seed: int = 1):
    """maxcut.hpp:121-147 restated; returns (nv, eu, ev, ew)."""
    q = 2 * width * height
    eu = np.zeros(q, np.uint32)
    ev = np.zeros(q, np.uint32)
    ew = np.zeros(q, np.float64)
    kind = 0 if weights == "unit" or weights[0] == "unit" else 1
    lo, hi = (1, 1) if kind == 0 else (weights[1], weights[2])
    rc = lib().orc_generate_torus(width, height, kind, lo, hi, seed, eu, ev, ew)
    if rc != 0:
        raise ValueError(f"torus generation failed ({rc})")
    return width * height, eu, ev, ew


def color_sets(nv, eu, ev, ew, set_off, set_vars):
    m = len(set_off) - 1
    colour = np.zeros(m, np.int32)
    ne = C.c_uint64(0)
    k = lib().orc_color_sets(nv, len(eu), np.ascontiguousarray(eu, np.uint32),
                             np.ascontiguousarray(ev, np.uint32), np.ascontiguousarray(ew, np.float64),
                             m, np.ascontiguousarray(set_off, np.uint64),
                             np.ascontiguousarray(set_vars, np.uint32), colour, C.byref(ne))
    return int(k), colour, int(ne.value)


STOP_REASONS = {0: "none", 1: "evaluation-budget", 2: "wall-clock", 3: "target-reached",
                4: "generation-limit"}


class OracleEngine:
    """ParallelEngine (engine_parallel.hpp:255-368) restated in C."""

    def __init__(self, nv, eu, ev, ew, set_off, set_vars, n, seed, colour=None, genotypes=None):
        L = lib()
        self.nv, self.n = int(nv), int(n)
        self._keep = [np.ascontiguousarray(eu, np.uint32), np.ascontiguousarray(ev, np.uint32),
                      np.ascontiguousarray(ew, np.float64), np.ascontiguousarray(set_off, np.uint64),
                      np.ascontiguousarray(set_vars, np.uint32)]
        col = None if colour is None else np.ascontiguousarray(colour, np.int32)
        gen = None if genotypes is None else np.ascontiguousarray(genotypes, np.uint8)
        self._keep += [col, gen]
        self.h = L.orc_engine_create(nv, len(eu), *self._keep[:3], len(set_off) - 1,
                                     self._keep[3], self._keep[4],
                                     None if col is None else col.ctypes.data, n, seed,
                                     None if gen is None else gen.ctypes.data)
        if not self.h:
            raise ValueError("oracle engine: invalid arguments")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_engine_destroy(self.h)
            self.h = None

    def set_termination(self, max_evaluations=None, target=None, max_generations=None):
        lib().orc_engine_set_termination(self.h, max_evaluations is not None, max_evaluations or 0.0,
                                         target is not None, target or 0.0,
                                         max_generations is not None, max_generations or 0)

    def run_generation(self) -> bool:
        return bool(lib().orc_engine_run_generation(self.h))

    def offer_elitist(self, genotype, fitness):
        lib().orc_engine_offer_elitist(self.h, np.ascontiguousarray(genotype, np.uint8), fitness)

    @property
    def num_groups(self):
        return int(lib().orc_engine_num_groups(self.h))

    @property
    def generation(self):
        return int(lib().orc_engine_generation(self.h))

    @property
    def stop_reason(self):
        return STOP_REASONS[lib().orc_engine_stop_reason(self.h)]

    @property
    def evaluator_calls(self):
        return int(lib().orc_engine_evaluator_calls(self.h))

    def population(self):
        g = np.zeros((self.n, self.nv), np.uint8)
        f = np.zeros(self.n, np.float64)
        lib().orc_engine_population(self.h, g.ctypes.data, f.ctypes.data)
        return g, f

    def elitist(self):
        g = np.zeros(self.nv, np.uint8)
        f = lib().orc_engine_elitist(self.h, g.ctypes.data)
        return g, f

    def group(self, c):
        size = lib().orc_engine_group(self.h, c, None, None)
        ids = np.zeros(size, np.uint64)
        off = np.zeros(size + 1, np.uint64)
        lib().orc_engine_group(self.h, c, ids.ctypes.data, off.ctypes.data)
        fp = np.zeros(int(off[-1]), np.uint64)
        lib().orc_engine_group_fp(self.h, c, fp.ctypes.data)
        return ids, off, fp

    def counters(self):
        k = self.num_groups
        s = np.zeros(k, np.uint64)
        c = np.zeros(k, np.uint64)
        lib().orc_engine_counters(self.h, s, c)
        return s, c

    def last_batches(self):
        """[(group id, donor, delta, present, accept)] of the last generation, each
        shaped (n, |G|) like GroupBatch (engine_parallel.hpp:62-97)."""
        cnt = lib().orc_engine_last_groups(self.h, None)
        ids = np.zeros(cnt, np.uint64)
        lib().orc_engine_last_groups(self.h, ids.ctypes.data)
        out = []
        for slot, gi in enumerate(ids):
            size = lib().orc_engine_group(self.h, int(gi), None, None)
            pairs = self.n * size
            d = np.zeros(pairs, np.int32)
            de = np.zeros(pairs, np.float64)
            p = np.zeros(pairs, np.uint8)
            a = np.zeros(pairs, np.uint8)
            lib().orc_engine_last_batch(self.h, slot, d, de, p, a)
            out.append((int(gi), d.reshape(self.n, size), de.reshape(self.n, size),
                        p.reshape(self.n, size), a.reshape(self.n, size)))
        return out

    def trace(self):
        cnt = lib().orc_engine_trace(self.h, None, None, None)
        f = np.zeros(cnt, np.float64)
        c = np.zeros(cnt, np.uint64)
        g = np.zeros(cnt, np.int64)
        lib().orc_engine_trace(self.h, f.ctypes.data, c.ctypes.data, g.ctypes.data)
        return f, c, g


_DT = {"Q": np.uint64, "d": np.float64, "B": np.uint8, "i": np.int32}


def read_dump(path: str) -> dict:
    """Parse a ref_driver named-array dump into {name: ndarray}."""
    out = {}
    with open(path, "rb") as fh:
        data = fh.read()
    pos = 0
    while pos < len(data):
        (ln,) = np.frombuffer(data, np.uint32, 1, pos)
        pos += 4
        name = data[pos:pos + int(ln)].decode()
        pos += int(ln)
        code = chr(data[pos])
        pos += 1
        (cnt,) = np.frombuffer(data, np.uint64, 1, pos)
        pos += 8
        dt = np.dtype(_DT[code])
        out[name] = np.frombuffer(data, dt, int(cnt), pos).copy()
        pos += int(cnt) * dt.itemsize
    return out


def run_ref(mode: str, *args: str, out: str | None = None, timeout: float = 600):
    """Run oracle/_ref/ref_driver; returns the parsed dump (run/color) or stdout."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError("oracle/_ref/ref_driver not built (needs /root/reference)")
    cmd = [REF_DRIVER, mode, *map(str, args)]
    if out is not None:
        cmd += ["--out", out]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    if res.returncode != 0:
        raise RuntimeError(f"ref_driver failed ({res.returncode}): {res.stderr}")
    return read_dump(out) if out is not None else res.stdout
