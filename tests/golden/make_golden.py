"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs oracle/_ref/ref_driver (the reference headers compiled by oracle/Makefile)
and stores its outputs as compressed .npz files next to this script.  Only
runnable where /root/reference exists (the build container); the fixtures
themselves travel with the repo and are what the GPU-box tests read.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

# (name, instance args, fos, n, seed, generations, keep full per-gen populations)
RUN_CASES = [
    ("c1_int", ["--torus", 10, 10, "--weights", "int:1:10", "--inst-seed", 1], "univariate", 32, 1, 20, True),
    ("c1_pm5", ["--torus", 10, 10, "--weights", "int:-5:5", "--inst-seed", 1], "univariate", 32, 3, 20, True),
    ("torus6_w", ["--torus", 6, 6, "--weights", "int:-3:5", "--inst-seed", 17], "univariate", 16, 91, 5, True),
    ("neigh12", ["--torus", 12, 12, "--weights", "int:1:10", "--inst-seed", 2], "neigh", 64, 5, 10, True),
    ("neigh_n40", ["--torus", 9, 7, "--weights", "int:-4:6", "--inst-seed", 4], "neigh", 40, 11, 8, True),
    ("bflt10_40x40", ["--torus", 40, 40, "--weights", "unit", "--inst-seed", 1], "bflt:10", 16, 7, 50, False),
    ("bflt4_8x8", ["--torus", 8, 8, "--weights", "int:1:9", "--inst-seed", 3], "bflt:4", 24, 2, 10, True),
    ("reg4_float", ["@reg", 60, 4, 21], "univariate", 32, 4, 10, True),
    ("reg3_float_neigh", ["@reg", 50, 3, 22], "neigh", 48, 6, 8, True),
    ("c2_small_gens", ["--torus", 100, 100, "--weights", "int:1:10", "--inst-seed", 1], "neigh", 64, 1, 2, False),
]

COLOR_CASES = [
    ("col_torus10_uni", ["--torus", 10, 10, "--weights", "unit"], "univariate"),
    ("col_torus10_neigh", ["--torus", 10, 10, "--weights", "unit"], "neigh"),
    ("col_torus100_neigh", ["--torus", 100, 100, "--weights", "unit"], "neigh"),
    ("col_torus7x5_uni", ["--torus", 7, 5, "--weights", "unit"], "univariate"),
    ("col_torus40_bflt10", ["--torus", 40, 40, "--weights", "unit"], "bflt:10"),
    ("col_reg8", ["@reg", 200, 8, 31], "univariate"),
    ("col_reg5odd", ["@reg", 64, 5, 32], "neigh"),
    # bounded / unbounded FLT (build_fixed_model over vig_similarity): pins
    # the sparse UPGMA of csrc/linkage.cu
    ("col_torus10_bflt3", ["--torus", 10, 10, "--weights", "unit"], "bflt:3"),
    ("col_torus10_bflt7", ["--torus", 10, 10, "--weights", "int:1:10"], "bflt:7"),
    ("col_reg64_bflt6", ["@reg", 64, 5, 33], "bflt:6"),
    ("col_reg50_bflt2", ["@reg", 50, 3, 34], "bflt:2"),
    ("col_torus7x5_flt", ["--torus", 7, 5, "--weights", "unit"], "flt"),
    ("col_torus12x9_bflt16", ["--torus", 12, 9, "--weights", "unit"], "bflt:16"),
]


# IMS runs (run_parallel with use_ims, run.hpp:72-82): (name, instance, fos,
# seed, base, subgenerations, extra termination args)
IMS_CASES = [
    ("ims_c1", ["--torus", 10, 10, "--weights", "int:1:10", "--inst-seed", 1], "univariate", 1, 16, 4,
     ["--max-evals", 3000]),
    ("ims_pm5", ["--torus", 10, 10, "--weights", "int:-5:5", "--inst-seed", 1], "univariate", 3, 8, 2,
     ["--max-evals", 4000]),
    ("ims_neigh", ["--torus", 12, 12, "--weights", "int:1:10", "--inst-seed", 2], "neigh", 5, 16, 4,
     ["--max-evals", 1500]),
    ("ims_target", ["--torus", 8, 8, "--weights", "unit", "--inst-seed", 1], "univariate", 2, 4, 4,
     ["--target", 128, "--max-evals", 100000]),
]


# Full-size replay fixtures (ref_driver run --light: per-generation packed
# populations are hashed here, fitness / elitist / calls / counters / traces
# kept whole): (name, torus w, h, weights, inst seed, fos, n, seed, gens).
# These pin the bit-sliced univariate kernels (gom_univ_tt_kernel,
# gom_univ_sliced_kernel) that run the BASELINE configs C3 and C5.
LIGHT_CASES = [
    ("c3_full", 1000, 1000, "int:1:10", 1, "univariate", 128, 1, 3),
    ("c5_n16", 316, 316, "int:1:10", 1, "univariate", 16, 2, 6),
    ("c5_n1024", 316, 316, "int:1:10", 1, "univariate", 1024, 3, 2),
    ("c1_long", 10, 10, "int:1:10", 1, "univariate", 32, 4, 60),
    ("c3_pm", 200, 150, "int:-6:9", 5, "univariate", 100, 9, 4),
]


def array_hash(*arrays) -> np.uint64:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest()[:8], np.uint64)[0]


def packed_hash(packed: np.ndarray) -> np.uint64:
    """Hash of one population as numpy.packbits of its (n, l) genotype bytes."""
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(packed).tobytes()).digest()[:8], np.uint64)[0]


# Float weights at BASELINE C4 size: random d-regular graphs from this repo's
# generator (the reference has none), handed to the reference as an edge-list
# file: (name, vertices, degree, generator seed, fos, n, seed, gens).
LIGHT_REGULAR_CASES = [
    ("c4_d4", 100000, 4, 4, "univariate", 128, 5, 2),
    ("c4_d8_small", 20000, 8, 8, "univariate", 64, 6, 3),
]


def make_light(cases):
    with tempfile.TemporaryDirectory() as tmp:
        for case in cases:
            name = case[0]
            if case in LIGHT_REGULAR_CASES:
                _, nv_, deg, gseed, fos, n, seed, gens = case
                import paper_2203_08680_b200 as G

                inst = G.generate_regular(nv_, deg, ("real",), seed=gseed)
                path = os.path.join(tmp, name + ".txt")
                G.save_edge_list(path, inst)
                src = ["--edges", path]
                w = h = iseed = 0
                weights = "real"
            else:
                _, w, h, weights, iseed, fos, n, seed, gens = case
                src = ["--torus", w, h, "--weights", weights, "--inst-seed", iseed]
            out = os.path.join(tmp, name + ".bin")
            d = O.run_ref("run", *src, "--fos", fos, "--n", n, "--seed", seed, "--gens", gens,
                          "--workers", os.cpu_count() or 4, "--light", out=out, timeout=7200)
            nv = int(d["num_vertices"][0])
            per = (n * nv + 7) // 8
            packed = d["packed"].reshape(gens, per)
            f = {"torus": np.array([w, h], np.uint64), "weights": np.array([weights]),
                 "regular": np.array(case[1:4] if case in LIGHT_REGULAR_CASES else [0, 0, 0], np.uint64),
                 "inst_seed": np.array([iseed], np.uint64), "fos_kind": np.array([fos]),
                 "n": np.array([n], np.uint64), "seed": np.array([seed], np.uint64),
                 "gens": np.array([gens], np.uint64), "num_vertices": d["num_vertices"],
                 "edges_hash": np.array([array_hash(d["edge_u"].astype(np.uint32), d["edge_v"].astype(np.uint32),
                                                    d["edge_w"].astype(np.float64))], np.uint64),
                 "group_off": d["group_off"],
                 "group_sets_hash": np.array([array_hash(d["group_sets"].astype(np.uint64))], np.uint64),
                 "init_hash": np.array([packed_hash(d["init_packed"])], np.uint64),
                 "init_fitness": d["init_fitness"], "init_elitist": d["init_elitist"],
                 "init_calls": d["init_calls"],
                 "pop_hash": np.array([packed_hash(p) for p in packed], np.uint64),
                 "fitness": d["fitness"], "elitist": d["elitist"], "calls": d["calls"],
                 "counter_steps": d["counter_steps"], "counter_calls": d["counter_calls"],
                 "trace_fitness": d["trace_fitness"], "trace_evals": d["trace_evals"],
                 "trace_generation": d["trace_generation"]}
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **f)
            print(f"{name}: nv={nv} groups={len(d['group_off']) - 1} best={d['elitist'][-1]} "
                  f"trace={len(d['trace_fitness'])}", flush=True)


def random_regular(nv: int, d: int, seed: int):
    """Random d-regular simple graph (configuration-model pairing, redrawn on
    self-loops/duplicates) with fp64 weights uniform in [0, 1).  The reference
    has no d-regular generator; this one only has to be
    deterministic, since fixtures store the edge list itself."""
    rs = np.random.RandomState(seed)
    assert nv * d % 2 == 0
    while True:
        stubs = np.repeat(np.arange(nv), d)
        rs.shuffle(stubs)
        a, b = stubs[0::2], stubs[1::2]
        u, v = np.minimum(a, b), np.maximum(a, b)
        if (u == v).any():
            continue
        key = u.astype(np.int64) * nv + v
        if len(np.unique(key)) != len(key):
            continue
        order = np.lexsort((v, u))
        w = rs.random_sample(len(u))
        return nv, u[order].astype(np.uint32), v[order].astype(np.uint32), w


def write_edge_list(path, nv, u, v, w):
    """maxcut.hpp:160-226 format (1-based, shortest round-trip floats)."""
    with open(path, "w") as fh:
        fh.write(f"{nv} {len(u)}\n")
        for a, b, x in zip(u, v, w):
            fh.write(f"{a + 1} {b + 1} {repr(float(x))}\n")


def instance_args(spec, tmp):
    if spec and spec[0] == "@reg":
        nv, u, v, w = random_regular(spec[1], spec[2], spec[3])
        path = os.path.join(tmp, f"reg_{spec[1]}_{spec[2]}_{spec[3]}.txt")
        write_edge_list(path, nv, u, v, w)
        return ["--edges", path]
    return [str(x) for x in spec]


def pop_hash(g: np.ndarray) -> np.uint64:
    return np.frombuffer(hashlib.sha256(g.tobytes()).digest()[:8], np.uint64)[0]


def main():
    with tempfile.TemporaryDirectory() as tmp:
        for name, inst, fos, n, seed, gens, full in RUN_CASES:
            out = os.path.join(tmp, name + ".bin")
            d = O.run_ref("run", *instance_args(inst, tmp), "--fos", fos, "--n", n, "--seed", seed,
                          "--gens", gens, "--workers", 3, out=out)
            d["n"] = np.array([n], np.uint64)
            d["seed"] = np.array([seed], np.uint64)
            d["gens"] = np.array([gens], np.uint64)
            d["fos_kind"] = np.array([fos])
            nv = int(d["num_vertices"][0])
            pops = d["genotypes"].reshape(gens, n, nv)
            d["pop_hash"] = np.array([pop_hash(p) for p in pops], np.uint64)
            if not full:
                d["final_genotypes"] = pops[-1].ravel().copy()
                for key in ("genotypes", "donor", "delta", "present", "accept"):
                    d.pop(key)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
            print(f"{name}: nv={nv} groups={len(d['group_off']) - 1} "
                  f"best={d['elitist'][-1]} trace={len(d['trace_fitness'])}")
        for name, inst, fos, seed, base, sub, term in IMS_CASES:
            r = json.loads(O.run_ref("ims", *instance_args(inst, tmp), "--fos", fos, "--seed", seed, "--ims",
                                     "--ims-base", base, "--ims-sub", sub, "--workers", 2, *term))
            tr = np.array(r["trace"], np.float64).reshape(-1, 3)
            d = {"best": np.array([r["best"]]), "reason": np.array([r["reason"]]),
                 "evaluations": np.array([r["evaluations"]]), "generations": np.array([r["generations"]]),
                 "populations": np.array([r["populations"]]), "trace_evals": tr[:, 1], "trace_fitness": tr[:, 2],
                 "seed": np.array([seed], np.uint64), "base": np.array([base]), "sub": np.array([sub]),
                 "fos_kind": np.array([fos]), "term": np.array([str(x) for x in term])}
            d.update(O.run_ref("color", *instance_args(inst, tmp), "--fos", fos,
                               out=os.path.join(tmp, name + ".bin")))
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
            print(f"{name}: best={r['best']} reason={r['reason']} pops={r['populations']} trace={len(tr)}")
        for name, inst, fos in COLOR_CASES:
            out = os.path.join(tmp, name + ".bin")
            d = O.run_ref("color", *instance_args(inst, tmp), "--fos", fos, out=out)
            d["fos_kind"] = np.array([fos])
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
            print(f"{name}: sets={len(d['set_off']) - 1} groups={len(d['group_off']) - 1} "
                  f"lmig_edges={int(d['lmig_edges'][0])}")


if __name__ == "__main__":
    if "--light" in sys.argv[1:]:
        names = [a for a in sys.argv[1:] if not a.startswith("--")]
        make_light([c for c in LIGHT_CASES + LIGHT_REGULAR_CASES if not names or c[0] in names])
    else:
        main()
