"""Builds libgomix_b200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2203_08680_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgomix_b200.so")
SOURCES = ["problem.cu", "gom.cu", "gom_univ.cu", "gom_univ_f64.cu", "gom_peer.cu", "gom_gen.cu", "gom_fi.cu", "engine.cu", "instances.cu", "linkage.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "gomix_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, probes: bool = False, variant: str = "",
          defines=()) -> str:
    """probes: an instrumented copy (-DGOMIX_PROBES: %globaltimer marks in
    the GOM kernels) as libgomix_b200_probes.so, loaded with
    GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so.
    variant/defines: an A/B copy built with extra -D flags as
    libgomix_b200_<variant>.so (same loading rule)."""
    tag = "probes" if probes else variant
    lib = LIB.replace(".so", f"_{tag}.so") if tag else LIB
    if not force and not tag and not _stale():
        return LIB
    objs = []
    build_dir = os.path.join(PKG, f"build_{tag}" if tag else "build")
    flags = FLAGS + (["-DGOMIX_PROBES"] if probes else []) + [f"-D{d}" for d in defines]
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(out)
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        with open(os.path.join(build_dir, os.path.basename(cmd[-3]) + ".ptxas.txt"), "w") as fh:
            fh.write(out)
    tmp = lib + ".tmp"
    subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
                    "-lcudart_static", "-ldl", "-lrt", "-lpthread"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2203_08680_b200.build [--force] [-v] [--probes] [--variant NAME -DMACRO ...]
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, probes="--probes" in sys.argv,
                variant=var, defines=defs))
