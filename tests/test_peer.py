"""The peer transport across PROCESSES (gom_peer.cuh, gomix_gpu_peer_export /
gomix_gpu_peer_connect): two ranks of one sharded population, one process
each, exchanging through CUDA IPC mappings of each other's exchange block —
here both on cuda:0 (gpurun gives one GPU; IPC works within a device), on an
8-GPU box over NVLink.  No NCCL: the GOM kernels' last CTAs publish, wait for
the other rank and run the global elitist scan themselves.  The result must
be bit-identical to one engine holding the whole population.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2203_08680_b200 as G

pytestmark = pytest.mark.gpu


def _problem(shape):
    inst = G.generate_torus(shape[0], shape[1], ("int", -3, 9), 5)
    return inst, G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))


def _rank(rank, world, port, shape, n, gens, q, queued=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst, P = _problem(shape)
        E = G.GpuParallelEngine(P, n, 11, mode="philox", rank=rank, world_size=world, transport="peer")
        if queued:  # the CUDA-graph path: device group order, no host sync between generations
            for _ in range(gens):
                E.run_generation_async()
            E.synchronize()
        else:
            for _ in range(gens):
                E.run_generation()
        g, f = E.population()
        eg, ef = E.elitist()  # collective: the owner's snapshot over peer memory
        _, steps, calls = E.group_counters()
        q.put((rank, g, f, eg, ef, steps, calls, E.generation(), None))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, None, None, None, None, None, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,n,gens,queued", [((24, 20), 128, 4, False), ((100, 100), 256, 3, False),
                                                 ((1000, 1000), 128, 3, True)])
def test_two_processes_peer_transport_equal_single_engine(shape, n, gens, queued):
    """queued: BASELINE C3 strong-scaled over 2 processes, generations queued
    as CUDA graphs (presence maps + device group order + one GOM launch per
    group, exchanges inside the kernels) — what bench.py --gpus N times."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 90 + (7 if queued else 0)
    procs = [ctx.Process(target=_rank, args=(r, world, port, shape, n, gens, q, queued)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        r = q.get(timeout=600)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        assert out[r][-1] is None, out[r][-1]
    inst, P = _problem(shape)
    if queued:  # the same graph path on one GPU
        E = G.GpuParallelEngine(P, n, 11, mode="philox")
        for _ in range(gens):
            E.run_generation_async()
        E.synchronize()
    else:
        E = G.GpuParallelEngine(P, n, 11, mode="philox", per_group_kernels=True, lane_per_solution=True)
        E.set_timing(True)  # launch by launch with the host group order, like the sharded path
        for _ in range(gens):
            E.run_generation()
    g, f = E.population()
    half = n // world
    for r in range(world):
        _, gr, fr, eg, ef, steps, calls, gen, _ = out[r]
        assert (gr == g[r * half:(r + 1) * half]).all()
        assert (fr == f[r * half:(r + 1) * half]).all()
        assert ef == E.elitist_fitness and (eg == E.elitist()[0]).all()
        assert gen == gens
        _, st1, ca1 = E.group_counters()
        assert (steps == st1).all() and (calls == ca1).all()
