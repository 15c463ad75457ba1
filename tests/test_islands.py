"""Multi-GPU IMS (paper_2203_08680_b200/islands.py).

CPU (gloo, world size 2 and 3): the collective best exchange — max fitness,
lowest owning rank broadcasts its genotype once per improvement, stop flags
propagate.  GPU: a single-rank island run reaches the target like run_gpu.
"""
import math
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2203_08680_b200 as G
from paper_2203_08680_b200.islands import BestExchange, run_islands


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = BestExchange(8)
    geno = lambda: np.full(8, rank, np.uint8)  # noqa: E731
    out = []
    # round 1: rank 1 (and in world 3 also rank 2) hold the best 5.0 -> owner 1
    fits = {0: 3.0, 1: 5.0, 2: 5.0}
    out.append(ex.exchange(fits[rank], False, geno))
    # round 2: nobody improved -> no genotype moves
    out.append(ex.exchange(fits[rank], False, geno))
    # round 3: rank 0 improves to 7 and is stopped -> genotype of rank 0, global stop
    out.append(ex.exchange(7.0 if rank == 0 else fits[rank], rank == 0, geno))
    # round 4: a rank without any best yet (None) still takes part
    out.append(ex.exchange(None if rank == world - 1 else (7.0 if rank == 0 else 5.0), False, geno))
    rows = ex.gather({"rank": rank})
    dist.destroy_process_group()
    q.put((rank, [(f, s, None if g is None else g.tolist()) for f, s, g in out], rows))


@pytest.mark.parametrize("world", [2, 3])
def test_best_exchange_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 500 + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (o, rows)) for r, o, rows in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        out, rows = res[rank]
        assert out[0] == (5.0, False, [1] * 8)          # lowest owning rank broadcast
        assert out[1] == (5.0, False, None)             # nothing new: no broadcast
        assert out[2] == (7.0, True, [0] * 8)           # improvement + stop from rank 0
        assert out[3][0] == 7.0 and out[3][2] is None   # the max stays; nothing re-sent
        assert rows == [{"rank": r} for r in range(world)]


@pytest.mark.gpu
def test_single_rank_islands_reach_target():
    inst = G.generate_torus(10, 10, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(100))
    target = float(inst.edge_w.sum())  # even torus, positive weights: the checkerboard cuts every edge
    r = run_islands(P, G.TerminationConfig(target_fitness=target, max_seconds=30.0), seed=1)
    assert r.reason == "target-reached"
    assert r.best_fitness == target
    assert r.seconds_to_target is not None and r.seconds_to_target <= r.seconds
    assert r.evaluations > 0 and r.populations[0] >= 1
    assert math.isfinite(r.seconds)
