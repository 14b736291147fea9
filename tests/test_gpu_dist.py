"""The multi-GPU protocol (paper_2202_05048_b200/dist.py) with the real CUDA
evaluator: two processes (gloo, world size 2) each drive their own GpuEvaluator context --
both on cuda:0, since this box has one GPU; the collectives are host-side and no kernel of
one rank waits for the other, so sharing the device is safe.

Checked bit-identical to one process:
* sharded calibration (images of every cache split over ranks, MIN/MAX then SUM allreduce of
  the device's local ranges / histograms, ref calibration.py:57-106);
* the KL sweep sharded by histogram (clipping.py:55-86) and reassembled;
* the grid split by dist.shard_plan and reassembled (measure_many, tuner.py:192-203);
* image-sharded single-config evaluation (tune_xgb's sequential evaluate, tuner.py:251-281).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE = (3, 64, 64)
PICKS = [0, 2, 13, 30, 47, 64, 81, 94]


def _data():
    from paper_2202_05048_b200 import build_model, make_dataset
    return build_model("resnet50", 0, shape=SHAPE), make_dataset(n_calib=300, n_eval=48, seed=0, shape=SHAPE)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_05048_b200 import GENERIC, enumerate_space
        from paper_2202_05048_b200.evaluator import GpuEvaluator
        g, d = _data()
        space = enumerate_space(GENERIC)
        ev = GpuEvaluator(g, d, 0, GENERIC, device=0)
        grid = ev.evaluate_grid(space)
        out = (ev.cache_ranges.copy(), ev.cache_counts.copy(), ev.kl_ranges.copy(), grid)
        ev.close()
        ev2 = GpuEvaluator(g, d, 0, GENERIC, device=0, image_sharded=True)
        acc = [ev2(space[i]) for i in PICKS]
        ev2.close()
        q.put((rank, out, acc))
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, a)) for r, o, a in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2202_05048_b200 import GENERIC, enumerate_space
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    g, d = _data()
    space = enumerate_space(GENERIC)
    ev = GpuEvaluator(g, d, 0, GENERIC, device=0)
    want_grid = ev.correct_counts(space)
    want_acc = ev.evaluate_many([space[i] for i in PICKS])
    for r in (0, 1):
        (ranges, counts, kl, grid), acc = res[r]
        assert np.array_equal(ranges, ev.cache_ranges), r
        assert np.array_equal(counts, ev.cache_counts), r
        assert np.array_equal(kl, ev.kl_ranges), r
        assert np.array_equal(grid, want_grid), r
        assert acc == want_acc, r
    ev.close()
