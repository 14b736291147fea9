"""Image-sharded single-config evaluation (the sequential xgb / GA
searches, ptqtune/tuner.py:251-281) over gloo, world size 2, on CPU: each rank takes
its contiguous eval slice (dist.eval_slice, the same split GpuEvaluator(image_sharded=True)
uploads), counts correct predictions there, SUM-allreduces -- the top-1 must equal the
single-process value for every config.  The per-rank "device" is the numpy oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import ptq_oracle as O

CFG_IDX = (0, 9, 45)


def _setup():
    from paper_2202_05048_b200.config import GENERIC, enumerate_space
    from paper_2202_05048_b200.dataset import make_dataset
    from paper_2202_05048_b200.fixtures import generate_fixture
    g = generate_fixture("lenet-ish", 1)
    d = make_dataset(n_calib=20, n_eval=13, seed=0)
    caches = {sc: O.calibrate(g, d.images[:4]) for sc in ("S1", "S2", "S3")}
    cfgs = [enumerate_space(GENERIC)[i] for i in CFG_IDX]
    return g, d, caches, cfgs


def _counts(g, d, caches, cfgs, lo, hi):
    ev_img = d.images[d.n_calib + lo: d.n_calib + hi]
    ev_lab = d.labels[d.n_calib + lo: d.n_calib + hi]
    return np.asarray([O.top1_count(O.run_quantized(O.quantize_model(g, caches[c.cache], c), ev_img), ev_lab)
                       for c in cfgs], dtype=np.int64)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_05048_b200 import dist as D
        g, d, caches, cfgs = _setup()
        r, n = D.world()
        lo, hi = D.eval_slice(13, r, n)
        tot = D.allreduce(_counts(g, d, caches, cfgs, lo, hi), "sum")
        q.put((rank, (lo, hi), tot))
    finally:
        tdist.destroy_process_group()


def test_eval_slice_partitions():
    from paper_2202_05048_b200.dist import eval_slice
    for n_eval in (1, 7, 1000):
        for world in (1, 2, 3, 8):
            if world > n_eval:
                with pytest.raises(ValueError):
                    [eval_slice(n_eval, r, world) for r in range(world)]
                continue
            sl = [eval_slice(n_eval, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n_eval
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


def test_image_sharded_counts_match_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [(0, 6), (6, 13)]
    g, d, caches, cfgs = _setup()
    want = _counts(g, d, caches, cfgs, 0, 13)
    for _, _, tot in res:
        assert np.array_equal(tot, want)


@pytest.mark.gpu
def test_gpu_image_sharded_slices_sum_to_full(monkeypatch, golden, ds, toys):
    """One GPU, two evaluators standing in for ranks 0 and 1 of 2 (dist.world patched,
    no collective): their eval slices' correct counts sum to the unsharded counts."""
    from paper_2202_05048_b200 import dist as D
    from paper_2202_05048_b200.config import GENERIC, enumerate_space
    from paper_2202_05048_b200.evaluator import GpuEvaluator
    from test_gpu_parity import golden_caches
    cfgs = enumerate_space(GENERIC)[:96:7]
    _, ranges, counts, nsamp, _ = golden_caches(golden, "resnet-toy")

    def make(kl=None, **kw):
        ev = GpuEvaluator(toys["resnet-toy"], ds, 0, GENERIC, calibrate=False, **kw)
        ev.install_caches(ranges, counts, nsamp, kl_ranges=kl)
        return ev

    full = make()
    want = full.correct_counts(cfgs)
    # the patched world would also shard the KL sweep by histogram (reassembled by a SUM
    # allreduce that needs a process group): hand the "ranks" the full KL table instead
    kl = full.kl_ranges.copy()
    full.close()
    got = np.zeros_like(want)
    for r in range(2):
        monkeypatch.setattr(D, "world", lambda r=r: (r, 2))
        ev = make(kl, image_sharded=True)
        assert ev.image_sharded and ev.n_eval_local == D.eval_slice(ev.n_eval, r, 2)[1] - D.eval_slice(ev.n_eval, r, 2)[0]
        got += ev.correct_counts(cfgs)
        ev.close()
    assert np.array_equal(got, want)
