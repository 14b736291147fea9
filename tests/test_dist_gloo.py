"""Multi-process (gloo, world size 2, CPU) test of the sharding protocol in
paper_2202_05048_b200/dist.py: calibration images of every cache dealt over
ranks, MIN/MAX allreduce of the local ranges, local histograms with the global
range, SUM allreduce -- must equal single-process calibration bit for bit; and
config shards (dist.shard_plan) must reassemble in order.  The per-rank "device" is
the numpy oracle here (the GPU path implements the same two calls through
ptq_calib_forward / ptq_calib_histogram)."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ptq_oracle as O


class OracleBackend:
    def __init__(self, g, d):
        self.g, self.d = g, d

    def forward_minmax(self, sizes, ids):
        self.per_cache = []
        out = []
        off = 0
        for k, n in enumerate(sizes):
            acts = []
            for i in ids[off:off + n]:
                a = {}
                O.run_fp32(self.g, self.d.images[i:i + 1], lambda t, v: a.__setitem__(t, v))
                acts.append(a)
            off += n
            self.per_cache.append(acts)
            names = [O.INPUT] + [nd.output for nd in self.g.nodes]
            r = np.zeros((len(names), 2), np.float32)
            for t, name in enumerate(names):
                if acts:
                    r[t] = (min(float(a[name].min()) for a in acts), max(float(a[name].max()) for a in acts))
                else:
                    r[t] = (np.inf, -np.inf)
            out.append(r)
        self.names = [O.INPUT] + [nd.output for nd in self.g.nodes]
        return np.stack(out)

    def histogram(self, ranges):
        out = np.zeros((len(self.per_cache), len(self.names), 2048), np.int64)
        for k, acts in enumerate(self.per_cache):
            for t, name in enumerate(self.names):
                for a in acts:
                    out[k, t] += O.histogram_counts(a[name], float(ranges[k, t, 0]), float(ranges[k, t, 1]))
        return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_05048_b200 import dist as D
        from paper_2202_05048_b200.dataset import make_dataset
        from paper_2202_05048_b200.fixtures import generate_fixture
        g = generate_fixture("lenet-ish", 1)
        d = make_dataset(n_calib=40, n_eval=8, seed=0)
        ranges, counts, n_img = D.sharded_calibration(OracleBackend(g, d), d.n_calib, 0, len(g.nodes) + 1)
        from paper_2202_05048_b200 import GENERIC, enumerate_space
        space = enumerate_space(GENERIC)
        idx = D.shard_plan(space, world)[rank]
        got = D.gather_counts(np.asarray(idx, dtype=np.int64) * 7, idx, len(space))
        if rank == 0:
            q.put((ranges, counts, n_img, got))
    finally:
        dist.destroy_process_group()


def test_sharded_calibration_matches_single_process(monkeypatch):
    from paper_2202_05048_b200 import config as C
    from paper_2202_05048_b200.dataset import make_dataset
    from paper_2202_05048_b200.fixtures import generate_fixture
    monkeypatch.setitem(C.SIZE_CLASSES, "S2", 5)
    monkeypatch.setitem(C.SIZE_CLASSES, "S3", 9)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ranges, counts, n_img, got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got.tolist() == [7 * i for i in range(96)]
    g = generate_fixture("lenet-ish", 1)
    d = make_dataset(n_calib=40, n_eval=8, seed=0)
    for k, sc in enumerate(("S1", "S2", "S3")):
        ids = C.select_images(d.n_calib, sc, 0)
        assert n_img[k] == len(ids)
        ref = O.calibrate(g, d.images[ids])
        for t, h in enumerate(ref.values()):
            assert (ranges[k, t, 0], ranges[k, t, 1]) == (np.float32(h.lo), np.float32(h.hi))
            assert np.array_equal(counts[k, t], h.counts)


def test_shard_plan_balanced_contiguous_variants():
    """dist.shard_plan: every config exactly once; each rank's block is whole (cache, scheme,
    clipping) variants, contiguous in variant order, with equal counts of Mixed=Off /
    FirstLastFp32 and per-tensor / per-channel configs at 2, 4 and 8 ranks."""
    from paper_2202_05048_b200 import GENERIC, enumerate_space
    from paper_2202_05048_b200 import dist as D
    from paper_2202_05048_b200.config import config_key
    space = enumerate_space(GENERIC)
    for n in (1, 2, 3, 4, 8):
        plan = D.shard_plan(space, n)
        assert sorted(i for p in plan for i in p) == list(range(len(space)))
        seen = {}
        for r, p in enumerate(plan):
            for i in p:
                v = config_key(space[i])[:3]
                assert seen.setdefault(v, r) == r          # a variant never straddles ranks
        if n in (2, 4, 8):
            assert len({len(p) for p in plan}) == 1
            for p in plan:
                keys = [config_key(space[i]) for i in p]
                assert sum(k[4] for k in keys) * 2 == len(p)     # half FirstLastFp32
                assert sum(k[3] for k in keys) * 2 == len(p)     # half per-channel
