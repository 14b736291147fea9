"""Call coalescing for the reference's threaded measure_many (tuner.py:192-203; SURVEY
8(f) item 1): concurrent evaluate(cfg) calls are served by fewer, larger batches and every
caller gets its own result or its own exception -- a failing item never fails the callers
that happened to share its batch (the reference's _safe_eval fails one trial, tuner.py:173-177)."""
import threading
import time

import pytest

from paper_2202_05048_b200.evaluator import Coalescer


def test_concurrent_calls_are_batched_and_routed():
    calls = []

    def batch(items):
        calls.append(list(items))
        time.sleep(0.02)                      # a GPU batch takes a while
        return [x * 10 for x in items]

    co = Coalescer(batch)
    out = {}

    def worker(i):
        out[i] = co(i)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(32)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out == {i: i * 10 for i in range(32)}
    assert sum(len(c) for c in calls) == 32
    assert len(calls) < 32                    # coalesced
    assert co.batches == [len(c) for c in calls]


def test_errors_reach_every_caller_of_the_batch():
    def batch(items):
        time.sleep(0.01)
        raise ValueError("bad config")

    co = Coalescer(batch)
    errs = []

    def worker():
        try:
            co(1)
        except ValueError as e:
            errs.append(str(e))

    ts = [threading.Thread(target=worker) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert errs == ["bad config"] * 8


def test_one_bad_item_fails_only_its_caller():
    def batch(items):
        time.sleep(0.01)
        if any(x < 0 for x in items):
            raise ValueError("bad config")
        return [x * 2 for x in items]

    co = Coalescer(batch)
    out, errs = {}, {}

    def worker(i):
        try:
            out[i] = co(i)
        except ValueError as e:
            errs[i] = str(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(-2, 14)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert errs == {-2: "bad config", -1: "bad config"}
    assert out == {i: 2 * i for i in range(14)}


def test_sequential_calls_still_work():
    co = Coalescer(lambda items: [x + 1 for x in items])
    assert [co(i) for i in range(5)] == [1, 2, 3, 4, 5]
    with pytest.raises(ZeroDivisionError):
        Coalescer(lambda items: [1 / 0 for _ in items])(3)
