"""Batch sampling of the trainer (train.py:332-347 epoch permutations): the
next-epoch permutation drawn ahead in the helper process must give exactly
the batch / slice sequence of drawing it inline, across several epochs."""

import time

import numpy as np

from paper_2603_00145_b200 import train as T


def _sampler(seed, m, b, prefetch, monkeypatch):
    monkeypatch.setenv("MGAUSS_PERM_PREFETCH", "1" if prefetch else "0")
    monkeypatch.setattr(T, "_PERM_PREFETCH_MIN", 1)
    t = T.Trainer.__new__(T.Trainer)  # host sampling state only (no device)
    t.m_points, t.config, t.rng = m, T.TrainConfig(batch_points=b), np.random.default_rng(seed)
    t._perm, t._cursor, t._permuter, t.slice_grids = None, 0, None, [None] * 7
    return t


def _draw(t, steps, pause=0.0):
    out = []
    for i in range(steps):
        idx = t._next_batch()
        out.append((idx.copy(), int(t.rng.integers(len(t.slice_grids)))))
        if pause:  # let the helper finish (it is never waited for)
            time.sleep(2.0 if i == 0 else pause)
    return out


def test_prefetched_permutations_match_inline(monkeypatch):
    m, b = 5000, 1536  # batches straddle epoch boundaries
    a = _draw(_sampler(3, m, b, False, monkeypatch), 25)
    t = _sampler(3, m, b, True, monkeypatch)
    try:
        got = _draw(t, 25, pause=0.05)
        # 25 x 1536 draws from a 5000-sample pool cross 7 epoch boundaries; the
        # first is drawn inline (the helper is still starting), the rest come
        # from the helper's two-ahead chain
        assert t._permuter.adopted >= 5
        # a trainer that outruns its helper draws inline, with the same result
        t2 = _sampler(3, m, b, True, monkeypatch)
        try:
            got2 = _draw(t2, 25)
        finally:
            t2.close()
    finally:
        t.close()
    for (ia, ja), (ib, jb) in zip(a, got2):
        np.testing.assert_array_equal(ia, ib)
        assert ja == jb
    for (ia, ja), (ib, jb) in zip(a, got):
        np.testing.assert_array_equal(ia, ib)
        assert ja == jb


def test_prefetch_mismatch_falls_back_inline(monkeypatch):
    m, b = 5000, 1536
    a = _sampler(5, m, b, False, monkeypatch)
    t = _sampler(5, m, b, True, monkeypatch)
    try:
        for s in (a, t):
            s._next_batch()
            s.rng.integers(7)
            s.rng.integers(3)  # an extra draw the prefetch did not replay
        for _ in range(6):
            np.testing.assert_array_equal(a._next_batch(), t._next_batch())
            assert a.rng.integers(7) == t.rng.integers(7)
    finally:
        t.close()


def test_prefetch_chain_restarts_after_midrun_mismatch(monkeypatch):
    """An unpredicted draw in the middle of a run drops the two-ahead chain;
    the next boundary draws inline, the chain restarts, and the sequence stays
    identical to drawing every permutation inline."""
    m, b = 4608, 1536  # exactly 3 batches per epoch
    a = _sampler(9, m, b, False, monkeypatch)
    t = _sampler(9, m, b, True, monkeypatch)
    try:
        for s in (a, t):
            for i in range(30):
                s._next_batch()
                s.rng.integers(7)
                if i == 14:
                    s.rng.integers(5)  # not in the predicted schedule
                if s is t:
                    time.sleep(1.0 if i == 0 else 0.03)
        adopted_before = t._permuter.adopted
        for _ in range(12):
            np.testing.assert_array_equal(a._next_batch(), t._next_batch())
            assert a.rng.integers(7) == t.rng.integers(7)
            time.sleep(0.03)
        assert adopted_before >= 3 and t._permuter.adopted > adopted_before  # the chain came back
    finally:
        t.close()
