"""Multi-process host logic on CPU (gloo, world_size 2): replica sharding + final merge.

The oracle stands in for each rank's local GPU solve; the collectives and the merge
(ordering, global replica indices, packed-state all-gather) are the product code."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_2501_19221_b200.distributed import shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for total in (1, 7, 64, 1000, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _model():
    rng = np.random.default_rng(7)
    n = 24
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < 0.4
    m = type("M", (), {})()
    m.n, m.rows, m.cols = n, iu[keep], ju[keep]
    m.values = rng.uniform(-1, 1, keep.sum())
    m.h = rng.uniform(-1, 1, n)
    m.offset = 0.25
    return m


def _local_oracle(model, seed, steps):
    ip, ix, dv = O.symmetric_csr(model.n, model.rows, model.cols, model.values)
    lam = O.pa_schedule(O.resolve_lambda0(model), steps)

    def run(begin, count):
        X = np.stack([O.uniform(seed, begin + r, 0, model.n, -1.0, 1.0) for r in range(count)])
        X, _ = O.pa_run(ip, ix, dv, model.h, lam, 0.05, 0.9, X, np.zeros_like(X))
        st = O.sign_pm(X)
        return st, O.energies_exact(model, st)
    return run


def _worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2501_19221_b200.distributed import sharded_solve
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _model()
        ss = sharded_solve(_local_oracle(m, 5, 40), total, m.n, 5)
        out[rank] = ([s.replica for s in ss.samples], [s.energy for s in ss.samples],
                     np.stack([s.state for s in ss.samples]).tolist(), ss.info["shard"])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [33, 64])
def test_replica_sharded_merge_equals_single_process(total):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), total, out), nprocs=world,
                       join=True, start_method="spawn")
    m = _model()
    st, en = _local_oracle(m, 5, 40)(0, total)
    order = np.argsort(en, kind="stable")
    for rank in range(world):
        reps, energies, states, shard = out[rank]
        assert reps == order.tolist()                     # global replica ids, stable ties
        assert np.array_equal(np.array(energies), en[order])
        assert np.array_equal(np.array(states, dtype=np.int8), st[order])
    assert out[0][3] == shard_range(total, world, 0) and out[1][3] == shard_range(total, world, 1)


# ---------------------------------------------------------------- row partition (config 5)
class _OracleRowSession:
    """numpy stand-in for one rank's vxq_session (PA, fp64): same exchange-buffer protocol
    (sign bits, [rows_alloc][W] uint32, bit r%32 of word r/32) as the GPU kernels."""

    def __init__(self, model, R, T, seed, rb, re, bufs):
        self.ip, self.ix, self.dv = O.symmetric_csr(model.n, model.rows, model.cols,
                                                     model.values)
        self.h = np.asarray(model.h)
        self.lam = O.pa_schedule(O.resolve_lambda0(model), T)
        self.rb, self.re, self.R = rb, re, R
        self.W = (R + 31) // 32
        X = np.stack([O.uniform(seed, r, 0, model.n, -1.0, 1.0) for r in range(R)])
        self.x = X[:, rb:re].copy()
        self.m = np.zeros_like(self.x)
        self.bufs = bufs
        self._write(0, self.x)

    def _words(self, k):
        return self.bufs[k & 1].numpy().view(np.uint32).reshape(-1, self.W)

    def _write(self, k, x):
        bits = (x >= 0)  # (R, local rows)
        words = np.zeros((self.re - self.rb, self.W), dtype=np.uint32)
        for r in range(self.R):
            words[:, r // 32] |= (bits[r].astype(np.uint32) << np.uint32(r % 32))
        self._words(k)[self.rb:self.re] = words

    def _spins(self, k):
        words = self._words(k)
        r = np.arange(self.R)
        bits = (words[:, r // 32] >> (r % 32).astype(np.uint32)) & 1  # (rows_alloc, R)
        return np.where(bits == 1, 1.0, -1.0).T

    def step(self, t):
        S = self._spins(t)
        for li, i in enumerate(range(self.rb, self.re)):
            f = np.zeros(self.R)
            for k in range(self.ip[i], self.ip[i + 1]):
                f = f + self.dv[k] * S[:, self.ix[k]]
            grad = (self.lam[t] * self.x[:, li] + f) + self.h[i]
            self.m[:, li] = 0.9 * self.m[:, li] - 0.05 * grad
            self.x[:, li] = np.clip(self.x[:, li] + self.m[:, li], -1.0, 1.0)
        self._write(t + 1, self.x)


def _rowpart_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2501_19221_b200.rowpart import drive, gather_inplace, row_split
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _model()
        R, T = 40, 25
        spans, B = row_split(m.n, world)
        W = (R + 31) // 32
        row_bytes = 4 * W
        bufs = [torch.zeros(B * world * row_bytes, dtype=torch.uint8) for _ in range(2)]
        sess = _OracleRowSession(m, R, T, 3, spans[rank][0], spans[rank][1], bufs)
        drive(sess, bufs, T, lambda b: gather_inplace(b, rank, world, B * row_bytes))
        out[rank] = sess._spins(T)[:, : m.n].astype(np.int8).tolist()
    finally:
        dist.destroy_process_group()


def test_row_partitioned_exchange_equals_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rowpart_worker, args=(world, _free_port(), out), nprocs=world,
                       join=True, start_method="spawn")
    m = _model()
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X = O.pa_init(3, 40, m.n)
    X, _ = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), 25), 0.05, 0.9, X,
                    np.zeros_like(X))
    want = O.sign_pm(X)
    for rank in range(world):
        assert np.array_equal(np.array(out[rank], dtype=np.int8), want)


def _rowpart_chunked_worker(rank, world, port, chunks, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2501_19221_b200.rowpart import (chunked_row_split, drive_chunked,
                                               gather_chunk_async)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _model()
        R, T = 40, 25
        spans, Bc = chunked_row_split(m.n, world, chunks)
        W = (R + 31) // 32
        row_bytes = 4 * W
        rows_alloc = chunks * world * Bc
        bufs = [torch.zeros(rows_alloc * row_bytes, dtype=torch.uint8) for _ in range(2)]
        sessions = [_OracleRowSession(m, R, T, 3, b, e, bufs) for b, e in spans[rank]]
        drive_chunked(sessions, bufs, T, lambda v: gather_chunk_async(v, rank, world),
                      world * Bc * row_bytes)
        out[rank] = sessions[0]._spins(T)[:, : m.n].astype(np.int8).tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [2, 3])
def test_row_partitioned_pipelined_exchange_equals_single_process(chunks):
    """Pipelined exchange (chunk c's async all-gather overlaps chunk c+1's step): the rows
    are owned chunk-interleaved across the ranks; the result equals the 1-process loop."""
    from paper_2501_19221_b200.rowpart import chunked_row_split
    spans, Bc = chunked_row_split(24, 2, chunks)
    owned = sorted(r for g in range(2) for b, e in spans[g] for r in range(b, e))
    assert owned == list(range(24))  # every row owned exactly once
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rowpart_chunked_worker, args=(world, _free_port(), chunks, out),
                       nprocs=world, join=True, start_method="spawn")
    m = _model()
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    X = O.pa_init(3, 40, m.n)
    X, _ = O.pa_run(ip, ix, dv, m.h, O.pa_schedule(O.resolve_lambda0(m), 25), 0.05, 0.9, X,
                    np.zeros_like(X))
    want = O.sign_pm(X)
    for rank in range(world):
        assert np.array_equal(np.array(out[rank], dtype=np.int8), want)
