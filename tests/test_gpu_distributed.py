"""GPU: row-partitioned sessions and replica sharding through the C-ABI on one B200.

Multi-rank NCCL runs need several GPUs; here (1 GPU) the row partition is exercised as
several sessions with different row ranges sharing one exchange buffer (no gather
needed), which is exactly what each rank computes, and world=1 through the public API."""

import numpy as np
import pytest

import oracle as O
import paper_2501_19221_b200 as vxq
from helpers import gen_complete, maxcut_model

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R", [96, 32])
@pytest.mark.parametrize("solver", ["pa", "sbm"])
@pytest.mark.parametrize("parts", [1, 2, 3])
def test_row_partition_sessions_match_sparse_path(solver, parts, R):
    """R = 32 is config 5's shape (PA: the cooperative 8-rows-per-warp step), here with row
    ranges that do not start at 0."""
    import torch

    from paper_2501_19221_b200.rowpart import GpuSession, exchange_row_bytes, row_split
    m = maxcut_model(3000, 3, 11) if solver == "pa" else gen_complete(8, 300, "gaussian")
    if solver == "pa":
        params = vxq.PaParams(steps=40, replicas=R, seed=4)
        ref = vxq.run_pa(m, params, path="sparse")
    else:
        params = vxq.SbmParams(steps=40, dt=0.05, replicas=R, seed=4, c0=0.1)
        ref = vxq.run_sbm(m, params, path="sparse")
    spans, B = row_split(m.n, parts)
    rb = exchange_row_bytes(solver, params.replicas)
    bufs = [torch.zeros(B * parts * rb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    stream = torch.cuda.current_stream().cuda_stream
    sess = [GpuSession(m, solver, params, b, e, B * parts, bufs, stream=stream)
            for b, e in spans]
    for t in range(params.steps):
        for s in sess:   # every "rank" writes its rows of the shared next buffer
            s.step(t)
    st, en, order, _ = sess[0].finish()
    assert np.array_equal(st, ref.states)
    assert np.array_equal(en, ref.energies)
    assert np.array_equal(order, ref.order)


def test_solve_rowpart_world1_public_api():
    from paper_2501_19221_b200.rowpart import solve_rowpart
    m = maxcut_model(5000, 3, 2)
    p = vxq.PaParams(steps=30, replicas=32, seed=1)
    ss = solve_rowpart("pa", m, p)
    ref = vxq.solve_pa(m, p, path="sparse")
    assert [s.replica for s in ss.samples] == [s.replica for s in ref.samples]
    assert [s.energy for s in ss.samples] == [s.energy for s in ref.samples]
    assert np.array_equal(ss.best.state, ref.best.state)
    assert ss.best.energy == O.energy_exact(m, ss.best.state)


@pytest.mark.parametrize("n,seed", [(1000, 5), (40_000, 9)])
def test_device_generator_matches_host_mirror(n, seed):
    """Config-5 family generated on the GPU == the numpy mirror (QUBO -> qubo_to_ising):
    couplings and fields bit-exact, offset == the exact sum of the terms (fsum)."""
    import math

    from paper_2501_19221_b200.device import GeneratedModel
    from paper_2501_19221_b200.instances import qubo_deg6_family
    g = GeneratedModel("qubo_deg6", n, seed)
    m = g.export()
    q, ref = qubo_deg6_family(n, seed)
    for f in ("rows", "cols", "values", "h"):
        assert np.array_equal(getattr(m, f), getattr(ref, f)), f
    terms = [float(v) / (2.0 if i == j else 4.0) for i, j, v in zip(q.rows, q.cols, q.values)]
    assert m.offset == math.fsum(terms)
    assert abs(m.offset - ref.offset) <= 1e-12 * max(1.0, abs(ref.offset))
    # solving the generated model == solving its exported host copy
    p = vxq.PaParams(steps=20, replicas=32, seed=3)
    a = vxq.run_pa(g, p)
    b = vxq.run_pa(m, p)
    assert np.array_equal(a.states, b.states) and np.array_equal(a.energies, b.energies)
    assert np.array_equal(a.energies[:4], O.energies_exact(m, a.states[:4]))


# ---------------------------------------------------------------- fused peer exchange
@pytest.mark.parametrize("solver", ["pa", "sbm"])
def test_solve_rowpart_world1_fused_exchange(solver):
    """exchange="p2p" (library-allocated IPC buffers, in-kernel stores + flag barrier) at
    world 1 == the sparse path."""
    from paper_2501_19221_b200.rowpart import solve_rowpart
    m = maxcut_model(4000, 3, 6) if solver == "pa" else gen_complete(5, 200, "gaussian")
    if solver == "pa":
        p = vxq.PaParams(steps=25, replicas=64, seed=2)
        ref = vxq.solve_pa(m, p, path="sparse")
    else:
        p = vxq.SbmParams(steps=25, dt=0.05, replicas=64, seed=2, c0=0.1)
        ref = vxq.solve_sbm(m, p, path="sparse")
    ss = solve_rowpart(solver, m, p, exchange="p2p")
    assert ss.info["exchange"] == "p2p"
    assert [s.replica for s in ss.samples] == [s.replica for s in ref.samples]
    assert [s.energy for s in ss.samples] == [s.energy for s in ref.samples]
    assert np.array_equal(ss.best.state, ref.best.state)


@pytest.mark.parametrize("solver,R", [("pa", 32), ("pa", 96), ("sbm", 64)])
def test_fused_exchange_stores_to_every_destination(solver, R):
    """One session with three destinations on this GPU (its own buffers + two stand-in
    peer copies): every step's rows land identically in all three copies, every copy's
    flag slot [rank] ends at T + 1, and the solve equals the sparse path.  The stand-in
    sources' flags are pre-published, so nothing waits on another process."""
    import ctypes

    import torch

    from paper_2501_19221_b200 import _lib
    from paper_2501_19221_b200.rowpart import GpuSession, exchange_row_bytes
    m = maxcut_model(2500, 3, 8) if solver == "pa" else gen_complete(6, 150, "gaussian")
    T = 12
    if solver == "pa":
        params = vxq.PaParams(steps=T, replicas=R, seed=7)
        ref = vxq.run_pa(m, params, path="sparse")
    else:
        params = vxq.SbmParams(steps=T, dt=0.05, replicas=R, seed=7, c0=0.1)
        ref = vxq.run_sbm(m, params, path="sparse")
    rb = exchange_row_bytes(solver, R)
    world, rank = 3, 0
    mk = lambda: torch.zeros(m.n * rb, dtype=torch.uint8, device="cuda")  # noqa: E731
    xb = [[mk() for _ in range(world)] for _ in range(2)]
    flags = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
    flags[rank][1:] = 1 << 60  # stand-in sources: already published every state
    stream = torch.cuda.current_stream().cuda_stream
    sess = GpuSession(m, solver, params, 0, m.n, m.n, [xb[0][rank], xb[1][rank]],
                      stream=stream)
    arr = ctypes.c_void_p * world
    _lib.check(_lib.load().vxq_session_set_peers(
        sess.handle, world, rank, 1, arr(*[b.data_ptr() for b in xb[0]]),
        arr(*[b.data_ptr() for b in xb[1]]), arr(*[f.data_ptr() for f in flags])))
    for t in range(T):
        sess.step(t)
    st, en, order, _ = sess.finish()
    torch.cuda.synchronize()
    for k in range(2):
        for g in range(1, world):
            assert torch.equal(xb[k][g], xb[k][rank]), (k, g)
    for g in range(world):
        assert int(flags[g][rank]) == (1 << 32) + T + 1
    assert np.array_equal(st, ref.states)
    assert np.array_equal(en, ref.energies)
    assert np.array_equal(order, ref.order)
    sess.close()


def test_fused_exchange_rejects_foreign_own_buffers():
    import ctypes

    import torch

    from paper_2501_19221_b200 import _lib
    from paper_2501_19221_b200.rowpart import GpuSession, exchange_row_bytes
    m = maxcut_model(500, 3, 1)
    params = vxq.PaParams(steps=3, replicas=32, seed=1)
    rb = exchange_row_bytes("pa", 32)
    bufs = [torch.zeros(m.n * rb, dtype=torch.uint8, device="cuda") for _ in range(3)]
    fl = torch.zeros(2, dtype=torch.int64, device="cuda")
    sess = GpuSession(m, "pa", params, 0, m.n, m.n, bufs[:2],
                      stream=torch.cuda.current_stream().cuda_stream)
    arr = ctypes.c_void_p * 2
    with pytest.raises(vxq.ValidationError):  # xbuf0[rank] must be the session's own
        _lib.check(_lib.load().vxq_session_set_peers(
            sess.handle, 2, 0, 1, arr(bufs[2].data_ptr(), bufs[0].data_ptr()),
            arr(bufs[1].data_ptr(), bufs[1].data_ptr()), arr(fl.data_ptr(), fl.data_ptr())))
    sess.close()


@pytest.mark.parametrize("solver", ["pa", "sbm"])
def test_chunked_row_sessions_match_sparse_path(solver):
    """Pipelined exchange ownership (chunk-interleaved rows, rowpart.chunked_row_split) for
    2 "ranks" x 3 chunks sharing one exchange buffer == the 1-GPU sparse path; and
    solve_rowpart(chunks=4) at world 1 through the public API."""
    import torch

    from paper_2501_19221_b200.rowpart import (GpuSession, chunked_row_split,
                                               exchange_row_bytes, solve_rowpart)
    m = maxcut_model(3000, 3, 13)
    if solver == "pa":
        params = vxq.PaParams(steps=30, replicas=64, seed=2)
        ref = vxq.run_pa(m, params, path="sparse")
    else:
        params = vxq.SbmParams(steps=30, dt=0.05, replicas=64, seed=2, c0=0.3)
        ref = vxq.run_sbm(m, params, path="sparse")
    spans, Bc = chunked_row_split(m.n, 2, 3)
    rows_alloc = 3 * 2 * Bc
    rb = exchange_row_bytes(solver, params.replicas)
    bufs = [torch.zeros(rows_alloc * rb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    stream = torch.cuda.current_stream().cuda_stream
    sess = [GpuSession(m, solver, params, b, e, rows_alloc, bufs, stream=stream)
            for g in range(2) for b, e in spans[g]]
    for t in range(params.steps):
        for s in sess:
            s.step(t)
    st, en, order, _ = sess[0].finish()
    assert np.array_equal(st, ref.states) and np.array_equal(en, ref.energies)
    ss = solve_rowpart(solver, m, params, chunks=4)
    assert [s.replica for s in ss.samples] == list(ref.order)


def test_session_snapshot_state_sbm():
    """A one-rank session over all rows, stopped after k < T steps of the T-step schedule,
    returns Q/P equal to the oracle's fp32 loop over the first k schedule entries."""
    import torch

    from paper_2501_19221_b200.rowpart import GpuSession, exchange_row_bytes
    m = gen_complete(8, 300, "gaussian")
    params = vxq.SbmParams(steps=100, dt=0.05, replicas=40, seed=3, c0=0.1)
    rb = exchange_row_bytes("sbm", params.replicas)
    bufs = [torch.zeros(m.n * rb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    sess = GpuSession(m, "sbm", params, 0, m.n, m.n, bufs)
    for t in range(17):
        sess.step(t)
    st, en, order, info = sess.finish(want_state=True)
    sess.close()
    ip, ix, dv = O.symmetric_csr(m.n, m.rows, m.cols, m.values)
    Q, P = O.sbm_init(3, 40, m.n, 1.0)
    Q, P = O.sbm_run(ip, ix, -dv, -m.h, O.sbm_schedule(1.0, 100)[:17], 0.05, 1.0, 0.1, 1.0, Q,
                     P, np.float32)
    assert np.array_equal(info["x"], Q.astype(np.float64))
    assert np.array_equal(info["m"], P.astype(np.float64))
    assert np.array_equal(en, O.energies_exact(m, st))


def test_shard_path_pins_dense_for_small_shards():
    """A replica shard smaller than the dense threshold (R >= 128) runs the global solve's
    tensor-core path (distributed.shard_path), so its rows equal the 1-GPU solve's."""
    from helpers import sk_model
    from paper_2501_19221_b200.distributed import shard_path
    m = sk_model(700, 4)
    full = vxq.PaParams(steps=20, replicas=256, seed=3)
    g = vxq.run_pa(m, full, want_state=True)
    assert g.info["path"] == "dense"
    path = shard_path(m, "pa", full, "fp32", "auto", 0)
    assert path == "dense"
    shard = vxq.run_pa(m, vxq.PaParams(steps=20, replicas=64, seed=3), path=path,
                       replica_begin=192, want_state=True)
    assert shard.info["path"] == "dense"
    assert np.array_equal(shard.x, g.x[192:256])
    assert np.array_equal(shard.energies, g.energies[192:256])
    # below the threshold globally: auto stays auto (the CSR paths are the same arithmetic)
    assert shard_path(m, "pa", vxq.PaParams(steps=20, replicas=64, seed=3), "fp32", "auto",
                      0) == "auto"
