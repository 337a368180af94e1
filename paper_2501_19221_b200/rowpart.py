"""Row-partitioned multi-GPU solves (BASELINE config 5).

Instances too large for replica sharding (up to 2e8 variables) are split by rows: rank g
owns rows [g*B, min(n, (g+1)*B)) with B = ceil(n / world) and updates them for every
replica each step; the step needs every row's state, so after each step the ranks
all-gather the exchange buffer (NCCL over NVLink):

    PA : the bit-packed spins, n * R / 8 bytes per step (1 bit per replica-variable)
    SBM: the fp32 positions q,  4 * n * R bytes per step (32x larger: SBM is exchange-bound)

Two exchanges:
  "nccl"  the caller all-gathers each new state in place (NCCL all_gather_into_tensor);
  "p2p"   fused: every rank's exchange buffers are shared over CUDA IPC (NVLink peer
          memory) and the step kernels store their rows straight into every rank's copy,
          with a per-step release/acquire flag barrier (vxq_session_set_peers) -- no
          collective between steps, the transfer overlaps the step.

Buffer k & 1 holds state k.  `drive()` is the per-step loop; it takes any session with
`step(t)` and an in-place gather, so the multi-rank logic is exercised on CPU with gloo
(tests/test_distributed.py) while the product path runs `vxq_session_*` kernels on the
GPU with NCCL.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .device import get_problem
from .errors import ValidationError
from .solvers import Sample, SampleSet, _opts, _seed


def row_split(n: int, world: int) -> tuple[list[tuple[int, int]], int]:
    """Equal contiguous row blocks (the exchange all-gather needs equal chunk sizes)."""
    B = -(-int(n) // int(world))
    return [(min(n, g * B), min(n, (g + 1) * B)) for g in range(world)], B


def gather_inplace(buf, rank: int, world: int, chunk_bytes: int, group=None):
    """All-gather chunk `rank` of `buf` (uint8 tensor, world * chunk_bytes) in place."""
    import torch.distributed as dist
    if world == 1:
        return
    dist.all_gather_into_tensor(buf, buf[rank * chunk_bytes:(rank + 1) * chunk_bytes],
                                group=group)


def drive(session, bufs, T: int, gather) -> None:
    """The row-partitioned loop: state 0 exchange, then step t / exchange t+1."""
    gather(bufs[0])
    for t in range(T):
        session.step(t)
        gather(bufs[(t + 1) & 1])


def chunked_row_split(n: int, world: int, chunks: int):
    """Row ownership for the pipelined exchange: the rows are cut into `chunks` x `world`
    equal blocks of Bc rows, chunk c being the contiguous global range
    [c*world*Bc, (c+1)*world*Bc) and rank g owning its g-th block.  Chunk c of the exchange
    buffer is then exactly the [world][Bc] layout an in-place all-gather fills, so each
    chunk can be exchanged on its own.  Returns (spans[g][c] = (row_begin, row_end), Bc);
    rows_alloc = chunks * world * Bc (trailing padding rows are never read)."""
    C, W = int(chunks), int(world)
    Bc = -(-int(n) // (C * W))
    spans = [[(min(n, (c * W + g) * Bc), min(n, (c * W + g + 1) * Bc)) for c in range(C)]
             for g in range(W)]
    return spans, Bc


def drive_chunked(sessions, bufs, T: int, gather_async, chunk_bytes: int) -> None:
    """Pipelined row-partitioned loop: per step, chunk c's rows are stepped and
    their exchange is started asynchronously (NCCL runs it on its own stream) while chunk
    c+1 steps, so all but the last chunk's all-gather overlap the step kernels.  Step t+1
    of every chunk waits for all of state t+1 (the steps read every row).

    sessions[c]: this rank's session over its rows of chunk c (all share `bufs`);
    gather_async(view) -> handle with .wait() (in-place all-gather of one chunk's
    [world][Bc] block); chunk_bytes = world * Bc * row_bytes."""
    C = len(sessions)

    def view(k, c):
        return bufs[k][c * chunk_bytes:(c + 1) * chunk_bytes]

    pend = [gather_async(view(0, c)) for c in range(C)]
    for t in range(T):
        for h in pend:  # state t complete on every row
            h.wait()
        pend = []
        for c in range(C):
            sessions[c].step(t)
            pend.append(gather_async(view((t + 1) & 1, c)))
    for h in pend:
        h.wait()


def gather_chunk_async(view, rank: int, world: int, group=None):
    """In-place all-gather of one chunk (uint8 tensor of world * piece bytes), async."""
    import torch.distributed as dist

    class _Done:
        def wait(self):
            return None

    if world == 1:
        return _Done()
    piece = view.numel() // world
    return dist.all_gather_into_tensor(view, view[rank * piece:(rank + 1) * piece],
                                       group=group, async_op=True)


class GpuSession:
    """One rank's vxq_session (GPU kernels over rows [row_begin, row_end))."""

    def __init__(self, model, solver: str, params, row_begin, row_end, rows_alloc, bufs,
                 precision="fp32", device=0, stream=None, replica_begin=0,
                 outputs_on_device=False):
        L = _lib.load()
        dp = get_problem(model, device)
        self._dp = dp
        opts = _opts(precision, "sparse", replica_begin, stream=stream,
                     on_device=outputs_on_device)
        self._opts = opts
        pa = sbm = None
        if solver == "pa":
            pa = _lib.PaParamsC(int(params.steps), float(params.learning_rate),
                                float(params.momentum), _lib.nan_if_none(params.lambda0),
                                int(params.replicas), _seed(params.seed))
        else:
            sbm = _lib.SbmParamsC(int(params.steps), float(params.dt), float(params.a0),
                                  _lib.nan_if_none(params.c0), float(params.q_cap),
                                  float(params.init_noise), int(params.replicas),
                                  _seed(params.seed))
        h = ctypes.c_void_p()
        _lib.check(L.vxq_session_create(dp.handle, 0 if solver == "pa" else 1,
                                        ctypes.byref(pa) if pa else None,
                                        ctypes.byref(sbm) if sbm else None, int(row_begin),
                                        int(row_end), int(rows_alloc),
                                        ctypes.c_void_p(bufs[0].data_ptr()),
                                        ctypes.c_void_p(bufs[1].data_ptr()), ctypes.byref(opts),
                                        ctypes.byref(h)))
        self.handle = h
        self.R = int(params.replicas)
        self.n = int(model.n)

    def step(self, t: int):
        _lib.check(_lib.load().vxq_session_step(self.handle, int(t)))

    def finish_device(self, states_ptr: int, energies_ptr: int, order_ptr: int = 0):
        """finish() into caller-owned device buffers (session created with
        outputs_on_device=True)."""
        out = _lib.OutputsC()
        out.states, out.energies = ctypes.c_void_p(states_ptr), ctypes.c_void_p(energies_ptr)
        out.order = ctypes.c_void_p(order_ptr) if order_ptr else None
        _lib.check(_lib.load().vxq_session_finish(self.handle, ctypes.byref(out)))

    def finish(self, want_state: bool = False):
        """States/energies/order after the steps taken; want_state (a session over all
        rows only): also info["x"], info["m"] = X, M (PA) or Q, P (SBM) as (R, n) fp64."""
        st = np.empty((self.R, self.n), dtype=np.int8)
        en = np.empty(self.R)
        order = np.empty(self.R, dtype=np.int64)
        out = _lib.OutputsC()
        out.states, out.energies, out.order = _lib.ptr(st), _lib.ptr(en), _lib.ptr(order)
        x = m = None
        if want_state:
            x = np.empty((self.R, self.n))
            m = np.empty((self.R, self.n))
            out.x, out.m = _lib.ptr(x), _lib.ptr(m)
        _lib.check(_lib.load().vxq_session_finish(self.handle, ctypes.byref(out)))
        return st, en, order, {"lambda0": out.lambda0_used, "c0": out.c0_used, "x": x, "m": m}

    def close(self):
        if self.handle:
            _lib.load().vxq_session_destroy(self.handle)
            self.handle = None

    __del__ = close


def exchange_row_bytes(solver: str, replicas: int, precision: str = "fp32") -> int:
    v = ctypes.c_int64()
    _lib.check(_lib.load().vxq_exchange_row_bytes(0 if solver == "pa" else 1, int(replicas),
                                                  1 if precision == "fp64" else 0,
                                                  ctypes.byref(v)))
    return int(v.value)


class _RawBuf:
    """Device pointer with the tensor-like data_ptr() GpuSession expects."""

    def __init__(self, ptr: int):
        self.ptr = int(ptr)

    def data_ptr(self) -> int:
        return self.ptr


class PeerExchange:
    """IPC-shared exchange buffers + flags of one rank for the fused ("p2p") exchange.

    Allocates this rank's two exchange buffers and its flag array with vxq_exchange_alloc,
    shares their IPC handles with every rank (all_gather_object) and opens the peers'.
    ``ptrs[k][g]`` is rank g's buffer k (0, 1 = exchange buffers, 2 = flags)."""

    def __init__(self, buf_bytes: int, world: int, rank: int, device: int, group=None):
        import torch.distributed as dist
        L = _lib.load()
        self.world, self.rank, self.device, self.group = world, rank, device, group
        self.own, self.opened = [], []
        self.epoch = 0  # bumped per attached session (flag values carry it)
        for nbytes in (buf_bytes, buf_bytes, 8 * world):
            p = ctypes.c_void_p()
            _lib.check(L.vxq_exchange_alloc(device, int(nbytes), ctypes.byref(p)))
            self.own.append(int(p.value))
        handles = []
        for p in self.own:
            h = (ctypes.c_ubyte * _lib.IPC_HANDLE_BYTES)()
            _lib.check(L.vxq_ipc_handle(ctypes.c_void_p(p), h))
            handles.append(bytes(h))
        if world > 1:
            every = [None] * world
            dist.all_gather_object(every, handles, group=group)
        else:
            every = [handles]
        self.ptrs = [[0] * world for _ in range(3)]
        for g in range(world):
            for k in range(3):
                if g == rank:
                    self.ptrs[k][g] = self.own[k]
                    continue
                p = ctypes.c_void_p()
                h = (ctypes.c_ubyte * _lib.IPC_HANDLE_BYTES).from_buffer_copy(every[g][k])
                _lib.check(L.vxq_ipc_open(h, device, ctypes.byref(p)))
                self.ptrs[k][g] = int(p.value)
                self.opened.append(int(p.value))

    def bufs(self):
        return [_RawBuf(self.own[0]), _RawBuf(self.own[1])]

    def attach(self, session: "GpuSession"):
        """Bind a new session (every rank attaches its sessions in the same order; callers
        reusing the exchange put a barrier between sessions)."""
        self.epoch += 1
        arr = ctypes.c_void_p * self.world
        _lib.check(_lib.load().vxq_session_set_peers(
            session.handle, self.world, self.rank, self.epoch, arr(*self.ptrs[0]),
            arr(*self.ptrs[1]), arr(*self.ptrs[2])))

    def close(self):
        import torch.distributed as dist
        L = _lib.load()
        for p in self.opened:
            L.vxq_ipc_close(ctypes.c_void_p(p))
        self.opened = []
        if self.world > 1:  # no rank frees memory a peer may still have mapped
            dist.barrier(group=self.group)
        for p in self.own:
            L.vxq_exchange_free(ctypes.c_void_p(p))
        self.own = []


def solve_rowpart(solver: str, model, params, group=None, precision: str = "fp32",
                  timing: dict | None = None, exchange: str = "nccl",
                  chunks: int = 1) -> SampleSet:
    """Row-partitioned PA/SBM over the ranks of `group` (one GPU per rank).

    exchange="nccl": in-place all-gather after every step -- with chunks > 1 pipelined
    (chunked_row_split / drive_chunked: chunk c's all-gather overlaps chunk c+1's step);
    "p2p": the fused peer-memory exchange (PeerExchange).  Every rank returns the same
    best-first SampleSet.  With a single rank this is the ordinary sparse path
    (bit-identical)."""
    import torch
    import torch.distributed as dist

    if solver not in ("pa", "sbm"):
        raise ValidationError("solver must be 'pa' or 'sbm'")
    params.validate()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = torch.cuda.current_device()
    n = int(model.n)
    spans, B = row_split(n, world)
    rb = exchange_row_bytes(solver, params.replicas, precision)
    rows_alloc = B * world
    if exchange not in ("nccl", "p2p"):
        raise ValidationError("exchange must be 'nccl' or 'p2p'")
    px = None
    if exchange == "p2p":
        px = PeerExchange(rows_alloc * rb, world, rank, dev, group)
        bufs = px.bufs()
    elif chunks <= 1:
        bufs = [torch.zeros(rows_alloc * rb, dtype=torch.uint8, device=f"cuda:{dev}")
                for _ in range(2)]
    stream = torch.cuda.current_stream()
    t0 = time.perf_counter()
    if exchange == "nccl" and chunks > 1:
        cspans, Bc = chunked_row_split(n, world, chunks)
        rows_alloc = chunks * world * Bc
        bufs = [torch.zeros(rows_alloc * rb, dtype=torch.uint8, device=f"cuda:{dev}")
                for _ in range(2)]
        sessions = [GpuSession(model, solver, params, b, e, rows_alloc, bufs, precision, dev,
                               stream.cuda_stream) for b, e in cspans[rank]]
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        drive_chunked(sessions, bufs, int(params.steps),
                      lambda v: gather_chunk_async(v, rank, world, group), world * Bc * rb)
        ev1.record(stream)
        st, en, order, info = sessions[0].finish()
        for s_ in sessions:
            s_.close()
        if timing is not None:
            torch.cuda.synchronize()
            timing["loop_ms"] = ev0.elapsed_time(ev1)
            timing["exchange_bytes_per_step"] = rows_alloc * rb
        samples = [Sample(st[r].copy(), float(en[r]), int(r)) for r in order]
        return SampleSet(samples=samples, replica_count=int(params.replicas), seed=params.seed,
                         wall_time=time.perf_counter() - t0,
                         info={**info, "world": world, "rank": rank, "rows": cspans[rank],
                               "path": "rowpart", "exchange": f"nccl-pipelined x{chunks}"})
    sess = GpuSession(model, solver, params, spans[rank][0], spans[rank][1], rows_alloc, bufs,
                      precision, dev, stream.cuda_stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if px is not None:
        px.attach(sess)  # pushes state 0 to the peers; steps then exchange by themselves
        for t in range(int(params.steps)):
            sess.step(t)
    else:
        drive(sess, bufs, int(params.steps),
              lambda b: gather_inplace(b, rank, world, B * rb, group))
    ev1.record(stream)
    st, en, order, info = sess.finish()
    sess.close()
    if px is not None:
        px.close()
    if timing is not None:
        torch.cuda.synchronize()
        timing["loop_ms"] = ev0.elapsed_time(ev1)
        timing["exchange_bytes_per_step"] = rows_alloc * rb
    samples = [Sample(st[r].copy(), float(en[r]), int(r)) for r in order]
    return SampleSet(samples=samples, replica_count=int(params.replicas), seed=params.seed,
                     wall_time=time.perf_counter() - t0,
                     info={**info, "world": world, "rank": rank, "rows": spans[rank],
                           "path": "rowpart", "exchange": exchange})
