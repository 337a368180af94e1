"""Synthetic instances of the BASELINE.json configurations (seeded, vectorised).

These build canonical ``IsingModel`` arrays directly (sorted unique i<j COO), which is
what the reference's ``from_terms`` would produce (model.py:81-104) without its
O(terms) Python dict.  Used by bench.py and the tests.

  cfg1  dense random QUBO N=100 on all i<=j pairs, Q ~ U[-1,1] (drawn like gen_random,
        generators.py:321-323) -> qubo_to_ising (transforms.py:36-56)
  cfg2  Sherrington-Kirkpatrick N=10^4: J_ij = +-1/sqrt(N) i.i.d., h = 0
  cfg3  Pegasus P16 (5640 fabric qubits, 40,484 couplers; pegasus_edges), J, h ~ U[-1,1]
        drawn like gen_random("edge_list", "uniform") (generators.py:289-333).  The
        reference ships no Pegasus generator; pegasus_edges builds it.
  cfg4  3-regular MaxCut N=10^6 (configuration model, loops/multi-edges dropped),
        J = +1, h = 0: minimising sum s_i s_j maximises the cut, cut = (|E| - H) / 2
  cfg5  random QUBO, mean degree 6, diagonal and off-diagonal ~ U[-1,1] -> Ising
"""

from __future__ import annotations

import numpy as np

from .model import IsingModel, QuboModel
from .transforms import qubo_to_ising


def _philox(seed, index=0):
    bits = np.random.Philox(key=np.uint64(seed))
    if index:
        bits = bits.jumped(index)
    return np.random.Generator(bits)


def cfg1_qubo(seed: int = 2501, n: int = 100) -> tuple[QuboModel, IsingModel]:
    rng = _philox(seed)
    iu, ju = np.triu_indices(n, 0)
    vals = rng.uniform(-1.0, 1.0, size=len(iu))
    q = QuboModel(n=n, rows=iu.astype(np.int64), cols=ju.astype(np.int64), values=vals + 0.0)
    return q, qubo_to_ising(q)


def sk(n: int = 10_000, seed: int = 2) -> IsingModel:
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    J = np.where(rng.random(len(iu)) < 0.5, -1.0, 1.0) / np.sqrt(n)
    return IsingModel(n=n, h=np.zeros(n), rows=iu.astype(np.int64), cols=ju.astype(np.int64),
                      values=J)


def random_edges(n: int, m: int, seed: int):
    rng = np.random.default_rng(seed)
    keys = np.zeros(0, dtype=np.int64)
    while keys.size < m:
        a = rng.integers(0, n, 2 * (m - keys.size) + 16)
        b = rng.integers(0, n, a.size)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        k = (lo * n + hi)[lo != hi]
        keys = np.unique(np.concatenate([keys, k]))
    keys = np.sort(rng.choice(keys, m, replace=False))
    return keys // n, keys % n


# Pegasus P(m) offsets (the standard shift pattern, offsets index 0): vertical qubit k of
# a tile meets horizontal qubits shifted by _PEG_OFF0[k]; horizontal qubit k is shifted by
# _PEG_OFF1[k].
_PEG_OFF0 = (2, 2, 2, 2, 10, 10, 10, 10, 6, 6, 6, 6)
_PEG_OFF1 = (6, 6, 6, 6, 2, 2, 2, 2, 10, 10, 10, 10)


def pegasus_edges(m: int = 16) -> tuple[int, np.ndarray]:
    """Edge list of the Pegasus graph P(m), fabric nodes only (the D-Wave Advantage
    topology the paper's instances use; the reference has no generator for it,
    SPEC.md:239).

    A qubit is (u, w, k, z): orientation u (0 vertical, 1 horizontal), perpendicular
    offset w < m, qubit index k < 12, parallel offset z < m-1.  Three coupler classes:
      external  (u,w,k,z)-(u,w,k,z+1)            same line, consecutive segments
      odd       (u,w,k,z)-(u,w,k+1,z), k even     paired neighbours
      internal  (0,w,k,z)-(1, z+[kk<OFF0[k]], kk, w-[k<OFF1[kk]])   crossing lines
    restricted to the fabric (qubits with at least one internal coupler: for u, tiles
    w=0 drop k < min(OFF), tiles w=m-1 drop k >= 12-(12-max(OFF))).  Qubits are
    relabelled 0..n-1 in (u, w, k, z) order.  P(16): 5640 qubits, 40,484 couplers,
    maximum degree 15.  Returns (n, edges[E, 2]) in generation order
    (external, odd, internal).
    """
    if m < 2:
        raise ValueError("pegasus needs m >= 2")
    m1 = m - 1
    start = (min(_PEG_OFF1), min(_PEG_OFF0))
    end = (12 - max(_PEG_OFF1), 12 - max(_PEG_OFF0))

    def krange(u, w):
        return range(start[u] if w == 0 else 0, 12 - (end[u] if w == m1 else 0))

    def lin(u, w, k, z):
        return ((u * m + w) * 12 + k) * m1 + z

    def fabric(u, w, k, z):
        return (w > 0 or k >= start[u]) and (w < m1 or k < 12 - end[u])

    e = []
    for u in (0, 1):
        for w in range(m):
            for k in krange(u, w):
                for z in range(m1 - 1):
                    e.append((lin(u, w, k, z), lin(u, w, k, z + 1)))
    for u in (0, 1):
        for w in range(m):
            for k in krange(u, w)[::2]:
                for z in range(m1):
                    e.append((lin(u, w, k, z), lin(u, w, k + 1, z)))
    for w in range(m):
        for kk in range(12):
            for k in range(0 if w else _PEG_OFF1[kk], 12 if w < m1 else _PEG_OFF1[kk]):
                for z in range(m1):
                    a = (0, w, k, z)
                    b = (1, z + (kk < _PEG_OFF0[k]), kk, w - (k < _PEG_OFF1[kk]))
                    if fabric(*a) and fabric(*b):
                        e.append((lin(*a), lin(*b)))
    e = np.asarray(e, dtype=np.int64)
    used, e = np.unique(e, return_inverse=True)
    return int(used.size), e.reshape(-1, 2)


def pegasus(m: int = 16, seed: int = 16) -> IsingModel:
    """gen_random("edge_list", "uniform", seed, edges=pegasus_edges(m)) restated
    (generators.py:289-333): couplings drawn first in edge-list order, then biases, from
    one Philox stream; J, h ~ U[-1, 1]."""
    from .model import canonical_pairs

    n, e = pegasus_edges(m)
    rng = _philox(seed)
    J = rng.uniform(-1.0, 1.0, size=e.shape[0])
    h = rng.uniform(-1.0, 1.0, size=n)
    r, c, v = canonical_pairs(e[:, 0], e[:, 1], J, n, allow_diagonal=False)
    return IsingModel(n=n, h=h, rows=r, cols=c, values=v)


def maxcut3(n: int = 1_000_000, seed: int = 4) -> IsingModel:
    rng = np.random.default_rng(seed)
    stubs = np.repeat(np.arange(n, dtype=np.int64), 3)
    rng.shuffle(stubs)
    a, b = stubs[0::2], stubs[1::2]
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    keep = lo != hi
    key = np.unique(lo[keep] * n + hi[keep])
    return IsingModel(n=n, h=np.zeros(n), rows=key // n, cols=key % n,
                      values=np.ones(key.size))


def random_qubo_deg6(n: int, seed: int = 5) -> IsingModel:
    r, c = random_edges(n, 3 * n, seed)
    rng = _philox(seed)
    off = rng.uniform(-1.0, 1.0, r.size)
    diag = rng.uniform(-1.0, 1.0, n)
    rows = np.concatenate([r, np.arange(n)])
    cols = np.concatenate([c, np.arange(n)])
    vals = np.concatenate([off, diag])
    order = np.lexsort((cols, rows))
    q = QuboModel(n=n, rows=rows[order], cols=cols[order], values=vals[order] + 0.0)
    return qubo_to_ising(q)


# ------------------------------------------------------------- config-5 family (device)
_M32 = np.uint64(0xFFFFFFFF)


def _mulhilo(a, b):
    a_lo, a_hi = a & _M32, a >> np.uint64(32)
    b_lo, b_hi = b & _M32, b >> np.uint64(32)
    p0, p1, p2, p3 = a_lo * b_lo, a_lo * b_hi, a_hi * b_lo, a_hi * b_hi
    mid = (p0 >> np.uint64(32)) + (p1 & _M32) + (p2 & _M32)
    hi = p3 + (p1 >> np.uint64(32)) + (p2 >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, a * b


def philox_raw(seed: int, stream: int, k) -> np.ndarray:
    """Vectorised Philox4x64-10 draw k of stream `stream` (ctr = (k/4+1, 0, stream, 0),
    key = (seed, 0)) -- the numpy replica-stream layout, any stream index."""
    k = np.asarray(k, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c0 = k // np.uint64(4) + np.uint64(1)
        c1 = np.zeros_like(c0)
        c2 = np.full_like(c0, np.uint64(stream))
        c3 = np.zeros_like(c0)
        k0, k1 = np.uint64(seed), np.uint64(0)
        M0, M1 = np.uint64(0xD2E7470EE14C6C93), np.uint64(0xCA5A826395121157)
        W0, W1 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBB67AE8584CAA73B)
        for _ in range(10):
            hi0, lo0 = _mulhilo(M0, c0)
            hi1, lo1 = _mulhilo(M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0, k1 = k0 + W0, k1 + W1
        out = np.stack([c0, c1, c2, c3])
    return out[(k % np.uint64(4)).astype(np.int64), np.arange(k.size)]


def _unit_uniform(raw):
    return -1.0 + 2.0 * ((raw >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0))


def qubo_deg6_family(n: int, seed: int) -> tuple[QuboModel, IsingModel]:
    """Host mirror of the device generator (csrc/generate.cu, family 0) for small n."""
    S = 1 << 40
    i = np.arange(n, dtype=np.uint64)
    keys = []
    for c in range(3):
        off = np.uint64(1) + philox_raw(seed, S + c, i) % np.uint64(n - 1)
        j = (i + off) % np.uint64(n)
        lo, hi = np.minimum(i, j), np.maximum(i, j)
        keys.append(lo * np.uint64(n) + hi)
    key = np.unique(np.concatenate(keys))
    r, c_ = (key // np.uint64(n)).astype(np.int64), (key % np.uint64(n)).astype(np.int64)
    qoff = _unit_uniform(philox_raw(seed, S + 3, key))
    qdiag = _unit_uniform(philox_raw(seed, S + 4, i))
    rows = np.concatenate([r, np.arange(n)])
    cols = np.concatenate([c_, np.arange(n)])
    vals = np.concatenate([qoff, qdiag])
    order = np.lexsort((cols, rows))
    q = QuboModel(n=n, rows=rows[order], cols=cols[order], values=vals[order] + 0.0)
    return q, qubo_to_ising(q)


CONFIGS = {
    "cfg1": dict(desc="dense random QUBO N=100 -> Ising, R=64, T=1000", R=64, T=1000),
    "cfg2": dict(desc="dense Sherrington-Kirkpatrick N=10^4 (J=+-1/sqrt N), R=1024, T=1000",
                 R=1024, T=1000),
    "cfg3": dict(desc="Pegasus P16 N=5640 (40,484 couplers), R=4096, T=1000",
                 R=4096, T=1000),
    "cfg4": dict(desc="3-regular MaxCut N=10^6, R=256, T=1000", R=256, T=1000),
    "cfg5": dict(desc="random QUBO N=2x10^8 mean degree 6, R=32", R=32, T=100),
}


def build(name: str, n: int | None = None) -> IsingModel:
    if name == "cfg1":  # --n scales the same dense random QUBO family (general dense J)
        return cfg1_qubo(n=n or 100)[1]
    if name == "cfg2":
        return sk(n or 10_000)
    if name == "cfg3":
        return pegasus()
    if name == "cfg4":
        return maxcut3(n or 1_000_000)
    if name == "cfg5":
        from .device import GeneratedModel
        return GeneratedModel("qubo_deg6", n or 200_000_000, seed=5)
    raise KeyError(name)
