"""Test helpers: instance builders and brute force (test infrastructure only).

``gen_complete`` restates the reference generator used by its own solver tests
(generators.py:289-333, topology "complete"): couplings on all i<j pairs in
lexicographic order drawn first, then biases, from rng_stream(seed).
"""

from __future__ import annotations

import numpy as np

from paper_2501_19221_b200 import IsingModel


def rng_stream(seed, index=0):
    bits = np.random.Philox(key=np.uint64(seed))
    if index:
        bits = bits.jumped(index)
    return np.random.Generator(bits)


def gen_complete(seed, n, dist="uniform", a=-1.0, b=1.0, with_biases=True) -> IsingModel:
    rng = rng_stream(seed)
    iu, ju = np.triu_indices(n, 1)

    def draw(size):
        if dist == "uniform":
            return rng.uniform(a, b, size=size)
        if dist == "int_uniform":
            return rng.integers(int(a), int(b) + 1, size=size).astype(np.float64)
        if dist == "gaussian":
            return rng.standard_normal(size)
        raise ValueError(dist)

    vals = draw(len(iu))
    h = draw(n) if with_biases else np.zeros(n)
    return IsingModel.from_arrays(n, iu, ju, vals + 0.0, h=h, canonical=True)


def model_from_golden(g, prefix) -> IsingModel:
    return IsingModel(n=int(g[f"{prefix}_n"]), h=g[f"{prefix}_h"], rows=g[f"{prefix}_rows"],
                      cols=g[f"{prefix}_cols"], values=g[f"{prefix}_values"],
                      offset=float(g[f"{prefix}_offset"]))


def all_spin_states(n: int) -> np.ndarray:
    bits = (np.arange(2 ** n)[:, None] >> np.arange(n)[None, :]) & 1
    return (2 * bits - 1).astype(np.int8)


def brute_force_min(model) -> float:
    """Exhaustive minimum via exact per-state sums (oracle.energy_exact), n <= 16."""
    import oracle
    S = all_spin_states(model.n).astype(np.float64)
    quad = (S[:, model.rows] * S[:, model.cols]) @ model.values
    E = quad + S @ model.h + model.offset
    # exact re-evaluation of the candidates within float noise of the minimum
    cand = np.where(E <= E.min() + 1e-9)[0]
    return min(oracle.energy_exact(model, S[c]) for c in cand)


def random_regular_edges(n, d, seed):
    """Configuration-model d-regular multigraph, self-loops/multi-edges dropped."""
    rng = np.random.default_rng(seed)
    stubs = np.repeat(np.arange(n, dtype=np.int64), d)
    rng.shuffle(stubs)
    a, b = stubs[0::2], stubs[1::2]
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    keep = lo != hi
    key = np.unique(lo[keep] * n + hi[keep])
    return key // n, key % n


def maxcut_model(n, d, seed) -> IsingModel:
    """3-regular MaxCut as minimisation of sum s_i s_j (J = +1, h = 0): BASELINE cfg 4."""
    r, c = random_regular_edges(n, d, seed)
    return IsingModel.from_arrays(n, r, c, np.ones(len(r)), canonical=True)


def sk_model(n, seed) -> IsingModel:
    """Sherrington-Kirkpatrick: J_ij = +-1/sqrt(N), h = 0 (BASELINE cfg 2)."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    J = np.where(rng.random(len(iu)) < 0.5, -1.0, 1.0) / np.sqrt(n)
    return IsingModel.from_arrays(n, iu, ju, J, canonical=True)
