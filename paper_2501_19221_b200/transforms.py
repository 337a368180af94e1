"""QUBO-in adapter: qubo_to_ising (reference transforms.py:36-56), vectorised.

The reference loops over the QUBO terms in canonical (i, j) order:
  i == j:  h[i] += v/2,               offset += v/2
  i <  j:  J_ij = v/4, h[i] += v/4, h[j] += v/4, offset += v/4
Here the same contributions are applied with np.add.at over an index array laid
out in that exact term order (h[i] before h[j] within a term), and the offset is a
sequential np.add.accumulate, so the result is bit-identical to the reference.
"""

from __future__ import annotations

import numpy as np

from .model import IsingModel, QuboModel


def qubo_to_ising(q) -> IsingModel:
    n = int(q.n)
    rows = np.asarray(q.rows, dtype=np.int64)
    cols = np.asarray(q.cols, dtype=np.int64)
    vals = np.asarray(q.values, dtype=np.float64)
    diag = rows == cols
    half = vals / 2.0
    quarter = vals / 4.0
    # per-term h contributions in term order: diag -> (i, v/2); off -> (i, v/4), (j, v/4)
    cnt = np.where(diag, 1, 2)
    pos = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    total = int(cnt.sum())
    idx = np.empty(total, dtype=np.int64)
    add = np.empty(total, dtype=np.float64)
    idx[pos] = rows
    add[pos] = np.where(diag, half, quarter)
    off = ~diag
    idx[pos[off] + 1] = cols[off]
    add[pos[off] + 1] = quarter[off]
    h = np.zeros(n)
    np.add.at(h, idx, add)
    contrib = np.where(diag, half, quarter)
    offset = float(np.add.accumulate(np.concatenate([[float(q.offset)], contrib]))[-1]) \
        if contrib.size else float(q.offset)
    return IsingModel(n=n, h=h, rows=rows[off], cols=cols[off], values=quarter[off] + 0.0,
                      offset=offset)


__all__ = ["qubo_to_ising", "QuboModel"]
