"""Instance files at scale: the reference's quadratic text/JSON formats.

Mirrors qubokit/instance_io.py:82-152 for the models on this path (Ising "spin" and QUBO
"binary" domains; HUBO files are outside the dynamics loop and raise ValidationError):

    # format: quadratic            (optional; a 3-field body implies quadratic)
    # offset: <float repr>         (optional)
    n m d                          (d = spin | binary)
    i j v                          (m lines, 1-based; i == j is a field / diagonal term)

Reading is vectorised (pandas C parser with round-trip float parsing, so every value is
the correctly rounded double Python's float() would give) and accumulates duplicates in
file order exactly like the reference (h[i] += v sequentially; couplings via the dict
accumulation of model.from_terms), so large instances load bit-identically.
"""

from __future__ import annotations

import io
import json
from pathlib import Path

import numpy as np

from .errors import ValidationError
from .model import IsingModel, QuboModel, canonical_pairs

FORMAT_QUADRATIC = "quadratic"


def _quadratic(n: int, domain: str, i, j, v, offset: float):
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    if i.size and (min(i.min(), j.min()) < 0 or max(i.max(), j.max()) >= n):
        k = int(np.argmax((i < 0) | (j < 0) | (i >= n) | (j >= n)))
        raise ValidationError(f"term index pair ({i[k]}, {j[k]}) out of range for n={n}")
    if domain == "spin":
        diag = i == j
        h = np.zeros(n)
        np.add.at(h, i[diag], v[diag])  # file order, like h[i] += v (instance_io.py:69-73)
        if not np.all(np.isfinite(h)):
            raise ValidationError("field vector must be finite")
        r, c, val = canonical_pairs(i[~diag], j[~diag], v[~diag], n, allow_diagonal=False)
        return IsingModel(n=n, h=h, rows=r, cols=c, values=val, offset=float(offset))
    if domain == "binary":
        r, c, val = canonical_pairs(i, j, v, n, allow_diagonal=True)
        return QuboModel(n=n, rows=r, cols=c, values=val, offset=float(offset))
    raise ValidationError(f"unknown domain tag {domain!r}")


def model_to_dict(model) -> dict:
    """JSON mirror of the text schema, 1-based indices (instance_io.py:33-50)."""
    if isinstance(model, QuboModel) or (not hasattr(model, "h") and hasattr(model, "rows")):
        terms = [[int(i) + 1, int(j) + 1, float(v)]
                 for i, j, v in zip(model.rows, model.cols, model.values)]
        return {"format": FORMAT_QUADRATIC, "n": int(model.n), "domain": "binary",
                "offset": float(model.offset), "terms": terms}
    terms = [[int(i) + 1, int(i) + 1, float(v)] for i, v in enumerate(model.h) if v != 0.0]
    terms += [[int(i) + 1, int(j) + 1, float(v)]
              for i, j, v in zip(model.rows, model.cols, model.values)]
    return {"format": FORMAT_QUADRATIC, "n": int(model.n), "domain": "spin",
            "offset": float(model.offset), "terms": terms}


def model_from_dict(data: dict):
    fmt = data.get("format")
    if fmt != FORMAT_QUADRATIC:
        raise ValidationError(f"unsupported instance format {fmt!r} (only quadratic models "
                              f"enter the dynamics loop)")
    n = int(data["n"])
    t = np.asarray(data["terms"], dtype=np.float64).reshape(-1, 3)
    return _quadratic(n, data["domain"], t[:, 0].astype(np.int64) - 1,
                      t[:, 1].astype(np.int64) - 1, t[:, 2], float(data.get("offset", 0.0)))


def write_instance(path, model) -> Path:
    """Write a model (text, or JSON for a .json suffix) like instance_io.py:82-101."""
    path = Path(path)
    data = model_to_dict(model)
    if path.suffix == ".json":
        path.write_text(json.dumps(data, indent=2) + "\n")
        return path
    lines = [f"# format: {FORMAT_QUADRATIC}"]
    if data["offset"] != 0.0:
        lines.append(f"# offset: {data['offset']!r}")
    lines.append(f"{data['n']} {len(data['terms'])} {data['domain']}")
    lines += [f"{i} {j} {v!r}" for i, j, v in data["terms"]]
    path.write_text("\n".join(lines) + "\n")
    return path


def read_instance(path):
    """Read a quadratic instance written by either implementation (text or JSON)."""
    path = Path(path)
    if path.suffix == ".json":
        return model_from_dict(json.loads(path.read_text()))
    import pandas as pd

    fmt = None
    offset = 0.0
    header = None
    body_start = 0
    text = path.read_text()
    lines = text.splitlines()
    for k, raw in enumerate(lines):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("#"):
            c = line[1:].strip()
            if c.startswith("format:"):
                fmt = c.split(":", 1)[1].strip()
            elif c.startswith("offset:"):
                offset = float(c.split(":", 1)[1])
            continue
        header = line.split()
        body_start = k + 1
        break
    if header is None or len(header) != 3:
        raise ValidationError(f"{path}: missing or malformed 'n m d' header line")
    n, m, domain = int(header[0]), int(header[1]), header[2]
    if fmt not in (None, FORMAT_QUADRATIC):
        raise ValidationError(f"{path}: unsupported format {fmt!r} (quadratic only)")
    body = "\n".join(ln for ln in lines[body_start:] if ln.strip() and not ln.lstrip().startswith("#"))
    if m == 0 and not body:
        return _quadratic(n, domain, [], [], [], offset)
    try:
        df = pd.read_csv(io.StringIO(body), sep=r"\s+", header=None, engine="c",
                         float_precision="round_trip", dtype={0: np.int64, 1: np.int64})
    except Exception as e:  # noqa: BLE001
        raise ValidationError(f"{path}: malformed term lines ({e})") from e
    if df.shape[0] != m:
        raise ValidationError(f"{path}: header declares {m} terms, found {df.shape[0]}")
    if df.shape[1] != 3:
        raise ValidationError(f"{path}: quadratic line needs 'i j v' (HUBO instances are "
                              f"outside the dynamics-loop scope)")
    return _quadratic(n, domain, df[0].to_numpy() - 1, df[1].to_numpy() - 1,
                      df[2].to_numpy(dtype=np.float64), offset)
