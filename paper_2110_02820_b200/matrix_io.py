"""Matrix file ingestion (reference npcg::io, core/src/matrix_io.cpp:29-248;
SURVEY 8(f) row f4), mirroring include/npcg/matrix_io.hpp for Python users:
matrix-market (coordinate real/integer, general/symmetric), csv-dense and
raw-f64 (two little-endian uint64 dims + row-major little-endian doubles).
Parse failures raise RuntimeError("load_matrix - <path>:<line>: <what>");
an unknown format name raises ValueError (the reference's invalid_argument)."""
from __future__ import annotations

import numpy as np

FORMATS = ("matrix-market", "csv-dense", "raw-f64")


def parse_format(name: str) -> str:
    if name not in FORMATS:
        raise ValueError(f"parse_format: unknown format '{name}'")
    return name


def format_name(fmt: str) -> str:
    return parse_format(fmt)


def _fail(path, line, what):
    raise RuntimeError(f"load_matrix - {path}:{line}: {what}")


def _is_symmetric(m: np.ndarray) -> bool:
    if m.shape[0] != m.shape[1]:
        return False
    scale = max(1.0, float(np.abs(m).max()) if m.size else 0.0)
    return bool(np.abs(m - m.T).max() <= 1e-12 * scale) if m.size else True


def _read_mm(path):
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"load_matrix - cannot open {path}") from None
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        _fail(path, 1, "empty file")
    head = lines[0].split()
    head += [""] * (5 - len(head))
    if head[0] != "%%MatrixMarket" or head[1].lower() != "matrix":
        _fail(path, 1, "expected a MatrixMarket banner")
    if head[2].lower() != "coordinate":
        _fail(path, 1, "only coordinate format is supported")
    if head[3].lower() not in ("real", "integer"):
        _fail(path, 1, "only real-valued matrices are supported")
    if head[4].lower() not in ("symmetric", "general"):
        _fail(path, 1, "only general or symmetric matrices are supported")
    mirror = head[4].lower() == "symmetric"
    k, count, rows, cols = 1, -1, 0, 0
    while k < len(lines):
        s = lines[k]
        k += 1
        if not s or s[0] == "%":
            continue
        try:
            rows, cols, count = (int(t) for t in s.split()[:3])
        except ValueError:
            _fail(path, k, "malformed size line")
        break
    if count < 0:
        _fail(path, k, "missing size line")
    if rows < 1 or cols < 1:
        _fail(path, k, "dimensions must be positive")
    if mirror and rows != cols:
        _fail(path, k, "a symmetric matrix must be square")
    m = np.zeros((rows, cols), order="F")
    got = 0
    while k < len(lines):
        s = lines[k]
        k += 1
        if not s or s[0] == "%":
            continue
        t = s.split()
        try:
            i, j, v = int(t[0]), int(t[1]), float(t[2])
        except (ValueError, IndexError):
            _fail(path, k, "malformed entry")
        if not (1 <= i <= rows and 1 <= j <= cols):
            _fail(path, k, "entry index out of range")
        if mirror and j > i:
            _fail(path, k, "symmetric entries must lie on or below the diagonal")
        m[i - 1, j - 1] = v
        if mirror:
            m[j - 1, i - 1] = v
        got += 1
    if got != count:
        _fail(path, k, f"expected {count} entries, found {got}")
    return m


def _read_csv(path):
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"load_matrix - cannot open {path}") from None
    rows = []
    with f:
        for no, s in enumerate(f.read().split("\n"), start=1):
            if not s:
                continue
            toks = s.split(",")
            if len(toks) > 1 and toks[-1] == "":
                toks.pop()  # a trailing comma ends the row
            row = []
            for tok in toks:
                try:
                    if tok != tok.rstrip() and not tok.strip():
                        raise ValueError
                    row.append(float(tok))
                except ValueError:
                    _fail(path, no, f"malformed number '{tok}'")
            if rows and len(row) != len(rows[0]):
                _fail(path, no, "inconsistent column count")
            rows.append(row)
    if not rows:
        _fail(path, 1, "empty file")
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def _read_raw(path):
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"load_matrix - cannot open {path}") from None
    if len(data) < 16:
        raise RuntimeError(f"load_matrix - {path}: truncated raw-f64 header")
    r, c = (int(v) for v in np.frombuffer(data[:16], dtype="<u8"))
    if not (1 <= r <= 1 << 24 and 1 <= c <= 1 << 24):
        raise RuntimeError(f"load_matrix - {path}: implausible raw-f64 dimensions")
    if len(data) < 16 + 8 * r * c:
        raise RuntimeError(f"load_matrix - {path}: truncated raw-f64 payload")
    return np.asfortranarray(np.frombuffer(data[16:16 + 8 * r * c], dtype="<f8").reshape(r, c))


def load_matrix(path: str, fmt: str) -> np.ndarray:
    return {"matrix-market": _read_mm, "csv-dense": _read_csv, "raw-f64": _read_raw}[parse_format(fmt)](path)


def save_matrix(path: str, m, fmt: str) -> None:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim == 1:
        m = m.reshape(-1, 1)
    fmt = parse_format(fmt)
    if fmt == "raw-f64":
        with open(path, "wb") as f:
            f.write(np.array(m.shape, dtype="<u8").tobytes())
            f.write(np.ascontiguousarray(m, dtype="<f8").tobytes())
        return
    with open(path, "w") as f:
        if fmt == "csv-dense":
            for row in m:
                f.write(",".join(repr(float(v)) for v in row) + "\n")
            return
        sym = _is_symmetric(m)  # the symmetric writer stores the lower triangle
        ents = [(i, j, m[i, j]) for j in range(m.shape[1]) for i in range(j if sym else 0, m.shape[0])
                if m[i, j] != 0.0]
        f.write(f"%%MatrixMarket matrix coordinate real {'symmetric' if sym else 'general'}\n")
        f.write(f"{m.shape[0]} {m.shape[1]} {len(ents)}\n")
        for i, j, v in ents:
            f.write(f"{i + 1} {j + 1} {float(v)!r}\n")


def load_vector(path: str, fmt: str) -> np.ndarray:
    m = load_matrix(path, fmt)
    if m.shape[1] != 1:
        raise RuntimeError(f"load_vector - {path}: expected a single column")
    return m[:, 0].copy()


def require_symmetric(m, context: str) -> np.ndarray:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise RuntimeError(f"{context}: matrix must be square")
    if not _is_symmetric(m):
        raise RuntimeError(f"{context}: matrix is not symmetric")
    return m
