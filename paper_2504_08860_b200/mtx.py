"""Matrix Market ingest and output.

Mirrors /root/reference/pkg/src/hbp_spmv/formats.py: ``MatrixMarketError``
(:37-38), ``MatrixMarketHeader`` (:41-48), ``parse_matrix_market``
(:124-194), ``write_matrix_market`` (:197-209), ``load_mtx`` / ``save_mtx``
(:212-219), ``expand_symmetric`` (:222-240) -- same accepted dialect
(coordinate; real / integer / pattern; general / symmetric), same error
classes and message fragments.

Text parsing is host work (the file is text); ``read_matrix_market_arrays``
returns the 0-based host arrays, and ``parse_matrix_market`` hands them to
the device ``TripletMatrix`` whose canonicalisation (sort + duplicate sums
in np.add.reduceat order) runs on the GPU.
"""
from __future__ import annotations

import io
from dataclasses import dataclass
from typing import TextIO

import numpy as np

__all__ = ["MatrixMarketError", "MatrixMarketHeader", "read_matrix_market_arrays",
           "parse_matrix_market", "write_matrix_market", "load_mtx", "save_mtx",
           "expand_symmetric"]

_FIELDS = ("real", "integer", "pattern")
_SYMMETRIES = ("general", "symmetric")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input (formats.py:37-38)."""


@dataclass(frozen=True)
class MatrixMarketHeader:
    object: str
    format: str
    field: str
    symmetry: str


def read_matrix_market_arrays(stream: TextIO | str):
    """Validate and tokenize a coordinate Matrix Market text.

    Returns (header, rows, cols, i, j, v): 0-based int64 indices and f64
    values in file order (duplicates not yet summed)."""
    text = stream if isinstance(stream, str) else stream.read()
    lines = text.splitlines()
    if not lines:
        raise MatrixMarketError("empty input")
    banner = lines[0].split()
    if len(banner) != 5 or banner[0].lower() != "%%matrixmarket":
        raise MatrixMarketError(f"malformed banner: {lines[0]!r}")
    obj, fmt, fld, sym = (t.lower() for t in banner[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}")
    if fmt != "coordinate":
        raise MatrixMarketError(f"unsupported format {fmt!r}")
    if fld not in _FIELDS:
        raise MatrixMarketError(f"unsupported field {fld!r}")
    if sym not in _SYMMETRIES:
        raise MatrixMarketError(f"unsupported symmetry {sym!r}")
    header = MatrixMarketHeader(obj, fmt, fld, sym)

    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MatrixMarketError("missing size line")
    size = body[0].split()
    if len(size) != 3:
        raise MatrixMarketError(f"size line must have 3 integers: {body[0]!r}")
    try:
        rows, cols, nnz = (int(t) for t in size)
    except ValueError as exc:
        raise MatrixMarketError(f"non-integer size line: {body[0]!r}") from exc
    if rows < 0 or cols < 0 or nnz < 0:
        raise MatrixMarketError("negative dimension in size line")

    per = 2 if fld == "pattern" else 3
    tokens = " ".join(body[1:]).split()
    if len(tokens) != nnz * per:
        raise MatrixMarketError(f"declared {nnz} entries but found "
                                f"{len(tokens) / per:g} entry lines")
    tok = np.array(tokens, dtype=str).reshape(nnz, per)
    try:
        i = tok[:, 0].astype(np.int64)
        j = tok[:, 1].astype(np.int64)
    except ValueError as exc:
        raise MatrixMarketError(f"non-integer entry index: {exc}") from exc
    if fld == "pattern":
        v = np.ones(nnz, dtype=np.float64)
    else:
        try:
            v = tok[:, 2].astype(np.float64)
        except ValueError as exc:
            raise MatrixMarketError(f"bad entry value: {exc}") from exc
    if nnz and (i.min() < 1 or i.max() > rows or j.min() < 1 or j.max() > cols):
        raise MatrixMarketError("entry index out of declared bounds")
    return header, rows, cols, i - 1, j - 1, v


def parse_matrix_market(stream: TextIO | str):
    """formats.py:124-194: (header, canonical device TripletMatrix)."""
    from .formats import TripletMatrix
    header, rows, cols, i, j, v = read_matrix_market_arrays(stream)
    return header, TripletMatrix(rows, cols, i, j, v).canonicalized()


def write_matrix_market(matrix) -> str:
    """formats.py:197-209: 'general' real coordinate text, %.17g values
    (round-trips doubles exactly)."""
    out = io.StringIO()
    out.write("%%MatrixMarket matrix coordinate real general\n")
    out.write(f"{matrix.rows} {matrix.cols} {matrix.nnz}\n")
    r, c, v = (matrix.to_numpy() if hasattr(matrix, "to_numpy")
               else (np.asarray(matrix.row), np.asarray(matrix.col), np.asarray(matrix.val)))
    out.writelines("%d %d %.17g\n" % (a + 1, b + 1, x)
                   for a, b, x in zip(r.tolist(), c.tolist(), v.tolist()))
    return out.getvalue()


def load_mtx(path):
    with open(path, "r", encoding="ascii") as fh:
        return parse_matrix_market(fh)


def save_mtx(matrix, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(write_matrix_market(matrix))


def expand_symmetric(matrix):
    """formats.py:222-240: mirror the off-diagonal entries (device); output
    nnz = 2 nnz - diag.  Rejects non-square matrices and inputs holding both
    (i, j) and (j, i) for some i != j."""
    import torch
    from .formats import TripletMatrix
    if matrix.rows != matrix.cols:
        raise ValueError("symmetric expansion requires a square matrix")
    off = matrix.row != matrix.col
    key = matrix.row * matrix.cols + matrix.col
    mirror = matrix.col * matrix.cols + matrix.row
    if bool(torch.isin(key[off], mirror[off]).any().item()):
        raise ValueError("matrix holds both (i,j) and (j,i); symmetry ambiguous")
    row = torch.cat((matrix.row, matrix.col[off]))
    col = torch.cat((matrix.col, matrix.row[off]))
    val = torch.cat((matrix.val, matrix.val[off]))
    return TripletMatrix(matrix.rows, matrix.cols, row, col, val).canonicalized()
