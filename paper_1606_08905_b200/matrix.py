"""Input normalisation and row partitioning (numakmeans matrix.py, the parts on the path).

``check_matrix`` keeps the reference's contract (matrix.py:35-49): a 2-D,
C-contiguous float64 array with n, d >= 1 and every value finite, else
``MatrixFormatError`` naming the first bad row.  ``kmeans()`` does the cheap
shape/dtype half on the host and the O(nd) finite scan on the GPU after the
upload (knb_check_finite), with the same error.

``partition_rows`` is the reference's split (matrix.py:196-213): contiguous
ranges whose sizes differ by at most one, remainder to the lowest ids.  Here
it assigns row shards to GPUs.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np


class MatrixFormatError(ValueError):
    """Malformed input matrix: wrong rank, empty, or non-finite values."""


class RowRange(NamedTuple):
    start: int
    stop: int
    node: int

    def __len__(self):
        return self.stop - self.start


def check_shape(m, keep_f32: bool = False) -> np.ndarray:
    """Host half of check_matrix: C-contiguous float64 (float32 kept as is when
    ``keep_f32``), 2-D, n, d >= 1 (no finite scan)."""
    m = np.ascontiguousarray(m, dtype=np.float32 if keep_f32 else np.float64)
    if m.ndim != 2:
        raise MatrixFormatError(f"expected a 2-D matrix, got ndim={m.ndim}")
    n, d = m.shape
    if n < 1 or d < 1:
        raise MatrixFormatError(f"matrix must be at least 1x1, got {n}x{d}")
    return m


def check_matrix(m) -> np.ndarray:
    """Full host-side check_matrix (matrix.py:35-49), for callers that want it eagerly."""
    m = check_shape(m)
    finite = np.isfinite(m)
    if not finite.all():
        bad = int(np.flatnonzero(~finite.all(axis=1))[0])
        raise MatrixFormatError(f"non-finite value in row {bad}")
    return m


def partition_rows(n: int, parts: int, nodes: int = 1) -> list[RowRange]:
    """Split [0, n) into ``parts`` contiguous ranges, sizes differing by <= 1 (matrix.py:196-213)."""
    if parts < 1 or nodes < 1:
        raise ValueError("parts and nodes must be >= 1")
    base, rem = divmod(n, parts)
    per_node, extra = divmod(parts, nodes)
    node_of = []
    for node in range(nodes):
        node_of.extend([node] * (per_node + (1 if node < extra else 0)))
    out, start = [], 0
    for w in range(parts):
        size = base + (1 if w < rem else 0)
        out.append(RowRange(start, start + size, node_of[w] if w < len(node_of) else nodes - 1))
        start += size
    return out
