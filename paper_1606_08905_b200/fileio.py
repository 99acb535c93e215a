"""KNRM matrix files (numakmeans matrix.py:18-109, format SPEC.md:97).

A file is a 28-byte little-endian header -- magic ``KNRM``, u32 version 1, u64 n,
u64 d, u32 dtype code 0 (= f64) -- followed by the row-major f64 payload, or the
payload alone ("raw", shape supplied by the caller).  Errors keep the reference's
types and message fragments: ``MatrixFormatError`` for malformed files,
``MatrixIOError`` for failed reads/writes.

Loading maps the payload (``np.memmap``) instead of reading the whole file into a
bytes object and copying it, so a file can be handed to ``kmeans()`` -- which
copies it to HBM once -- without a second host copy.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .matrix import MatrixFormatError, check_matrix

MAGIC = b"KNRM"
FORMAT_VERSION = 1
DTYPE_F64 = 0
_HEADER = struct.Struct("<4sIQQI")
HEADER_SIZE = _HEADER.size  # 28


class MatrixIOError(OSError):
    """I/O failure while reading or writing a matrix file."""


def save_matrix(m, path, raw: bool = False) -> None:
    """Write ``m`` (validated like check_matrix) with the KNRM header, or raw."""
    m = check_matrix(m)
    n, d = m.shape
    offset = 0
    try:
        with open(path, "wb") as fh:
            if not raw:
                fh.write(_HEADER.pack(MAGIC, FORMAT_VERSION, n, d, DTYPE_F64))
                offset = HEADER_SIZE
            m.astype("<f8", copy=False).tofile(fh)
    except OSError as exc:
        raise MatrixIOError(f"write failed for {path} at byte offset {offset}: {exc}") from exc


def read_header(path) -> tuple[int, int]:
    """(n, d) from a KNRM header, with the reference's checks."""
    try:
        size = os.path.getsize(path)
        with open(path, "rb") as fh:
            head = fh.read(HEADER_SIZE)
    except OSError as exc:
        raise MatrixIOError(f"read failed for {path}: {exc}") from exc
    if len(head) < HEADER_SIZE:
        raise MatrixFormatError(f"{path}: file too short for header (expected >= {HEADER_SIZE} bytes, got {size})")
    magic, version, n, d, code = _HEADER.unpack(head)
    if magic != MAGIC:
        raise MatrixFormatError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise MatrixFormatError(f"{path}: unsupported format version {version}")
    if code != DTYPE_F64:
        raise MatrixFormatError(f"{path}: unknown dtype code {code}")
    return int(n), int(d)


def load_matrix(path, raw: bool = False, n: int | None = None, d: int | None = None,
                check_finite: bool = True) -> np.ndarray:
    """The file's rows as an (n, d) f64 array (memory-mapped, read-only).

    ``check_finite=False`` leaves the O(nd) scan to the device (kmeans() runs it there
    after the upload, with the same error)."""
    if raw:
        if n is None or d is None:
            raise MatrixFormatError("raw files carry no shape; pass n and d explicitly")
        offset = 0
    else:
        n, d = read_header(path)
        offset = HEADER_SIZE
    try:
        payload = os.path.getsize(path) - offset
    except OSError as exc:
        raise MatrixIOError(f"read failed for {path}: {exc}") from exc
    expected = n * d * 8
    if payload != expected:
        raise MatrixFormatError(
            f"{path}: payload length mismatch, expected {expected} bytes for {n}x{d}, got {payload}")
    if n < 1 or d < 1:
        raise MatrixFormatError(f"matrix must be at least 1x1, got {n}x{d}")
    try:
        m = np.memmap(path, dtype="<f8", mode="r", offset=offset, shape=(n, d))
    except OSError as exc:  # pragma: no cover - depends on the filesystem
        raise MatrixIOError(f"read failed for {path}: {exc}") from exc
    if check_finite:
        finite = np.isfinite(m).all(axis=1)
        if not finite.all():
            raise MatrixFormatError(f"non-finite value in row {int(np.flatnonzero(~finite)[0])}")
    return m
