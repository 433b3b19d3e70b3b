"""TSKM matrix files (reference include/skinnyqr/io.hpp:9-21, src/io.cpp:41-86) and their fast path to
the device.

Format, version 1, little endian: magic "TSKM", version u8 (= 1), element size u32 (= 8), rows u64,
cols u64, then m*n FP64 values in column order (25-byte header).  The payload is the in-memory
layout, so reading is a flat copy - and on this side of the boundary a flat *stream*: matrix_read_device
moves the payload through two pinned staging buffers straight into a column-major device tensor,
without ever holding the matrix in host memory (files larger than host RAM but not than HBM load).
"""
from __future__ import annotations

import os
import struct

import numpy as np

from . import DimensionError, Error

MAGIC = b"TSKM"
VERSION = 1
ELEM_SIZE = 8
HEADER_BYTES = 25  # io.hpp:23


class IoError(Error):
    pass


class FormatError(Error):
    pass


class TruncationError(Error):
    pass


class SizeOverflowError(Error):
    pass


def matrix_write(path, x):
    """io.cpp:41-59.  x: anything numpy can view as a 2-D float64 array (stored in column order)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError("matrix_write: need a 2-D matrix")
    try:
        with open(path, "wb") as f:
            f.write(MAGIC + struct.pack("<BIQQ", VERSION, ELEM_SIZE, a.shape[0], a.shape[1]))
            np.asfortranarray(a).T.astype("<f8", copy=False).tofile(f)
    except OSError as exc:
        raise IoError(f"matrix_write: cannot write '{path}': {exc}") from exc


def read_header(path):
    """Returns (m, n) after the checks of io.cpp:61-84."""
    try:
        with open(path, "rb") as f:
            h = f.read(HEADER_BYTES)
    except OSError as exc:
        raise IoError(f"matrix_read: cannot open '{path}'") from exc
    if len(h) != HEADER_BYTES:
        raise TruncationError(f"matrix_read: '{path}' shorter than header")
    if h[:4] != MAGIC:
        raise FormatError(f"matrix_read: bad magic in '{path}'")
    version, elem, m, n = struct.unpack("<BIQQ", h[4:])
    if version != VERSION:
        raise FormatError(f"matrix_read: unsupported version in '{path}'")
    if elem != ELEM_SIZE:
        raise FormatError(f"matrix_read: unsupported element size in '{path}'")
    if m == 0 or n == 0:
        raise DimensionError(f"matrix_read: zero dimension in '{path}'")
    if m > (2**64 - 1) // 8 // n:
        raise SizeOverflowError(f"matrix_read: m*n overflows addressable size in '{path}'")
    if os.path.getsize(path) < HEADER_BYTES + 8 * m * n:
        raise TruncationError(f"matrix_read: truncated payload in '{path}'")
    return m, n


def matrix_read(path):
    """io.cpp:61-86: Fortran-ordered (m, n) float64 array."""
    m, n = read_header(path)
    data = np.fromfile(path, dtype="<f8", count=m * n, offset=HEADER_BYTES)
    if data.size != m * n:
        raise TruncationError(f"matrix_read: truncated payload in '{path}'")
    return data.reshape((n, m)).T  # column order on disk == Fortran order in memory


def matrix_read_device(path, ctx, chunk_bytes=256 << 20):
    """Streams the payload into a column-major CUDA tensor of shape (m, n) (stride (1, m)): pread into
    one pinned buffer while the other is in flight on a copy stream.  No CPU fallback - needs torch
    with a CUDA device, like everything else that touches the GPU."""
    import torch
    m, n = read_header(path)
    x = ctx.empty_matrix(m, n)
    flat = x.t().reshape(-1)  # the (n, m) row-major storage == the file's column order
    total = m * n
    per = max(1, min(total, chunk_bytes // 8))
    bufs = [torch.empty(per, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    stream = torch.cuda.Stream(device=flat.device)
    fd = os.open(path, os.O_RDONLY)
    try:
        off, i = 0, 0
        while off < total:
            cnt = min(per, total - off)
            b = bufs[i & 1]
            if i >= 2:
                done[i & 1].synchronize()  # the copy that last used this buffer has drained
            view = memoryview(b.numpy())[:cnt].cast("B")
            got, want = 0, 8 * cnt
            while got < want:
                r = os.preadv(fd, [view[got:]], HEADER_BYTES + 8 * off + got)
                if r <= 0:
                    raise TruncationError(f"matrix_read: truncated payload in '{path}'")
                got += r
            with torch.cuda.stream(stream):
                flat[off:off + cnt].copy_(b[:cnt], non_blocking=True)
                done[i & 1].record(stream)
            off += cnt
            i += 1
        stream.synchronize()
    finally:
        os.close(fd)
    return x
