"""Graph files (drop-in for graphlb/io.py), read natively by libgraphlb_b200.so.

* ``load_dimacs_gr`` / ``load_edge_list`` parse the reference's text formats
  (io.py:26-122) in C++ with the same grammar, the same ``ParseError``
  messages and ``CsrGraph.from_edges`` grouping, and return a host CsrGraph.
* ``read_csr_bin(path, device=d)`` loads the binary "CSRG" cache
  (io.py:125-170) straight into HBM: the file is memory-mapped and streamed
  through the narrowing upload, no int64 copies in between; without
  ``device`` it returns a host CsrGraph like the reference.
* ``write_csr_bin`` writes that cache format byte for byte.
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib
from .graph import INDEX_DTYPE, CsrGraph, DeviceCsrGraph

BIN_MAGIC = b"CSRG"
BIN_VERSION = 1


class ParseError(ValueError):
    """Malformed graph file; the message carries the file path and line number (io.py:17-23)."""

    def __init__(self, path, line_no: int | None, message: str):
        loc = f"{path}" if line_no is None else f"{path}:{line_no}"
        super().__init__(f"{loc}: {message}")
        self.path = str(path)
        self.line_no = line_no


def _raise_parse(path, status: int, what: str):
    msg = _lib.lib().glb_last_error().decode(errors="replace")
    if status == _lib.GLB_EPARSE:
        line, _, text = msg.partition("\t")
        ln = int(line)
        raise ParseError(path, None if ln < 0 else ln, text)
    _lib.check(status, what)


def _read_text(path, kind: int) -> CsrGraph:
    n, m, wflag = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    row, col, w = _lib._p64(), _lib._p64(), _lib._p64()
    st = _lib.lib().glb_read_text_graph(os.fsencode(path), kind, ctypes.byref(n), ctypes.byref(m),
                                        ctypes.byref(wflag), ctypes.byref(row), ctypes.byref(col),
                                        ctypes.byref(w))
    if st != _lib.GLB_OK:
        _raise_parse(path, st, "glb_read_text_graph")
    try:
        def take(p, count):
            out = np.empty(count, dtype=INDEX_DTYPE)
            if count:
                ctypes.memmove(out.ctypes.data, p, count * 8)
            return out

        rows = take(row, n.value + 1)
        cols = take(col, m.value)
        wts = take(w, m.value) if wflag.value else None
    finally:
        for p in (row, col, w):
            if p:
                _lib.lib().glb_free(ctypes.cast(p, ctypes.c_void_p))
    return CsrGraph(n.value, m.value, rows, cols, wts)


def load_dimacs_gr(path) -> CsrGraph:
    """9th-DIMACS `.gr` file: `c` comments, one `p sp <nodes> <arcs>` line,
    `a <src> <dst> <weight>` arcs with 1-based ids (io.py:26-81)."""
    return _read_text(path, 0)


def load_edge_list(path, weighted: bool = False) -> CsrGraph:
    """Whitespace-separated `u v [w]` lines, `#` comments; node count is
    max id + 1; without ``weighted`` the weight column is ignored (io.py:84-122)."""
    return _read_text(path, 2 if weighted else 1)


def write_csr_bin(g: CsrGraph, path) -> None:
    """The binary CSR cache (io.py:125-138): magic, version u32, N u64, E u64,
    row_offsets, col_indices, a weights flag byte, weights; little-endian int64."""
    with open(path, "wb") as fh:
        fh.write(BIN_MAGIC)
        fh.write(struct.pack("<I", BIN_VERSION))
        fh.write(struct.pack("<QQ", g.num_nodes, g.num_edges))
        fh.write(np.asarray(g.row_offsets).astype("<i8").tobytes())
        fh.write(np.asarray(g.col_indices).astype("<i8").tobytes())
        if g.weights is None:
            fh.write(struct.pack("<B", 0))
        else:
            fh.write(struct.pack("<B", 1))
            fh.write(np.asarray(g.weights).astype("<i8").tobytes())


def read_csr_bin(path, device: int | None = None):
    """Read the binary CSR cache (io.py:141-170).  With ``device`` the file goes
    straight to HBM and a DeviceCsrGraph comes back (no host arrays)."""
    if device is not None:
        h = ctypes.c_void_p()
        st = _lib.lib().glb_graph_load_csrg(os.fsencode(path), int(device), ctypes.byref(h))
        if st != _lib.GLB_OK:
            _raise_parse(path, st, "glb_graph_load_csrg")
        n, m, wflag = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _lib.check(_lib.lib().glb_graph_info(h, ctypes.byref(n), ctypes.byref(m),
                                             ctypes.byref(wflag), None))
        return DeviceCsrGraph(h.value, n.value, m.value, bool(wflag.value), int(device))
    data = open(path, "rb").read()
    if data[:4] != BIN_MAGIC:
        raise ParseError(path, None, "bad magic, not a CSR cache file")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != BIN_VERSION:
        raise ParseError(path, None, f"unsupported cache version {version}")
    n, m = struct.unpack_from("<QQ", data, 8)
    off = 24
    rows = np.frombuffer(data, dtype="<i8", count=n + 1, offset=off)
    off += (n + 1) * 8
    cols = np.frombuffer(data, dtype="<i8", count=m, offset=off)
    off += m * 8
    if off >= len(data):
        raise ParseError(path, None, "truncated cache file")
    flag = data[off]
    off += 1
    weights = np.frombuffer(data, dtype="<i8", count=m, offset=off) if flag else None
    return CsrGraph(int(n), int(m), rows.astype(INDEX_DTYPE), cols.astype(INDEX_DTYPE),
                    None if weights is None else weights.astype(INDEX_DTYPE))
