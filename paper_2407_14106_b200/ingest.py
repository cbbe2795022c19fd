"""Ingestion formats (reference proj/src/graph.cpp:68-109,
302-336, proj/src/partition.cpp:458-493) through libgte_b200's parsers
(csrc/ingest.cpp): edge-list text (multi-threaded), GTF1 binary features,
permutation text. Errors are DataError with the reference's wording."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check

VP, I64 = C.c_void_p, C.c_int64


def _bind():
    L = _lib.lib()
    if not getattr(L, "_ingest_bound", False):
        L.gte_parse_edge_list.argtypes = [C.c_char_p, I64, I64, C.POINTER(VP)]
        L.gte_edges_info.argtypes = [VP, C.POINTER(I64), C.POINTER(I64)]
        L.gte_edges_copy.argtypes = [VP, VP, VP]
        L.gte_edges_destroy.argtypes = [VP]
        L.gte_gtf1_decode.argtypes = [C.c_char_p, I64, C.POINTER(I64), C.POINTER(I64), VP]
        L.gte_gtf1_encode.argtypes = [I64, I64, VP, VP, C.POINTER(I64)]
        L.gte_parse_permutation.argtypes = [C.c_char_p, I64, C.POINTER(I64), VP, VP]
        L._ingest_bound = True
    return L


def parse_edge_list(text: bytes | str, num_nodes_hint: int | None = None):
    """-> (num_nodes, src int64, dst int64); build the CSR with
    partition.graph_from_edges (GPU)."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    L = _bind()
    h = VP()
    check(L.gte_parse_edge_list(b, len(b), -1 if num_nodes_hint is None else int(num_nodes_hint), C.byref(h)))
    try:
        n, m = I64(), I64()
        L.gte_edges_info(h, C.byref(n), C.byref(m))
        src = np.empty(max(m.value, 1), np.int64)
        dst = np.empty(max(m.value, 1), np.int64)
        L.gte_edges_copy(h, src.ctypes.data, dst.ctypes.data)
        return n.value, src[: m.value], dst[: m.value]
    finally:
        L.gte_edges_destroy(h)


def load_edge_list(path: str, num_nodes_hint: int | None = None):
    with open(path, "rb") as f:
        return parse_edge_list(f.read(), num_nodes_hint)


def decode_gtf1(data: bytes) -> np.ndarray:
    """GTF1 bytes -> float32 [N, f]."""
    L = _bind()
    n, f = I64(), I64()
    check(L.gte_gtf1_decode(data, len(data), C.byref(n), C.byref(f), None))
    out = np.empty((n.value, f.value), np.float32)
    check(L.gte_gtf1_decode(data, len(data), C.byref(n), C.byref(f), out.ctypes.data if out.size else None))
    return out


def encode_gtf1(m) -> bytes:
    a = np.ascontiguousarray(m, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("features: 2-D matrix expected")
    L = _bind()
    ln = I64()
    L.gte_gtf1_encode(a.shape[0], a.shape[1], a.ctypes.data, None, C.byref(ln))
    buf = C.create_string_buffer(ln.value)
    check(L.gte_gtf1_encode(a.shape[0], a.shape[1], a.ctypes.data, buf, C.byref(ln)))
    return buf.raw


def parse_permutation(text: bytes | str):
    """-> (forward, inverse) int64."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    L = _bind()
    n = I64()
    check(L.gte_parse_permutation(b, len(b), C.byref(n), None, None))
    fw = np.empty(max(n.value, 1), np.int64)
    iv = np.empty(max(n.value, 1), np.int64)
    check(L.gte_parse_permutation(b, len(b), C.byref(n), fw.ctypes.data, iv.ctypes.data))
    return fw[: n.value], iv[: n.value]


def format_permutation(forward) -> str:
    """partition.cpp save_permutation: "old pos" per line."""
    return "".join(f"{i} {int(p)}\n" for i, p in enumerate(np.asarray(forward)))
