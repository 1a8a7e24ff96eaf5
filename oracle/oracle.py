"""ctypes wrapper around oracle/liboracle.so (built from oracle/gcr_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only callers.  The product
package never imports this module.

Every function is a marshalling shim over the C oracle; see gcr_oracle.c for
the definitions and their citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gcr_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

# status codes / classes / flags, numeric values fixed by DESIGN.md §3
OK, E_INVAL, E_STATE, E_TIMEOUT, E_PEER, E_LAYOUT, E_CHAIN, E_CORRUPT, E_VERSION, E_VERIFY, E_NOMEM = range(11)
FULL, INCREMENTAL = 0, 1
CLASS_PRESENT, CLASS_ZERO, CLASS_PARENT = 0, 1, 2
PE_PARENT, PE_PRESENT, PE_ZERO = 1, 4, 8


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 (plain C, no SIMD intrinsics)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-Wall", "-Wextra",
                               "-o", LIB + ".tmp", SRC])
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u8p, u32p, u64p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        L.orc_crc32c.restype = C.c_uint32
        L.orc_crc32c.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_page_record.restype = None
        L.orc_page_record.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, u32p, u8p]
        L.orc_checkpoint.restype = C.c_int
        L.orc_checkpoint.argtypes = [C.c_uint32, C.c_uint32, u32p, u64p, u64p, C.POINTER(C.c_void_p),
                                     C.c_int, u32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.POINTER(C.c_void_p), u64p]
        L.orc_checkpoint_ex.restype = C.c_int
        L.orc_checkpoint_ex.argtypes = [C.c_uint32, C.c_uint32, u32p, u64p, u64p, C.POINTER(C.c_void_p),
                                        C.c_int, u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                        C.POINTER(C.c_void_p), u64p]
        L.orc_encode_page.restype = C.c_uint64
        L.orc_encode_page.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_decode_page.restype = None
        L.orc_decode_page.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.orc_restore.restype = C.c_int
        L.orc_restore.argtypes = [C.POINTER(C.c_void_p), u64p, C.c_uint32, C.c_uint32, C.c_uint32, u64p,
                                  C.POINTER(C.c_void_p), u64p, u64p]
        L.orc_free.restype = None
        L.orc_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def crc32c(data) -> int:
    """CRC32C of a bytes-like or numpy buffer."""
    a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    a = np.ascontiguousarray(a).view(np.uint8)
    return lib().orc_crc32c(C.c_void_p(_ptr(a) if a.size else None), a.size)


def page_record(page: np.ndarray, mode: int = FULL, d_prev: int = 0):
    """(digest, class) of one page -- c.1 steps 3-5."""
    page = np.ascontiguousarray(page).view(np.uint8)
    d = C.c_uint32()
    c = C.c_uint8()
    lib().orc_page_record(C.c_void_p(_ptr(page)), page.size, mode, d_prev, C.byref(d), C.byref(c))
    return d.value, c.value


def encode_page(page) -> bytes:
    """f4 stored form of one page (R-19): the coded form if shorter, else raw."""
    page = np.ascontiguousarray(page).view(np.uint8)
    out = np.zeros(max(page.size, 16), np.uint8)
    n = lib().orc_encode_page(C.c_void_p(_ptr(page)), page.size, C.c_void_p(_ptr(out)))
    return out[:n].tobytes()


def decode_page(stored: bytes, length: int) -> np.ndarray:
    src = np.frombuffer(bytes(stored) + b"\0", dtype=np.uint8)
    out = np.zeros(length, np.uint8)
    lib().orc_decode_page(C.c_void_p(_ptr(src)), len(stored), C.c_void_p(_ptr(out)), length)
    return out


def checkpoint(page_size: int, registry, contents, mode: int = FULL, d_prev=None,
               generation: int = 1, parent_generation: int = 0, compress: bool = False):
    """Canonical image stream (bytes) of the registry.

    registry: list of (alloc_id, vaddr, nbytes); contents: list of uint8 numpy
    arrays (len == nbytes each).  compress: f4 stored forms (R-19).
    Returns (status, stream_bytes or None)."""
    n = len(registry)
    ids = np.array([r[0] for r in registry], dtype=np.uint32)
    va = np.array([r[1] for r in registry], dtype=np.uint64)
    by = np.array([r[2] for r in registry], dtype=np.uint64)
    cont = [np.ascontiguousarray(c).view(np.uint8) for c in contents]
    ptrs = (C.c_void_p * n)(*[_ptr(c) for c in cont])
    if d_prev is not None:
        dp = np.ascontiguousarray(d_prev, dtype=np.uint32)
        dpp, ndp = dp.ctypes.data_as(C.POINTER(C.c_uint32)), dp.size
    else:
        dpp, ndp = None, 0
    out = C.c_void_p()
    out_len = C.c_uint64()
    st = lib().orc_checkpoint_ex(page_size, n, ids.ctypes.data_as(C.POINTER(C.c_uint32)),
                                 va.ctypes.data_as(C.POINTER(C.c_uint64)), by.ctypes.data_as(C.POINTER(C.c_uint64)),
                                 ptrs, mode, dpp, ndp, generation, parent_generation, 1 if compress else 0,
                                 C.byref(out), C.byref(out_len))
    if st != OK:
        return st, None
    try:
        data = C.string_at(out.value, out_len.value)
    finally:
        lib().orc_free(out)
    return st, data


def restore(streams, page_size: int, sizes, contents):
    """Apply a chain of streams onto contents (list of writable uint8 numpy
    arrays, modified in place).  Returns (status, verify_failures, first_bad)."""
    k = len(streams)
    bufs = [np.frombuffer(s, dtype=np.uint8) for s in streams]
    sp = (C.c_void_p * k)(*[_ptr(b) for b in bufs])
    lens = np.array([len(s) for s in streams], dtype=np.uint64)
    by = np.array(sizes, dtype=np.uint64)
    for c in contents:
        assert c.flags.writeable and c.flags.c_contiguous and c.dtype == np.uint8
    cp = (C.c_void_p * len(contents))(*[_ptr(c) for c in contents])
    vf = C.c_uint64()
    fb = C.c_uint64()
    st = lib().orc_restore(sp, lens.ctypes.data_as(C.POINTER(C.c_uint64)), k, page_size, len(sizes),
                           by.ctypes.data_as(C.POINTER(C.c_uint64)), cp, C.byref(vf), C.byref(fb))
    return st, vf.value, fb.value


# ---- stream parsing helpers for tests (pure layout) ----------
HEADER_BYTES = 96


def parse(stream: bytes) -> dict:
    """Split a canonical stream into its sections (no validation)."""
    h = np.frombuffer(stream[:HEADER_BYTES], dtype=np.uint8)
    u32 = lambda o: int(h[o:o + 4].view(np.uint32)[0])
    u64 = lambda o: int(h[o:o + 8].view(np.uint64)[0])
    hdr = dict(magic=bytes(stream[:8]), version=u32(8), page_size=u32(12), generation=u64(16),
               parent_generation=u64(24), n_allocs=u32(32), flags=u32(36), n_pages=u64(40),
               n_present=u64(48), n_zero=u64(56), n_parent=u64(64), n_entries=u64(72),
               image_bytes=u64(80), meta_crc32c=u32(88), reserved=u32(92))
    o = HEADER_BYTES
    at = np.frombuffer(stream[o:o + 24 * hdr["n_allocs"]], dtype=np.uint8); o += 24 * hdr["n_allocs"]
    pm = np.frombuffer(stream[o:o + 16 * hdr["n_entries"]], dtype=np.uint8); o += 16 * hdr["n_entries"]
    dg = np.frombuffer(stream[o:o + 4 * hdr["n_pages"]], dtype=np.uint32); o += 4 * hdr["n_pages"]
    stored = None
    if hdr["flags"] & 2:  # f4: stored length of every PRESENT page
        stored = np.frombuffer(stream[o:o + 4 * hdr["n_present"]], dtype=np.uint32); o += 4 * hdr["n_present"]
    data = stream[o:]
    pmr = pm.reshape(-1, 16)
    entries = [(int(r[0:8].view(np.uint64)[0]), int(r[8:12].view(np.uint32)[0]), int(r[12:16].view(np.uint32)[0]))
               for r in pmr]
    atr = at.reshape(-1, 24)
    allocs = [(int(r[0:8].view(np.uint64)[0]), int(r[8:16].view(np.uint64)[0]), int(r[16:20].view(np.uint32)[0]))
              for r in atr]
    return dict(header=hdr, allocs=allocs, entries=entries, digests=dg, stored=stored, data=data)
