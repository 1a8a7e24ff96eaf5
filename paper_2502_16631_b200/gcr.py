"""Thin ctypes binding of libgcr.so (include/gcr.h).  Argument marshalling only:
every step of the snapshot path runs in the library's sm_100a kernels.

Functions keep the C names (gcr_create, gcr_lock, ...).  `Context` and `Image`
are small conveniences that raise GcrError on a non-OK status.  There is no CPU
fallback: if libgcr.so is missing this module fails at import time.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GCR_LIBRARY") or os.path.join(PKG, "libgcr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

# ---- enums -------------------------------------------------------------------
GCR_OK, GCR_E_INVAL, GCR_E_STATE, GCR_E_TIMEOUT, GCR_E_PEER, GCR_E_LAYOUT, GCR_E_CHAIN, \
    GCR_E_CORRUPT, GCR_E_VERSION, GCR_E_VERIFY, GCR_E_NOMEM, GCR_E_CUDA, GCR_E_IO = range(13)
STATUS_NAMES = ["OK", "E_INVAL", "E_STATE", "E_TIMEOUT", "E_PEER", "E_LAYOUT", "E_CHAIN", "E_CORRUPT",
                "E_VERSION", "E_VERIFY", "E_NOMEM", "E_CUDA", "E_IO"]
GCR_IO_SYNC = 1
GCR_RUNNING, GCR_LOCKED, GCR_CHECKPOINTED, GCR_RELEASED = 0, 1, 2, 3
GCR_FULL, GCR_INCREMENTAL = 0, 1
GCR_PE_PARENT, GCR_PE_PRESENT, GCR_PE_ZERO = 1, 4, 8


class gcr_config(C.Structure):
    _fields_ = [("page_size", C.c_uint32), ("n_copy_streams", C.c_uint32), ("chunk_bytes", C.c_uint64),
                ("n_staging_slots", C.c_uint32), ("verify", C.c_uint32), ("lock_timeout_ms", C.c_uint64),
                ("direct_min_bytes", C.c_uint64), ("compress", C.c_uint32), ("in_scan_pack", C.c_uint32)]


_STAT_FIELDS = ["lock_ns", "unlock_ns", "checkpoint_ns", "restore_ns", "scan_dev_ns", "scan_launches", "scan_bytes",
                "compact_dev_ns", "pack_dev_ns", "drain_ns", "restore_h2d_ns", "scatter_dev_ns", "verify_dev_ns",
                "verify_launches", "pages_scanned", "pages_zero", "pages_parent", "pages_written", "image_bytes",
                "n_entries", "verify_failures", "first_bad_page", "restore_h2d_bytes", "kernel_launches",
                "pinned_alloc_ns", "direct_bytes", "restore_direct_bytes", "release_ns", "remap_ns",
                "released_bytes", "present_raw_bytes", "codec_dev_ns", "decode_dev_ns"]


class gcr_stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in _STAT_FIELDS]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f in _STAT_FIELDS}


class gcr_image_hdr(C.Structure):
    _fields_ = [("magic", C.c_char * 8), ("version", C.c_uint32), ("page_size", C.c_uint32),
                ("generation", C.c_uint64), ("parent_generation", C.c_uint64), ("n_allocs", C.c_uint32),
                ("flags", C.c_uint32), ("n_pages", C.c_uint64), ("n_present", C.c_uint64), ("n_zero", C.c_uint64),
                ("n_parent", C.c_uint64), ("n_entries", C.c_uint64), ("image_bytes", C.c_uint64),
                ("meta_crc32c", C.c_uint32), ("reserved", C.c_uint32)]


class gcr_alloc_rec(C.Structure):
    _fields_ = [("vaddr", C.c_uint64), ("bytes", C.c_uint64), ("alloc_id", C.c_uint32), ("reserved", C.c_uint32)]


class gcr_pagemap_entry(C.Structure):
    _fields_ = [("vaddr", C.c_uint64), ("nr_pages", C.c_uint32), ("flags", C.c_uint32)]


assert C.sizeof(gcr_image_hdr) == 96 and C.sizeof(gcr_alloc_rec) == 24 and C.sizeof(gcr_pagemap_entry) == 16

_vp, _u32, _u64 = C.c_void_p, C.c_uint32, C.c_uint64
_P = C.POINTER
_SIGS = {
    "gcr_config_default": [_P(gcr_config)],
    "gcr_create": [C.c_int, _P(gcr_config), _P(_vp)],
    "gcr_destroy": [_vp],
    "gcr_register": [_vp, _u64, _u64, _P(_u32)],
    "gcr_unregister": [_vp, _u32],
    "gcr_watch_stream": [_vp, _vp],
    "gcr_reserve_host": [_vp, _u64],
    "gcr_lock": [_vp],
    "gcr_checkpoint": [_vp, C.c_int, _P(_vp)],
    "gcr_restore": [_vp, _P(_vp), _u32],
    "gcr_unlock": [_vp],
    "gcr_get_phase": [_vp, _P(C.c_int)],
    "gcr_get_stats": [_vp, _P(gcr_stats)],
    "gcr_ctx_stream": [_vp, _P(_vp)],
    "gcr_mem_alloc": [_vp, _u64, _P(_u64)],
    "gcr_mem_free": [_vp, _u64],
    "gcr_release": [_vp],
    "gcr_checkpoint_abort": [_vp, _vp],
    "gcr_probe_link": [_vp, _u64, _P(C.c_double), _P(C.c_double)],
    "gcr_image_header": [_vp, _P(gcr_image_hdr)],
    "gcr_image_allocs": [_vp, _P(_P(gcr_alloc_rec)), _P(_u32)],
    "gcr_image_pagemap": [_vp, _P(_P(gcr_pagemap_entry)), _P(_u64)],
    "gcr_image_digests": [_vp, _P(_P(_u32)), _P(_u64)],
    "gcr_image_data": [_vp, _P(_P(C.c_uint8)), _P(_u64)],
    "gcr_image_stored": [_vp, _P(_P(_u32)), _P(_u64)],
    "gcr_image_free": [_vp],
    "gcr_image_stream_size": [_vp, _P(_u64)],
    "gcr_image_serialize": [_vp, _vp, _u64],
    "gcr_image_import": [_vp, _vp, _u64, _P(_vp)],
    "gcr_image_write_file": [_vp, C.c_char_p, _u32, _u32],
    "gcr_image_read_file": [_vp, C.c_char_p, _u32, _P(_vp)],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
    globals()[_name] = _f
gcr_last_error = _lib.gcr_last_error
gcr_last_error.argtypes = [_vp]
gcr_last_error.restype = C.c_char_p

EXPORTED = list(_SIGS) + ["gcr_last_error"]


class GcrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def default_config(**over) -> gcr_config:
    cfg = gcr_config()
    gcr_config_default(C.byref(cfg))
    for k, v in over.items():
        setattr(cfg, k, v)
    return cfg


class Image:
    """A ctx-owned snapshot image (pinned host memory)."""

    def __init__(self, ctx: "Context", handle: int):
        self.ctx = ctx
        self.handle = C.c_void_p(handle)

    def header(self) -> gcr_image_hdr:
        h = gcr_image_hdr()
        self.ctx._check(gcr_image_header(self.handle, C.byref(h)))
        return h

    def stream(self) -> bytes:
        n = C.c_uint64()
        self.ctx._check(gcr_image_stream_size(self.handle, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self.ctx._check(gcr_image_serialize(self.handle, buf, n.value))
        return buf.raw

    def digests(self):
        import numpy as np
        p = _P(_u32)()
        n = C.c_uint64()
        self.ctx._check(gcr_image_digests(self.handle, C.byref(p), C.byref(n)))
        if n.value == 0:
            return np.zeros(0, np.uint32)
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    def pagemap(self):
        p = _P(gcr_pagemap_entry)()
        n = C.c_uint64()
        self.ctx._check(gcr_image_pagemap(self.handle, C.byref(p), C.byref(n)))
        return [(p[i].vaddr, p[i].nr_pages, p[i].flags) for i in range(n.value)]

    def pagemap_array(self):
        """Zero-copy numpy structured view {vaddr u64, nr_pages u32, flags u32} of
        the pinned pagemap (valid until free)."""
        import numpy as np
        p = _P(gcr_pagemap_entry)()
        n = C.c_uint64()
        self.ctx._check(gcr_image_pagemap(self.handle, C.byref(p), C.byref(n)))
        dt = np.dtype([("vaddr", "<u8"), ("nr_pages", "<u4"), ("flags", "<u4")])
        if n.value == 0:
            return np.zeros(0, dt)
        buf = (C.c_uint8 * (16 * n.value)).from_address(C.addressof(p.contents))
        return np.frombuffer(buf, dtype=dt)

    def stored(self):
        """f4 images: stored length of every PRESENT page (numpy copy); else None."""
        import numpy as np
        p = _P(_u32)()
        n = C.c_uint64()
        self.ctx._check(gcr_image_stored(self.handle, C.byref(p), C.byref(n)))
        if not p:
            return None
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0, np.uint32)

    def data_view(self):
        """Zero-copy numpy view of the pinned image data (valid until free)."""
        import numpy as np
        p = _P(C.c_uint8)()
        n = C.c_uint64()
        self.ctx._check(gcr_image_data(self.handle, C.byref(p), C.byref(n)))
        if n.value == 0:
            return np.zeros(0, np.uint8)
        return np.ctypeslib.as_array(p, shape=(n.value,))

    def write_file(self, path: str, threads: int = 0, sync: bool = True):
        """Storage tier (f3): write the canonical stream to `path`."""
        self.ctx._check(gcr_image_write_file(self.handle, os.fsencode(path), threads, GCR_IO_SYNC if sync else 0))

    def free(self):
        if self.handle:
            self.ctx._check(gcr_image_free(self.handle))
            self.handle = C.c_void_p(None)


class Context:
    """One libgcr context per (process, device)."""

    def __init__(self, device: int = 0, **cfg):
        self.device = device
        self.cfg = default_config(**cfg)
        h = C.c_void_p()
        st = gcr_create(device, C.byref(self.cfg), C.byref(h))
        if st != GCR_OK:
            raise GcrError(st, "gcr_create failed")
        self.h = h

    def _check(self, st: int):
        if st != GCR_OK:
            raise GcrError(st, gcr_last_error(self.h).decode())
        return st

    def status(self, st: int) -> int:
        return st

    def close(self):
        if self.h:
            gcr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register(self, dptr: int, nbytes: int) -> int:
        aid = C.c_uint32()
        self._check(gcr_register(self.h, dptr, nbytes, C.byref(aid)))
        return aid.value

    def register_tensor(self, t) -> int:
        return self.register(t.data_ptr(), t.numel() * t.element_size())

    def unregister(self, aid: int):
        self._check(gcr_unregister(self.h, aid))

    def watch_stream(self, stream_handle: int):
        self._check(gcr_watch_stream(self.h, C.c_void_p(stream_handle)))

    def reserve_host(self, nbytes: int):
        self._check(gcr_reserve_host(self.h, nbytes))

    def lock(self) -> int:
        return self._check(gcr_lock(self.h))

    def try_lock(self) -> int:
        return gcr_lock(self.h)

    def checkpoint(self, mode: int = GCR_FULL) -> Image:
        out = C.c_void_p()
        self._check(gcr_checkpoint(self.h, mode, C.byref(out)))
        return Image(self, out.value)

    def checkpoint_abort(self, img: "Image"):
        """Undo the last checkpoint (CHECKPOINTED -> LOCKED); frees img."""
        self._check(gcr_checkpoint_abort(self.h, img.handle))
        img.handle = C.c_void_p(None)

    def restore(self, chain) -> int:
        arr = (C.c_void_p * len(chain))(*[im.handle.value for im in chain])
        return self._check(gcr_restore(self.h, arr, len(chain)))

    def try_restore(self, chain) -> int:
        arr = (C.c_void_p * len(chain))(*[im.handle.value for im in chain])
        return gcr_restore(self.h, arr, len(chain))

    def unlock(self):
        self._check(gcr_unlock(self.h))

    def mem_alloc(self, nbytes: int) -> int:
        """Releasable device memory (gcr_mem_alloc): returns its device address."""
        p = C.c_uint64()
        self._check(gcr_mem_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def mem_free(self, dptr: int):
        self._check(gcr_mem_free(self.h, dptr))

    def alloc_tensor(self, nbytes: int, device: int | None = None):
        """A torch uint8 CUDA tensor over fresh gcr_mem_alloc memory on the ctx's
        device (zero-copy, via __cuda_array_interface__).  The tensor keeps the
        Context alive (the memory is the ctx's); it stays valid until mem_free /
        close, and across release -> restore (the address does not change)."""
        import torch
        dptr = self.mem_alloc(nbytes)
        dev = self.device if device is None else device

        class _Mem:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (dptr, False),
                                        "version": 3, "strides": None}
        m = _Mem()
        m.ctx = self  # the tensor's base object holds the ctx: no gcr_destroy under a live tensor
        return torch.as_tensor(m, device=f"cuda:{dev}")

    def release(self):
        self._check(gcr_release(self.h))

    def try_release(self) -> int:
        return gcr_release(self.h)

    def try_unlock(self) -> int:
        return gcr_unlock(self.h)

    def phase(self) -> int:
        p = C.c_int()
        self._check(gcr_get_phase(self.h, C.byref(p)))
        return p.value

    def stats(self) -> dict:
        s = gcr_stats()
        self._check(gcr_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def stream(self) -> int:
        p = C.c_void_p()
        self._check(gcr_ctx_stream(self.h, C.byref(p)))
        return p.value or 0

    def import_stream(self, data: bytes) -> Image:
        out = C.c_void_p()
        buf = C.create_string_buffer(data, len(data))
        self._check(gcr_image_import(self.h, buf, len(data), C.byref(out)))
        return Image(self, out.value)

    def read_file(self, path: str, threads: int = 0) -> Image:
        """Storage tier (f3): a new image from a stream file."""
        out = C.c_void_p()
        self._check(gcr_image_read_file(self.h, os.fsencode(path), threads, C.byref(out)))
        return Image(self, out.value)

    def probe_link(self, nbytes: int = 1 << 30):
        """(D2H GB/s, H2D GB/s) between the image pool and a staging slot."""
        d, h = C.c_double(), C.c_double()
        self._check(gcr_probe_link(self.h, nbytes, C.byref(d), C.byref(h)))
        return d.value, h.value

    def last_error(self) -> str:
        return gcr_last_error(self.h).decode()
