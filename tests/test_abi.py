"""CPU-only: the C-ABI libraries load and export every symbol their headers
declare; the Python binding covers every declared function (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(g(?:cr|sy)_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def built():
    from paper_2502_16631_b200 import build
    return build.build()


def test_gcr_exports_every_declared_symbol(built):
    names = _declared("gcr.h")
    assert len(names) == 32
    lib = ctypes.CDLL(built["libgcr.so"])
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_synth_exports_every_declared_symbol(built):
    names = _declared("gcr_synth.h")
    lib = ctypes.CDLL(built["libgcr_synth.so"])
    assert names and not [n for n in names if not hasattr(lib, n)]


def test_binding_covers_header(built):
    from paper_2502_16631_b200 import gcr
    assert sorted(gcr.EXPORTED) == _declared("gcr.h")


def C_sizeof(t):
    import ctypes
    return ctypes.sizeof(t)


def test_config_defaults_without_gpu(built):
    from paper_2502_16631_b200 import gcr
    cfg = gcr.default_config()
    assert (cfg.page_size, cfg.n_copy_streams, cfg.chunk_bytes, cfg.verify, cfg.lock_timeout_ms) == \
        (65536, 2, 1 << 30, 1, 10000)   # chunk: SURVEY §8(b) default 1 GiB; lock timeout: "10 seconds by default"
    assert cfg.direct_min_bytes == 16 << 20
    assert cfg.compress == 0 and C_sizeof(gcr.gcr_config) == 48
    assert gcr.gcr_config_default(None) == gcr.GCR_E_INVAL


def test_invalid_config_rejected_before_touching_cuda(built):
    import ctypes as C
    from paper_2502_16631_b200 import gcr
    h = C.c_void_p()
    for over in (dict(page_size=3000), dict(page_size=2048), dict(page_size=1 << 22), dict(n_copy_streams=0),
                 dict(chunk_bytes=65536 + 4096), dict(chunk_bytes=4 << 30),
                 dict(n_staging_slots=1), dict(n_staging_slots=17), dict(compress=2)):  # slots: 0 or n_copy_streams..16
        cfg = gcr.default_config(**over)
        assert gcr.gcr_create(0, C.byref(cfg), C.byref(h)) == gcr.GCR_E_INVAL, over


def test_null_handles(built):
    from paper_2502_16631_b200 import gcr
    assert gcr.gcr_destroy(None) == gcr.GCR_E_INVAL
    assert gcr.gcr_lock(None) == gcr.GCR_E_INVAL
    assert gcr.gcr_image_free(None) == gcr.GCR_E_INVAL
    assert gcr.gcr_release(None) == gcr.GCR_E_INVAL
    assert gcr.gcr_checkpoint_abort(None, None) == gcr.GCR_E_INVAL
    assert gcr.gcr_probe_link(None, 1 << 20, None, None) == gcr.GCR_E_INVAL
    assert gcr.gcr_mem_free(None, 0) == gcr.GCR_E_INVAL
    assert gcr.gcr_mem_alloc(None, 1 << 20, None) == gcr.GCR_E_INVAL
