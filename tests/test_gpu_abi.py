"""-m gpu: boundary behaviour of libgcr through the C-ABI -- the phase machine
(S:161), the lock timeout with rollback, registry
validation (R-2) and stats."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def test_phase_machine_rejects_every_illegal_pair(G):
    gcr, _ = G
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda").fill_(7)
    ctx = gcr.Context(0)
    h = ctx.h
    try:
        ctx.register_tensor(t)
        img_ptr = C.c_void_p()
        aid = C.c_uint32()

        def calls():
            return {
                "register": lambda: gcr.gcr_register(h, t.data_ptr() + (1 << 19), 16, C.byref(aid)),
                "unregister": lambda: gcr.gcr_unregister(h, 999),
                "watch": lambda: gcr.gcr_watch_stream(h, None),
                "reserve": lambda: gcr.gcr_reserve_host(h, 0),
                "lock": lambda: gcr.gcr_lock(h),
                "checkpoint": lambda: gcr.gcr_checkpoint(h, 0, C.byref(img_ptr)),
                "unlock": lambda: gcr.gcr_unlock(h),
            }
        legal = {gcr.GCR_RUNNING: {"register", "unregister", "watch", "reserve", "lock"},
                 gcr.GCR_LOCKED: {"checkpoint", "unlock"},
                 gcr.GCR_CHECKPOINTED: {"unlock"}}
        # illegal calls change nothing
        for phase, setup in ((gcr.GCR_RUNNING, []), (gcr.GCR_LOCKED, ["lock"]),
                             (gcr.GCR_CHECKPOINTED, ["lock", "checkpoint"])):
            assert ctx.phase() == gcr.GCR_RUNNING
            for name in setup:
                assert calls()[name]() == gcr.GCR_OK
            assert ctx.phase() == phase
            for name, f in calls().items():
                if name in legal[phase]:
                    continue
                assert f() == gcr.GCR_E_STATE, (phase, name)
                assert ctx.phase() == phase
            if phase != gcr.GCR_RUNNING:
                assert gcr.gcr_unlock(h) == gcr.GCR_OK
        # restore from RUNNING is illegal
        ctx.lock()
        img = ctx.checkpoint()
        ctx.unlock()
        assert ctx.try_restore([img]) == gcr.GCR_E_STATE
    finally:
        ctx.close()


def test_lock_timeout_rolls_back_and_succeeds_once_idle(G):
    """A never-completing kernel on a watched stream -> TIMEOUT after the
    configured timeout, phase RUNNING, memory unchanged; release it -> lock OK."""
    gcr, synth = G
    L = synth.synth_lib()
    hp, dp = C.c_uint64(), C.c_uint64()
    assert L.gsy_flag_alloc(C.byref(hp), C.byref(dp)) == 0
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda").fill_(9)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    ctx = gcr.Context(0, lock_timeout_ms=200)
    try:
        ctx.register_tensor(t)
        ctx.watch_stream(s.cuda_stream)
        assert L.gsy_spin_until_flag(dp.value, C.c_void_p(s.cuda_stream)) == 0
        import time
        t0 = time.perf_counter()
        st = ctx.try_lock()
        dt = time.perf_counter() - t0
        assert st == gcr.GCR_E_TIMEOUT and ctx.phase() == gcr.GCR_RUNNING
        assert 0.19 <= dt < 2.0
        L.gsy_flag_set(hp.value, 1)
        s.synchronize()
        assert ctx.try_lock() == gcr.GCR_OK
        assert (t.cpu().numpy() == 9).all()
        ctx.unlock()
    finally:
        L.gsy_flag_set(hp.value, 1)
        torch.cuda.synchronize()
        ctx.close()
        L.gsy_flag_free(hp.value)


def test_default_lock_timeout_is_ten_seconds(G):
    gcr, _ = G
    assert gcr.default_config().lock_timeout_ms == 10000


def test_register_validation(G):
    gcr, _ = G
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h = torch.empty(4096, dtype=torch.uint8).pin_memory()
    ctx = gcr.Context(0)
    try:
        base = t.data_ptr()
        bad = [(base + 8, 4096), (base, 4100), (base, 0), (0, 4096), (h.data_ptr(), 4096)]
        for dptr, n in bad:
            with pytest.raises(gcr.GcrError) as e:
                ctx.register(dptr, n)
            assert e.value.status == gcr.GCR_E_INVAL, (dptr - base, n)
        a = ctx.register(base, 1 << 19)
        with pytest.raises(gcr.GcrError):
            ctx.register(base + (1 << 18), 1 << 19)        # overlap
        b = ctx.register(base + (1 << 19), 1 << 19)         # adjacent is fine
        assert b == a + 1
        ctx.unregister(a)
        with pytest.raises(gcr.GcrError):
            ctx.unregister(a)
        with pytest.raises(gcr.GcrError) as e:
            ctx.lock()
            ctx.unlock()
            ctx.lock()
            ctx.checkpoint(gcr.GCR_INCREMENTAL)           # no parent yet (R-8)
        assert e.value.status == gcr.GCR_E_CHAIN
        ctx.unlock()
    finally:
        ctx.close()


def test_restore_at_new_addresses_by_allocation_index(G, orc):
    """R-14: an image restores into a registry of the same sizes at other VAs."""
    gcr, synth = G
    P = 65536
    sizes = [3 * P + 512, P]
    src = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes]
    for i, t in enumerate(src):
        synth.gpu_fill(t.data_ptr(), t.numel(), 4242, i, synth.RANDOM)
    torch.cuda.synchronize()
    a = gcr.Context(0, page_size=P)
    b = gcr.Context(0, page_size=P)
    try:
        for t in src:
            a.register_tensor(t)
        a.lock()
        s = a.checkpoint().stream()
        a.unlock()
        dst = [torch.full((n,), 0x3C, dtype=torch.uint8, device="cuda") for n in sizes]
        for t in dst:
            b.register_tensor(t)
        b.lock()
        b.restore([b.import_stream(s)])
        b.unlock()
        for x, y in zip(src, dst):
            assert torch.equal(x, y)
    finally:
        a.close()
        b.close()


def test_stats_and_launch_counter(G):
    gcr, synth = G
    P = 65536
    t = torch.empty(8 * P, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), t.numel(), 1, 0, synth.RANDOM)
    t[P:2 * P].zero_()
    ctx = gcr.Context(0, page_size=P)
    try:
        ctx.register_tensor(t)
        k0 = ctx.stats()["kernel_launches"]
        ctx.lock()
        img = ctx.checkpoint()
        s = ctx.stats()
        assert (s["pages_scanned"], s["pages_zero"], s["pages_written"], s["image_bytes"]) == (8, 1, 7, 7 * P)
        assert s["n_entries"] == 3 and s["scan_launches"] == 1 and s["kernel_launches"] > k0
        assert s["checkpoint_ns"] > 0 and s["scan_dev_ns"] > 0
        ctx.restore([img])
        s = ctx.stats()
        assert s["verify_failures"] == 0 and s["restore_h2d_bytes"] == 7 * P and s["verify_launches"] == 1
        ctx.unlock()
    finally:
        ctx.close()


def test_unwatched_lock_waits_for_non_blocking_side_streams(G):
    """No watched stream: lock must see the WHOLE device idle, including a
    torch side stream (cudaStreamNonBlocking) running a never-ending kernel ->
    TIMEOUT with phase RUNNING; once the kernel ends, lock succeeds."""
    gcr, synth = G
    L = synth.synth_lib()
    hp, dp = C.c_uint64(), C.c_uint64()
    assert L.gsy_flag_alloc(C.byref(hp), C.byref(dp)) == 0
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda").fill_(5)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()  # non-blocking w.r.t. the legacy stream
    ctx = gcr.Context(0, lock_timeout_ms=300)
    try:
        ctx.register_tensor(t)
        assert L.gsy_spin_until_flag(dp.value, C.c_void_p(s.cuda_stream)) == 0
        import time
        t0 = time.perf_counter()
        st = ctx.try_lock()
        dt = time.perf_counter() - t0
        assert st == gcr.GCR_E_TIMEOUT and ctx.phase() == gcr.GCR_RUNNING
        assert 0.29 <= dt < 3.0
        L.gsy_flag_set(hp.value, 1)
        assert ctx.try_lock() == gcr.GCR_OK  # waits for the kernel to end, well within 300 ms
        ctx.unlock()
    finally:
        L.gsy_flag_set(hp.value, 1)
        torch.cuda.synchronize()
        ctx.close()
        L.gsy_flag_free(hp.value)


def test_checkpoint_abort_restores_the_parent_state(G, orc):
    """gcr_checkpoint_abort undoes the last checkpoint: image freed, phase
    LOCKED, generation re-issued, and the next incremental diffs against the
    parent from BEFORE the aborted checkpoint."""
    gcr, synth = G
    P = 65536
    t = torch.empty(8 * P, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), t.numel(), 5, 0, synth.RANDOM)
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P)
    try:
        ctx.register_tensor(t)
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        synth.gpu_xor_u32(t.data_ptr() + 2 * P, 1)
        torch.cuda.synchronize()
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        assert inc.header().generation == 2 and inc.header().n_present == 1
        ctx.checkpoint_abort(inc)
        assert ctx.phase() == gcr.GCR_LOCKED
        # abort only the LAST checkpoint's image, only from CHECKPOINTED
        assert gcr.gcr_checkpoint_abort(ctx.h, full.handle) == gcr.GCR_E_STATE
        ctx.unlock()
        synth.gpu_xor_u32(t.data_ptr() + 5 * P, 1)  # another page: both now differ from `full`
        torch.cuda.synchronize()
        ctx.lock()
        inc2 = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        h = inc2.header()
        assert h.generation == 2 and h.parent_generation == 1 and h.n_present == 2
        assert gcr.gcr_checkpoint_abort(ctx.h, full.handle) == gcr.GCR_E_INVAL
        ref = t.cpu().numpy().copy()
        t.fill_(0xA5)
        ctx.restore([full, inc2])
        assert np.array_equal(t.cpu().numpy(), ref)
        ctx.unlock()
    finally:
        ctx.close()
