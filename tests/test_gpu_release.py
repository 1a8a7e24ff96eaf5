"""-m gpu: releasing device memory at checkpoint and re-backing the SAME
addresses at restore: "releasing all GPU resources"
 and "Restore resources such as device memory back to the GPU,
memory mappings to their original addresses".

Memory comes from gcr_mem_alloc (VA reservation + physical allocation).  The
images are compared byte for byte with the oracle's stream, as everywhere;
after release the physical memory must be back with the driver (cudaMemGetInfo)
and after restore every byte must equal the checkpointed state at the
unchanged address."""
import numpy as np
import pytest

from gpu_util import first_diff, host_copies, oracle_stream, registry_of

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _blocks(ctx, synth, sizes, seed, P, zero_pages=()):
    ts = []
    for i, n in enumerate(sizes):
        t = ctx.alloc_tensor(n)
        assert t.data_ptr() % (2 * MiB) == 0 and t.numel() == n
        synth.gpu_fill(t.data_ptr(), n, seed, i, synth.RANDOM)
        ts.append(t)
    for (a, p) in zero_pages:
        ts[a][p * P:min((p + 1) * P, sizes[a])].zero_()
    torch.cuda.synchronize()
    return ts


def test_release_frees_hbm_and_restore_remaps_same_addresses(G, orc):
    gcr, synth = G
    P = 65536
    sizes = [5 * MiB + 48, 2 * MiB, 48]
    ctx = gcr.Context(0, page_size=P)
    try:
        ts = _blocks(ctx, synth, sizes, 4242, P, zero_pages=[(0, 3), (1, 0)])
        ptrs = [t.data_ptr() for t in ts]
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        exp = oracle_stream(orc, P, reg, cont)
        got = img.stream()
        assert got == exp, first_diff(got, exp)
        torch.cuda.synchronize()
        free0, _ = torch.cuda.mem_get_info()
        ctx.release()
        assert ctx.phase() == gcr.GCR_RELEASED
        s = ctx.stats()
        assert s["released_bytes"] == 6 * MiB + 2 * MiB + 2 * MiB  # granularity-rounded blocks
        free1, _ = torch.cuda.mem_get_info()
        assert free1 - free0 >= s["released_bytes"] - 2 * MiB, (free0, free1)
        # RELEASED admits only restore (and destroy): the memory is gone
        assert ctx.try_unlock() == gcr.GCR_E_STATE
        assert ctx.try_release() == gcr.GCR_E_STATE
        assert ctx.try_lock() == gcr.GCR_E_STATE
        assert ctx.phase() == gcr.GCR_RELEASED
        ctx.restore([img])
        assert ctx.phase() == gcr.GCR_LOCKED
        s = ctx.stats()
        assert s["remap_ns"] > 0 and s["verify_failures"] == 0
        free2, _ = torch.cuda.mem_get_info()
        assert free1 - free2 >= s["released_bytes"] - 2 * MiB
        for t, p, c in zip(ts, ptrs, cont):
            assert t.data_ptr() == p
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
        # the restored state is the parent of the next incremental: nothing is dirty
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        h = inc.header()
        assert h.n_present == 0 and h.n_zero + h.n_parent == h.n_pages
        ctx.unlock()
    finally:
        ctx.close()


def test_release_then_chain_restore(G, orc):
    """full -> mutate -> incremental -> release -> restore([full, inc]) == state at inc."""
    gcr, synth = G
    P = 4096
    sizes = [3 * MiB, 2 * MiB + 4096 + 16]
    ctx = gcr.Context(0, page_size=P, chunk_bytes=1 * MiB)
    rng = np.random.default_rng(5)
    try:
        ts = _blocks(ctx, synth, sizes, 77, P, zero_pages=[(0, 1)])
        reg = registry_of(ctx, ts)
        c0 = host_copies(ts)
        ctx.lock()
        i0 = ctx.checkpoint(gcr.GCR_FULL)
        e0 = oracle_stream(orc, P, reg, c0)
        assert i0.stream() == e0
        ctx.unlock()
        for _ in range(9):
            a = int(rng.integers(0, 2))
            off = 4 * int(rng.integers(0, sizes[a] // 4))
            synth.gpu_xor_u32(ts[a].data_ptr() + off, int(rng.integers(1, 1 << 32)))
        torch.cuda.synchronize()
        c1 = host_copies(ts)
        ctx.lock()
        i1 = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        e1 = oracle_stream(orc, P, reg, c1, mode=orc.INCREMENTAL, d_prev=orc.parse(e0)["digests"].copy(),
                           generation=2, parent_generation=1)
        assert i1.stream() == e1, first_diff(i1.stream(), e1)
        ctx.release()
        # a broken chain is rejected before anything is re-mapped: still RELEASED
        assert ctx.try_restore([i1]) == gcr.GCR_E_CHAIN
        assert ctx.phase() == gcr.GCR_RELEASED
        ctx.restore([i0, i1])
        for t, c in zip(ts, c1):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_release_requires_library_memory_fully_registered(G):
    gcr, synth = G
    ctx = gcr.Context(0)
    try:
        lib_t = ctx.alloc_tensor(4 * MiB)
        torch_t = torch.empty(MiB, dtype=torch.uint8, device="cuda").fill_(3)
        lib_t.fill_(9)
        # a caller-owned (torch) allocation cannot be released by the library
        a1 = ctx.register_tensor(lib_t)
        a2 = ctx.register_tensor(torch_t)
        ctx.lock()
        ctx.checkpoint(gcr.GCR_FULL)
        assert ctx.try_release() == gcr.GCR_E_INVAL
        assert ctx.phase() == gcr.GCR_CHECKPOINTED
        ctx.unlock()
        ctx.unregister(a2)
        # a block only partly registered would lose its other bytes
        ctx.unregister(a1)
        ctx.register(lib_t.data_ptr(), 2 * MiB)
        ctx.lock()
        ctx.checkpoint(gcr.GCR_FULL)
        assert ctx.try_release() == gcr.GCR_E_INVAL
        assert ctx.phase() == gcr.GCR_CHECKPOINTED
        ctx.unlock()
        # registered memory cannot be freed; unregistered can
        with pytest.raises(gcr.GcrError):
            ctx.mem_free(lib_t.data_ptr())
        with pytest.raises(gcr.GcrError):
            ctx.mem_free(lib_t.data_ptr() + 4096)
        assert int(lib_t[0].item()) == 9
    finally:
        ctx.close()


def test_mem_free_returns_memory(G):
    gcr, _ = G
    ctx = gcr.Context(0)
    try:
        torch.cuda.synchronize()
        f0, _ = torch.cuda.mem_get_info()
        p = ctx.mem_alloc(64 * MiB)
        f1, _ = torch.cuda.mem_get_info()
        assert f0 - f1 >= 62 * MiB
        aid = ctx.register(p, 64 * MiB)
        ctx.unregister(aid)
        ctx.mem_free(p)
        f2, _ = torch.cuda.mem_get_info()
        assert f2 - f1 >= 62 * MiB
        with pytest.raises(gcr.GcrError):
            ctx.mem_free(p)
    finally:
        ctx.close()


def test_failed_restore_from_released_stays_released(G, orc):
    """A restore from RELEASED whose verify fails leaves the phase RELEASED
    (content not valid: unlock refused) and drops the parent digest state; a
    good restore afterwards brings the state back (no unlock onto
    undefined memory)."""
    gcr, synth = G
    P = 65536
    sizes = [3 * MiB, 2 * MiB]
    ctx = gcr.Context(0, page_size=P)
    try:
        ts = _blocks(ctx, synth, sizes, 77, P)
        registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        bad = ctx.import_stream(img.stream())
        bad.data_view()[12345] ^= 1
        ctx.release()
        assert ctx.try_restore([bad]) == gcr.GCR_E_VERIFY
        assert ctx.phase() == gcr.GCR_RELEASED
        assert ctx.try_unlock() == gcr.GCR_E_STATE
        ctx.restore([img])
        assert ctx.phase() == gcr.GCR_LOCKED
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_alloc_tensor_keeps_the_context_alive(G):
    gcr, synth = G
    import gc
    ctx = gcr.Context(0)
    t = ctx.alloc_tensor(4 * MiB)
    del ctx
    gc.collect()
    t.fill_(3)  # the memory is still mapped: the tensor holds the ctx
    torch.cuda.synchronize()
    assert int(t[4 * MiB - 1].item()) == 3
