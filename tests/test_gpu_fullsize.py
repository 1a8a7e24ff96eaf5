"""-m gpu, BASELINE.json's full sizes in the launch configuration bench.py times
(default 1 GiB chunks, 2 copy streams, default direct_min): every sampled output is
recomputed by the oracle one page at a time from the CPU twin of the
generator, and whole-image properties that hold at any
size are checked exactly (counts, Σ nr_pages, framing, meta CRC, restore)."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _page_table(sizes, P):
    """Global page index -> (alloc, page, len), for the sampled pages."""
    starts = np.concatenate([[0], np.cumsum([(n + P - 1) // P for n in sizes])])
    return starts


def _image_offsets(pagemap, sizes, P):
    """Image-data offset of every PRESENT page (walk of the pagemap)."""
    offs = {}
    cur, g = 0, 0
    e = 0
    for a, n in enumerate(sizes):
        m = (n + P - 1) // P
        p = 0
        while p < m:
            va, nr, fl = pagemap[e]
            e += 1
            for q in range(p, p + nr):
                ln = min(P, n - q * P)
                if fl == 4:
                    offs[g] = cur
                    cur += ln
                g += 1
            p += nr
    return offs, cur


def _check_sampled(orc, w, img, P, sample, rng, mode=0, d_prev=None, expect_image=True):
    sizes = [s.nbytes for s in w.allocs]
    starts = _page_table(sizes, P)
    n = int(starts[-1])
    dig = img.digests()
    h = img.header()
    assert h.n_pages == n == dig.size
    pm = img.pagemap()
    assert sum(e[1] for e in pm) == n
    offs, total = _image_offsets(pm, sizes, P)
    assert total == h.image_bytes
    data = img.data_view() if expect_image else None
    picks = rng.choice(n, min(sample, n), replace=False)
    cls_of = {4: 0, 8: 1, 1: 2}
    # class per page from the pagemap, for the picks
    flags = np.empty(n, np.uint8)
    g = 0
    for (_, nr, fl) in pm:
        flags[g:g + nr] = cls_of[fl]
        g += nr
    for gp in picks:
        a = int(np.searchsorted(starts, gp, side="right") - 1)
        p = int(gp - starts[a])
        ln = min(P, sizes[a] - p * P)
        page = w.cpu_bytes(a, p * P, ln)
        d, c = orc.page_record(page, mode, int(d_prev[gp]) if d_prev is not None else 0)
        assert dig[gp] == d, (gp, a, p)
        assert flags[gp] == c, (gp, a, p)
        if c == 0 and expect_image:
            o = offs[int(gp)]
            assert np.array_equal(data[o:o + ln], page), (gp, a, p)
    return flags


def test_c3_llama8b_zero_shard_full_size(G, orc):
    """C3: Llama-3 8B ZeRO-3 shard, 16,060,522,496 B in 5 allocations."""
    gcr, synth = G
    w = synth.make_workload("C3")
    assert w.total_bytes == 16_060_522_496
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)
    try:
        for t in ts:
            ctx.register_tensor(t)
        ctx.reserve_host(w.total_bytes + (256 << 20))
        ctx.lock()
        img = ctx.checkpoint()
        h = img.header()
        assert h.n_zero == 0 and h.n_present == h.n_pages == 245_069 and h.image_bytes == w.total_bytes
        _check_sampled(orc, w, img, w.page_size, 300, np.random.default_rng(3))
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0
        rng = np.random.default_rng(33)
        for a, t in enumerate(ts):  # sampled bytes of the restored state
            for _ in range(20):
                off = int(rng.integers(0, t.numel() // 16)) * 16
                assert np.array_equal(t[off:off + 4096].cpu().numpy(), w.cpu_bytes(a, off, min(4096, t.numel() - off)))
        ctx.unlock()
    finally:
        ctx.close()


def test_c4_incremental_40gib_exact_counts_and_chain(G, orc):
    """C4: 40 x 1 GiB, full checkpoint, 1% of pages dirtied (XOR of one non-zero
    word each), incremental: exactly the dirty pages PRESENT, every other page
    PARENT; sampled digests vs the oracle; chain restore into poison."""
    gcr, synth = G
    w = synth.make_workload("C4", gib=40)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)
    try:
        for t in ts:
            ctx.register_tensor(t)
        R = w.total_bytes
        ctx.reserve_host(2 * R + (2 << 30))
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        d0 = full.digests()
        muts = synth.dirty_mutations(w, 0.01, rng_seed=4242)
        assert len(muts) == 6554
        synth.gpu_xor_batch([ts[a].data_ptr() + o for (a, o, x) in muts], [x for (a, o, x) in muts])
        torch.cuda.synchronize()
        w.mutations = muts
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        h = inc.header()
        assert (h.n_present, h.n_parent, h.n_zero) == (6554, 655_360 - 6554, 0)
        assert h.parent_generation == full.header().generation and h.image_bytes == 6554 * 65536
        rng = np.random.default_rng(44)
        dirty = {(a, o // 65536) for (a, o, x) in muts}
        starts = _page_table([s.nbytes for s in w.allocs], 65536)
        flags = _check_sampled(orc, w, inc, 65536, 150, rng, mode=1, d_prev=d0)
        for (a, p) in list(dirty)[:100]:  # the dirty pages themselves
            assert flags[int(starts[a]) + p] == 0
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([full, inc])
        st = ctx.stats()
        assert st["verify_failures"] == 0
        for (a, o, x) in muts[:50]:
            pg = o // 65536 * 65536
            assert np.array_equal(ts[a][pg:pg + 65536].cpu().numpy(), w.cpu_bytes(a, pg, 65536))
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 2097152])
def test_c5_16gib_zero_regions(G, orc, P):
    """C5: 16 GiB, 25% zero on 2 MiB-aligned regions -> z = 25% exactly at every P."""
    gcr, synth = G
    w = synth.make_workload("C5", gib=16, page_size=P)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P)
    try:
        for t in ts:
            ctx.register_tensor(t)
        ctx.reserve_host(w.total_bytes + (1 << 30))
        ctx.lock()
        img = ctx.checkpoint()
        h = img.header()
        n = (16 << 30) // P
        assert h.n_pages == n and h.n_zero == n // 4 and h.n_present == n - n // 4
        assert h.image_bytes == (16 << 30) * 3 // 4
        _check_sampled(orc, w, img, P, 200, np.random.default_rng(P))
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 2097152])
def test_c2_whole_stream_other_page_sizes(G, orc, P):
    """C2 at the sweep's extreme page sizes: the whole stream equals the oracle's."""
    gcr, synth = G
    from gpu_util import first_diff, oracle_stream
    w = synth.make_workload("C2", page_size=P)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = [(ctx.register_tensor(t), t.data_ptr(), t.numel()) for t in ts]
        ctx.reserve_host(w.total_bytes + (256 << 20))
        cont = [w.cpu_bytes(a) for a in range(len(ts))]
        ctx.lock()
        got = ctx.checkpoint().stream()
        exp = oracle_stream(orc, P, reg, cont)
        assert got == exp, first_diff(got, exp)
        ctx.unlock()
    finally:
        ctx.close()
