"""-m gpu, BASELINE.json's full sizes in the launch configuration bench.py times
(default 1 GiB chunks, 2 copy streams, default direct_min): EVERY output is
compared with the oracle -- every page's digest and class, the whole pagemap,
every image byte, the header and meta CRC -- by the slice-wise harness in
tests/fullsize_check.py, from the CPU twin of the
generator; restores are checked byte for byte against the CPU twin."""
import pytest

import fullsize_check as fc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _registered(ctx, ts):
    return [(ctx.register_tensor(t), t.data_ptr(), t.numel()) for t in ts]


def test_c3_llama8b_zero_shard_full_size(G, orc):
    """C3: Llama-3 8B ZeRO-3 shard, 16,060,522,496 B in 5 allocations: every
    page's digest and class, the whole pagemap, every image byte, header and
    meta CRC vs the oracle; restore into poison reproduces every byte."""
    gcr, synth = G
    w = synth.make_workload("C3")
    assert w.total_bytes == 16_060_522_496
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)
    try:
        reg = _registered(ctx, ts)
        ctx.reserve_host(w.total_bytes + (256 << 20))
        ctx.lock()
        img = ctx.checkpoint()
        h = img.header()
        assert h.n_zero == 0 and h.n_present == h.n_pages == 245_069 and h.image_bytes == w.total_bytes
        fc.check_image_full(orc, w, img, reg)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0
        fc.check_memory_full(w, ts)
        ctx.unlock()
    finally:
        ctx.close()


def test_c4_incremental_40gib_exact_and_chain(G, orc):
    """C4: 40 x 1 GiB, full checkpoint, 1% of pages dirtied (XOR of one non-zero
    word each), incremental.  Both images are compared with the oracle page by
    page (the incremental diffs against the ORACLE's digests of the full
    image); the chain [full, inc] restored into poison reproduces every byte."""
    gcr, synth = G
    w = synth.make_workload("C4", gib=40)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)
    try:
        reg = _registered(ctx, ts)
        R = w.total_bytes
        ctx.reserve_host(2 * R + (2 << 30))
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        d0 = fc.check_image_full(orc, w, full, reg, generation=1)
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
        fc.check_image_full(orc, w, inc, reg, mode=1, d_prev=d0, generation=2, parent_generation=1)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([full, inc])
        assert ctx.stats()["verify_failures"] == 0
        fc.check_memory_full(w, ts)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 2097152])
def test_c5_16gib_zero_regions(G, orc, P):
    """C5: 16 GiB, 25% zero on 2 MiB-aligned regions -> z = 25% exactly at every
    P; every page, the whole pagemap and image vs the oracle; restore into
    poison (zero fill of the ZERO runs) reproduces every byte."""
    gcr, synth = G
    w = synth.make_workload("C5", gib=16, page_size=P)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = _registered(ctx, ts)
        ctx.reserve_host(w.total_bytes + (1 << 30))
        ctx.lock()
        img = ctx.checkpoint()
        h = img.header()
        n = (16 << 30) // P
        assert h.n_pages == n and h.n_zero == n // 4 and h.n_present == n - n // 4
        assert h.image_bytes == (16 << 30) * 3 // 4
        fc.check_image_full(orc, w, img, reg)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0
        fc.check_memory_full(w, ts)
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
