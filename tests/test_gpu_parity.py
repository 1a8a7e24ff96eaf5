"""-m gpu: the CUDA path (through the C-ABI) against the oracle, element by
element, on the same seeded inputs (SURVEY §8(c) c.4 row 'GPU vs oracle').

Bit-exact is the bar: every stream byte (header, alloc table, pagemap,
digests, data) and every restored byte.  Integer/GF(2) arithmetic only, so
there is no tolerance."""
import numpy as np
import pytest

from gpu_util import first_diff, host_copies, oracle_stream, registry_of

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _mk(G, sizes, seed, kinds=None, zero_pages=(), P=65536):
    """Allocate + fill tensors: sizes in bytes; zero_pages = [(alloc, page)]."""
    gcr, synth = G
    ts = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, seed, i, kinds[i] if kinds else synth.RANDOM)
        ts.append(t)
    for (a, p) in zero_pages:
        ts[a][p * P:min((p + 1) * P, sizes[a])].zero_()
    torch.cuda.synchronize()
    return ts


@pytest.mark.parametrize("kind", range(7))
def test_gpu_generator_matches_cpu_twin(G, kind):
    gcr, synth = G
    n = 1 << 20
    t = torch.empty(n + 4096, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), n + 4096, 1234567, 3, kind, synth.ONE_F32)
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    exp = synth.gen_words(1234567, 3, 0, (n + 4096) // 8, kind, synth.ONE_F32).view(np.uint8)
    assert np.array_equal(got, exp)
    # any sub-range (counter-based)
    exp2 = synth.gen_words(1234567, 3, 1000, 77, kind, synth.ONE_F32).view(np.uint8)
    assert np.array_equal(got[8000:8000 + 77 * 8], exp2)


ALWAYS_STAGED = (1 << 64) - 1
DIRECT_MINS = [0, 1 << 20, ALWAYS_STAGED]   # every run direct / 1 MiB / every run staged


def _ckpt_restore_parity(G, orc, sizes, P, zero_pages=(), chunk=None, streams=2, seed=99, direct_min=1 << 20,
                         slots=0):
    gcr, synth = G
    ts = _mk(G, sizes, seed, zero_pages=zero_pages, P=P)
    cfg = dict(page_size=P, n_copy_streams=streams, direct_min_bytes=direct_min, n_staging_slots=slots)
    if chunk:
        cfg["chunk_bytes"] = chunk
    ctx = gcr.Context(0, **cfg)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        got = img.stream()
        exp = oracle_stream(orc, P, reg, cont, generation=1)
        assert got == exp, first_diff(got, exp)
        for t in ts:
            t.fill_(0xA5)
        st = ctx.stats()
        assert st["direct_bytes"] <= st["image_bytes"]
        if direct_min == 0 and P >= 65536:  # every PRESENT page is a whole tile (or slices of one)
            assert st["direct_bytes"] == st["image_bytes"]
        if direct_min == ALWAYS_STAGED:
            assert st["direct_bytes"] == 0
        ctx.restore([img])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        st = ctx.stats()
        assert st["verify_failures"] == 0
        if direct_min == 0:
            assert st["restore_direct_bytes"] == st["restore_h2d_bytes"]
        if direct_min == ALWAYS_STAGED:
            assert st["restore_direct_bytes"] == 0
        ctx.unlock()
        img.free()
    finally:
        ctx.close()


def test_c1_full_parity_and_round_trip(G, orc):
    """C1: one 64 MiB region as 4 contiguous allocations, 64 KiB pages, 25% zero."""
    gcr, synth = G
    w = synth.make_workload("C1")
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)
    try:
        reg = registry_of(ctx, ts)
        cont = [w.cpu_bytes(a) for a in range(len(ts))]
        for t, c in zip(ts, cont):  # the generator twin and the device agree
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.lock()
        img = ctx.checkpoint()
        h = img.header()
        assert (h.n_pages, h.n_present, h.n_zero, h.image_bytes) == (1024, 768, 256, 50_331_648)
        got = img.stream()
        exp = oracle_stream(orc, w.page_size, reg, cont)
        assert got == exp, first_diff(got, exp)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("direct_min", DIRECT_MINS)
@pytest.mark.parametrize("P", [4096, 8192, 16384, 32768, 65536, 131072, 262144, 2097152])
def test_page_sizes_tails_and_zero_pages(G, orc, P, direct_min):
    """Several tiles and a ragged tail per allocation at every page-size regime
    (group-owned pages, 2 groups/page, 4 groups/page, 64 KiB slices)."""
    rng = np.random.default_rng(P)
    sizes = []
    for i in range(5):
        pages = int(rng.integers(1, 9)) if P >= 131072 else int(rng.integers(1, 40))
        tail = int(rng.integers(0, P // 16)) * 16
        sizes.append(pages * P + tail if tail else pages * P)
    sizes += [16, 48, P + 16]  # degenerate small allocations
    zp = []
    for a, n in enumerate(sizes):
        m = (n + P - 1) // P
        for p in range(m):
            if rng.random() < 0.3:
                zp.append((a, p))
    _ckpt_restore_parity(G, orc, sizes, P, zero_pages=zp, seed=P + 1, direct_min=direct_min)


@pytest.mark.parametrize("mode", ["0", "2"])
@pytest.mark.parametrize("P", [4096, 65536, 262144])
def test_copy_kernel_variants(G, orc, P, mode, monkeypatch):
    """Default: K6 through the TMA bulk-copy ring, K4 as the vector copy.
    GCR_TMA_COPY=0: both vector copies; =2: both through the TMA ring (the
    A/B knob).  Everything staged: every byte still the oracle's."""
    monkeypatch.setenv("GCR_TMA_COPY", mode)
    rng = np.random.default_rng(P + 7)
    sizes = [int(rng.integers(3, 30)) * P + 4096, 5 * P, 2 * P + 48, 16]
    zp = [(0, 1), (1, 2), (1, 3)]
    _ckpt_restore_parity(G, orc, sizes, P, zero_pages=zp, seed=P + 9, direct_min=ALWAYS_STAGED)


@pytest.mark.parametrize("direct_min", [0, ALWAYS_STAGED, 256 << 10])
@pytest.mark.parametrize("chunk,streams", [(65536, 1), (131072, 3), (1 << 20, 2), (4 << 20, 8)])
def test_chunking_and_copy_streams(G, orc, chunk, streams, direct_min):
    """Many pipeline chunks (image offsets stitched across chunks, slots reused)."""
    P = 65536 if chunk >= 65536 else 4096
    sizes = [3 << 20, (5 << 20) + 4096, 64 * 1024 + 1024, 7 << 20]
    rng = np.random.default_rng(chunk)
    zp = [(a, int(p)) for a in range(4) for p in rng.choice((sizes[a] + P - 1) // P, min(3, (sizes[a] + P - 1) // P), replace=False)]
    _ckpt_restore_parity(G, orc, sizes, P, zero_pages=zp, chunk=max(chunk, P), streams=streams, seed=chunk,
                         direct_min=direct_min)


@pytest.mark.parametrize("streams,slots", [(1, 3), (2, 5), (3, 16)])
def test_more_staging_slots_than_streams(G, orc, streams, slots):
    """Chunk i packs into slot i mod n_slots (its pack waits for chunk i - n_slots's
    drain); 30+ chunks, all staged, so every slot is reused many times and the
    digests arrive in many batches (meta CRC joined from them)."""
    P = 65536
    sizes = [(9 << 20) + 4096, 3 << 20, (6 << 20) + 512, 16 + 4096]
    rng = np.random.default_rng(slots)
    zp = [(a, int(p)) for a in range(3) for p in rng.choice((sizes[a] + P - 1) // P, 5, replace=False)]
    _ckpt_restore_parity(G, orc, sizes, P, zero_pages=zp, chunk=1 << 19, streams=streams, seed=slots,
                         direct_min=ALWAYS_STAGED, slots=slots)


@pytest.mark.parametrize("groups", ["1", "0"])
@pytest.mark.parametrize("P", [4096, 8192])
def test_chunking_small_pages_many_chunks(G, orc, P, groups, monkeypatch):
    """Small pages over many chunks, partial last groups, tails: K1g page groups
    (default) and the plain K1 (GCR_SMALL_GROUPS=0) give the same stream."""
    monkeypatch.setenv("GCR_SMALL_GROUPS", groups)  # read at each layout build (lock)
    _ckpt_restore_parity(G, orc, [1 << 20, (1 << 20) + 4096 + 512, 12288, 5 * P + 16], P, chunk=65536, streams=3,
                         zero_pages=[(0, 3), (0, 4), (1, 0), (2, 1), (3, 5)], seed=5)


@pytest.mark.parametrize("ramp", ["1", "2"])
@pytest.mark.parametrize("P,chunk", [(4096, 1 << 20), (1 << 20, 8 << 20)])
def test_chunk_ramp_parity(G, orc, P, chunk, ramp, monkeypatch):
    """With GCR_CHUNK_RAMP=1 (2) a registry of >= 8 chunks gets ramped chunk sizes (1/8, 1/4, 1/2 chunk at
    both ends (at the end only), whole pages): image offsets, pagemap and digests stitched across
    chunks of every size, 4 KiB page groups (K1g) and 16-tile pages."""
    n = 9 * chunk
    sizes = [n // 2 + 16, n // 3 + 4096, n // 6 + P]
    zp = [(0, 1), (0, 2), (1, 3), (2, 0)]
    monkeypatch.setenv("GCR_CHUNK_RAMP", ramp)  # read by the library at each layout build (lock)
    _ckpt_restore_parity(G, orc, sizes, P, zero_pages=zp, chunk=chunk, streams=2, seed=77, direct_min=1 << 20)


def test_large_page_chunking(G, orc):
    P = 1 << 20
    _ckpt_restore_parity(G, orc, [5 * P + 4096, 3 * P, 2 * P + 16], P, chunk=2 * P, streams=2,
                         zero_pages=[(0, 1), (1, 2), (2, 2)], seed=6)


def _mutate(ts, rng, k, P):
    from paper_2502_16631_b200 import synth
    muts = []
    sizes = [t.numel() for t in ts]
    flat = [(a, p) for a, n in enumerate(sizes) for p in range((n + P - 1) // P)]
    for i in rng.choice(len(flat), k, replace=False):
        a, p = flat[int(i)]
        ln = min(P, sizes[a] - p * P)
        off = p * P + 4 * int(rng.integers(0, ln // 4))
        x = int(rng.integers(1, 1 << 32))
        synth.gpu_xor_u32(ts[a].data_ptr() + off, x)
        muts.append((a, p))
    torch.cuda.synchronize()
    return muts


@pytest.mark.parametrize("direct_min", [0, ALWAYS_STAGED])
@pytest.mark.parametrize("P", [4096, 8192, 65536, 262144])
def test_incremental_chain_parity(G, orc, P, direct_min):
    """Full, then two incrementals with exact dirty counts; every stream equals
    the oracle's; restore(I0, I1, I2) into poison == state at I2."""
    gcr, synth = G
    rng = np.random.default_rng(P + 7)
    sizes = [40 * P + 1024, 17 * P, 3 * P + 16]
    ts = _mk(G, sizes, 31, zero_pages=[(0, 2), (1, 5)], P=P)
    ctx = gcr.Context(0, page_size=P, chunk_bytes=max(P, 4 * 65536) * 4, direct_min_bytes=direct_min)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        i0 = ctx.checkpoint(gcr.GCR_FULL)
        e0 = oracle_stream(orc, P, reg, cont, generation=1)
        assert i0.stream() == e0
        dprev = orc.parse(e0)["digests"].copy()
        ctx.unlock()
        chain, states, gen = [i0], [cont], 1
        for k in (5, 11):
            _mutate(ts, rng, k, P)
            cont = host_copies(ts)
            ctx.lock()
            ii = ctx.checkpoint(gcr.GCR_INCREMENTAL)
            ei = oracle_stream(orc, P, reg, cont, mode=orc.INCREMENTAL, d_prev=dprev, generation=gen + 1,
                               parent_generation=gen)
            got = ii.stream()
            assert got == ei, first_diff(got, ei)
            h = ii.header()
            assert h.n_present + h.n_zero + h.n_parent == h.n_pages
            dprev = orc.parse(ei)["digests"].copy()
            ctx.unlock()
            gen += 1
            chain.append(ii)
            states.append(cont)
        for k in range(1, 4):
            ctx.lock()
            for t in ts:
                t.fill_(0xA5)
            ctx.restore(chain[:k])
            for t, c in zip(ts, states[k - 1]):
                assert np.array_equal(t.cpu().numpy(), c)
            ctx.unlock()
        # the next incremental after a restore diffs against the restored state
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        h = inc.header()
        assert h.n_present == 0 and h.parent_generation == chain[2].header().generation
        ctx.unlock()
    finally:
        ctx.close()


def test_cross_restore_oracle_stream_on_gpu_and_gpu_stream_on_oracle(G, orc):
    gcr, synth = G
    P = 65536
    sizes = [3 * P + 4096, 2 * P]
    ts = _mk(G, sizes, 77, zero_pages=[(0, 1)], P=P)
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        exp = oracle_stream(orc, P, reg, cont)
        ctx.lock()
        img = ctx.checkpoint()
        gs = img.stream()
        # oracle restores the GPU-written stream
        tgt = [np.full(n, 0xA5, np.uint8) for n in sizes]
        st, vf, fb = orc.restore([gs], P, sizes, tgt)
        assert (st, vf) == (orc.OK, 0)
        assert all(np.array_equal(a, b) for a, b in zip(tgt, cont))
        # the GPU restores the oracle-written stream
        imp = ctx.import_stream(exp)
        for t in ts:
            t.fill_(0x5A)
        ctx.restore([imp])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_corruption_and_validation(G, orc):
    gcr, synth = G
    P = 65536
    sizes = [4 * P, 2 * P + 512]
    ts = _mk(G, sizes, 78, zero_pages=[(0, 2)], P=P)
    ctx = gcr.Context(0, page_size=P)
    try:
        registry_of(ctx, ts)
        ctx.lock()
        img = ctx.checkpoint()
        s = img.stream()
        h = img.header()
        meta = 96 + 24 * 2 + 16 * h.n_entries + 4 * h.n_pages
        rng = np.random.default_rng(0)
        for off in list(range(0, 96)) + [int(x) for x in rng.integers(96, meta, 40)]:
            b = bytearray(s)
            b[off] ^= 0x10
            with pytest.raises(gcr.GcrError) as e:
                ctx.import_stream(bytes(b))
            assert e.value.status == gcr.GCR_E_CORRUPT, off
        # a flipped data byte: imported fine, restore reports exactly one bad page
        b = bytearray(s)
        b[meta + 100] ^= 1
        bad = ctx.import_stream(bytes(b))
        assert ctx.try_restore([bad]) == gcr.GCR_E_VERIFY
        st = ctx.stats()
        assert st["verify_failures"] == 1 and st["first_bad_page"] == 0
        # an incremental first in the chain
        ctx.restore([img])
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL) if ctx.phase() == gcr.GCR_LOCKED else None
        assert inc is not None
        assert ctx.try_restore([inc]) == gcr.GCR_E_CHAIN
        assert ctx.try_restore([img, img]) == gcr.GCR_E_CHAIN
        ctx.unlock()
        # layout mismatch: another registry
        other = gcr.Context(0, page_size=P)
        t2 = torch.empty(4 * P, dtype=torch.uint8, device="cuda")
        other.register_tensor(t2)
        other.lock()
        im2 = other.import_stream(s)
        assert other.try_restore([im2]) == gcr.GCR_E_LAYOUT
        other.unlock()
        other.close()
    finally:
        ctx.close()


def test_gpt2_small_full_size_parity(G, orc):
    """C2 at its full size (444 fp32 allocations, 1,493,277,696 B): the whole
    canonical stream equals the oracle's, then restore round-trips."""
    gcr, synth = G
    w = synth.make_workload("C2")
    assert w.total_bytes == 1_493_277_696 and len(w.allocs) == 444
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size)   # default direct_min: big tensors direct, small ones packed
    try:
        reg = registry_of(ctx, ts)
        ctx.reserve_host(w.total_bytes + (64 << 20))
        cont = [w.cpu_bytes(a) for a in range(len(ts))]
        ctx.lock()
        img = ctx.checkpoint()
        got = img.stream()
        exp = oracle_stream(orc, w.page_size, reg, cont)
        assert got == exp, first_diff(got, exp)
        st = ctx.stats()
        assert 0 < st["direct_bytes"] < st["image_bytes"]   # both drain paths used (wte, wpe... direct)
        del got, exp
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        for a in range(0, len(ts), 37):
            assert np.array_equal(ts[a].cpu().numpy(), cont[a])
        st = ctx.stats()
        assert st["verify_failures"] == 0 and 0 < st["restore_direct_bytes"] < st["restore_h2d_bytes"]
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 65536, 2097152])
def test_degenerate_all_zero_registry(G, orc, P):
    """Every page ZERO: an empty data section (image_bytes = 0), one ZERO entry
    per allocation, every digest Z(len); restore zero-fills poisoned memory."""
    gcr, _ = G
    sizes = [3 * P + 48, P, 16]
    ts = [torch.zeros(n, dtype=torch.uint8, device="cuda") for n in sizes]
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        exp = oracle_stream(orc, P, reg, host_copies(ts))
        got = img.stream()
        assert got == exp, first_diff(got, exp)
        h = img.header()
        assert h.n_present == 0 and h.image_bytes == 0 and h.n_zero == h.n_pages and h.n_entries == len(sizes)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert all(int(t.count_nonzero().item()) == 0 for t in ts)
        ctx.unlock()
    finally:
        ctx.close()


def test_degenerate_all_present_single_page_allocations(G, orc):
    """No ZERO page, one short page per allocation (every page is a tail page and
    starts an allocation): one PRESENT entry per allocation."""
    gcr, synth = G
    P = 65536
    sizes = [16 * (k + 1) for k in range(64)]
    ts = _mk(G, sizes, 4321)
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        exp = oracle_stream(orc, P, reg, cont)
        got = img.stream()
        assert got == exp, first_diff(got, exp)
        h = img.header()
        assert h.n_present == h.n_pages == len(sizes) and h.n_entries == len(sizes)
        assert h.image_bytes == sum(sizes)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()
