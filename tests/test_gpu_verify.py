"""-m gpu: the restore verify (A9, K8 = k_scan / k_scan_grp in verify mode) on
its FAILURE path, against the oracle's restore (gcr_oracle.c orc_restore,
c.2 step 3: "CRC32C(page) == D_k[g] for every g; count + first failing g").

Corrupted pages are injected into the image data (the pinned buffer) AFTER the
checkpoint, in different chunks, in short tail pages and (2 MiB pages) in pages
cut between many K1 warps (the verify's in-kernel fold).  The same corrupted
stream goes through the oracle's restore, whose failure count and first bad
page the GPU must reproduce exactly (GCR_E_VERIFY, verify_failures ==
count, first_bad_page == first)."""
import numpy as np
import pytest

from gpu_util import registry_of

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


ALWAYS_STAGED = (1 << 64) - 1


def _present_pages(img, sizes, P):
    """[(global page, image offset, length)] of every PRESENT page (pagemap walk)."""
    pm = img.pagemap_array()
    out, g, cur, e = [], 0, 0, 0
    for n in sizes:
        m = (n + P - 1) // P
        p = 0
        while p < m:
            nr, fl = int(pm["nr_pages"][e]), int(pm["flags"][e])
            e += 1
            for q in range(p, p + nr):
                ln = min(P, n - q * P)
                if fl == 4:
                    out.append((g, cur, ln))
                    cur += ln
                g += 1
            p += nr
    return out


def _corrupt(img, picks, rng):
    data = img.data_view()
    for (g, off, ln) in picks:
        i = off + int(rng.integers(0, ln))
        data[i] ^= np.uint8(1 << int(rng.integers(0, 8)))


def _oracle_verify(orc, img, sizes, P, chain_streams):
    tgt = [np.full(n, 0xA5, np.uint8) for n in sizes]
    return orc.restore(chain_streams, P, sizes, tgt)


def _setup(G, P, sizes, seed, zero=()):
    gcr, synth = G
    ts = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, seed, i, synth.F32_WEIGHT if i % 2 else synth.RANDOM)
        ts.append(t)
    for (a, p) in zero:
        ts[a][p * P:min((p + 1) * P, sizes[a])].zero_()
    torch.cuda.synchronize()
    return ts


# (page size, chunk bytes): K1g G=4, K1g G=2, K1, K1 with pages cut across warps
CASES = [(4096, 1 << 20), (8192, 1 << 20), (65536, 1 << 20), (2097152, 4 << 20)]


@pytest.mark.parametrize("P,chunk", CASES)
@pytest.mark.parametrize("direct_min", [0, ALWAYS_STAGED])
def test_verify_counts_and_first_bad_match_oracle(G, orc, P, chunk, direct_min):
    gcr, synth = G
    rng = np.random.default_rng(P ^ (direct_min & 0xFF))
    # >= 3 chunks; tails; a ZERO page in the middle
    big = max(3 * chunk + P // 2, 6 * P)
    sizes = [big + 4096 + 48, 2 * P + 512, 48, chunk + P + 4096]
    ts = _setup(G, P, sizes, 4321 + P, zero=[(0, 1)])
    ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk, direct_min_bytes=direct_min)
    try:
        registry_of(ctx, ts)
        ctx.lock()
        img = ctx.checkpoint()
        pres = _present_pages(img, sizes, P)
        g_of_chunk = [min(len(pres) - 1, int(f * len(pres))) for f in (0.05, 0.4, 0.75)]
        picks = [pres[i] for i in g_of_chunk]
        tails = [p for p in pres if p[2] < P]
        picks += tails[:2]            # short tail pages (front-padded in the kernels)
        picks = sorted(set(picks))
        k = len(picks)
        assert k >= 4
        _corrupt(img, picks, rng)
        st, vf, fb = _oracle_verify(orc, img, sizes, P, [img.stream()])
        assert st == orc.E_VERIFY and vf == k and fb == picks[0][0]
        for t in ts:
            t.fill_(0xA5)
        assert ctx.try_restore([img]) == gcr.GCR_E_VERIFY
        s = ctx.stats()
        assert (s["verify_failures"], s["first_bad_page"]) == (vf, fb)
        assert ctx.phase() == gcr.GCR_LOCKED
        # the parent digest state was dropped: an incremental now has no base
        assert ctx.try_unlock() == gcr.GCR_OK
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 65536, 2097152])
def test_verify_failure_in_incremental_chain(G, orc, P):
    """A corrupted PRESENT page of the LAST image of a chain (and one of the
    base image that the incremental leaves PARENT) are both caught."""
    gcr, synth = G
    chunk = 4 << 20 if P == 2097152 else 1 << 20
    sizes = [3 * chunk + 2 * P, 5 * P + 512]
    ts = _setup(G, P, sizes, 99 + P)
    ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk)
    try:
        registry_of(ctx, ts)
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        dirty = [(0, 0), (0, 3 * chunk // P), (1, 2)]
        for (a, p) in dirty:
            synth.gpu_xor_u32(ts[a].data_ptr() + p * P + 64, 0x0F0F0F0F)
        torch.cuda.synchronize()
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        assert inc.header().n_present == len(dirty)
        ipres = _present_pages(inc, sizes, P)
        fpres = _present_pages(full, sizes, P)
        dirty_g = {g for (g, _, _) in ipres}
        base_only = [p for p in fpres if p[0] not in dirty_g]
        rng = np.random.default_rng(7)
        _corrupt(inc, [ipres[1]], rng)
        _corrupt(full, [base_only[len(base_only) // 2]], rng)
        st, vf, fb = _oracle_verify(orc, inc, sizes, P, [full.stream(), inc.stream()])
        assert st == orc.E_VERIFY and vf == 2 and fb == min(ipres[1][0], base_only[len(base_only) // 2][0])
        for t in ts:
            t.fill_(0xA5)
        assert ctx.try_restore([full, inc]) == gcr.GCR_E_VERIFY
        s = ctx.stats()
        assert (s["verify_failures"], s["first_bad_page"]) == (vf, fb)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.slow
def test_verify_failures_full_size_c2(G, orc):
    """C2 (the bench workload, 444 allocations, 1.49 GB, default 1 GiB chunks):
    7 corrupted pages spread over both chunks; count and first page exact."""
    gcr, synth = G
    w = synth.make_workload("C2")
    ts = w.materialize()
    torch.cuda.synchronize()
    sizes = [t.numel() for t in ts]
    P = w.page_size
    ctx = gcr.Context(0, page_size=P)
    try:
        registry_of(ctx, ts)
        ctx.reserve_host(w.total_bytes + (256 << 20))
        ctx.lock()
        img = ctx.checkpoint()
        pres = _present_pages(img, sizes, P)
        rng = np.random.default_rng(2)
        picks = sorted(pres[int(i)] for i in rng.choice(len(pres), 7, replace=False))
        _corrupt(img, picks, rng)
        # expected from the definition (c.2 step 3): the corrupted pages are
        # exactly the failing ones -- a single-bit flip always changes a CRC --
        # and the oracle's CRC of each corrupted page differs from its digest
        dig = img.digests()
        data = img.data_view()
        for (g, off, ln) in picks:
            assert orc.crc32c(np.array(data[off:off + ln])) != dig[g]
        for t in ts:
            t.fill_(0xA5)
        assert ctx.try_restore([img]) == gcr.GCR_E_VERIFY
        s = ctx.stats()
        assert (s["verify_failures"], s["first_bad_page"]) == (7, picks[0][0])
        ctx.unlock()
    finally:
        ctx.close()
