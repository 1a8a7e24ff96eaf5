"""-m gpu: repeated checkpoint -> poison -> restore cycles with the pipeline's
concurrency exercised at every chunk boundary: many chunks, every PRESENT run
staged through K4 (which runs beside the persistent K1 and widens when the
scan ends), scattered zero/dirty pages so tiles mix classes.  A pack that
skipped or duplicated work would put wrong bytes in the image, and the
restore's verify (every page re-digested against the checkpoint's digests,
R-11) would report it.  The last image of each mode is also compared byte for
byte with the oracle's stream."""
import numpy as np
import pytest

from gpu_util import first_diff, host_copies, oracle_stream, registry_of

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MiB = 1 << 20
ALWAYS_STAGED = (1 << 64) - 1


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


@pytest.mark.parametrize("direct_min", [ALWAYS_STAGED, 1 << 20])
def test_repeated_cycles_verify_clean(G, orc, direct_min):
    gcr, synth = G
    P = 65536
    sizes = [96 * MiB + 4096, 64 * MiB, 33 * MiB + 16, 160 * MiB, 48 * MiB + 512]
    rng = np.random.default_rng(2024)
    ts = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, 555, i, synth.RANDOM)
        ts.append(t)
    flat = [(a, p) for a, n in enumerate(sizes) for p in range((n + P - 1) // P)]
    for k in rng.choice(len(flat), len(flat) // 4, replace=False):  # 25% zero pages, scattered
        a, p = flat[int(k)]
        ts[a][p * P:min((p + 1) * P, sizes[a])].zero_()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P, chunk_bytes=32 * MiB, direct_min_bytes=direct_min)
    try:
        reg = registry_of(ctx, ts)
        ctx.reserve_host(sum(sizes) * 3)
        ctx.lock()
        base = ctx.checkpoint(gcr.GCR_FULL)
        ctx.unlock()
        for it in range(24):
            # dirty ~5% of the pages (one non-zero XOR each)
            for k in rng.choice(len(flat), len(flat) // 20, replace=False):
                a, p = flat[int(k)]
                ln = min(P, sizes[a] - p * P)
                synth.gpu_xor_u32(ts[a].data_ptr() + p * P + 4 * int(rng.integers(0, ln // 4)),
                                  int(rng.integers(1, 1 << 32)))
            torch.cuda.synchronize()
            ctx.lock()
            mode = gcr.GCR_FULL if it % 2 == 0 else gcr.GCR_INCREMENTAL
            img = ctx.checkpoint(mode)
            if mode == gcr.GCR_FULL:
                for t in ts:
                    t.fill_(0xA5)
                ctx.restore([img])  # raises GcrError(E_VERIFY) on any wrong image byte
                assert ctx.stats()["verify_failures"] == 0, it
                base.free()
                base = img
            else:
                # the incremental must restore over its full parent too
                for t in ts:
                    t.fill_(0xA5)
                ctx.restore([base, img])
                assert ctx.stats()["verify_failures"] == 0, it
                img.free()
            ctx.unlock()
        cont = host_copies(ts)
        ctx.lock()
        last = ctx.checkpoint(gcr.GCR_FULL)
        exp = oracle_stream(orc, P, reg, cont, generation=last.header().generation)
        got = last.stream()
        assert got == exp, first_diff(got, exp)
        ctx.unlock()
    finally:
        ctx.close()
