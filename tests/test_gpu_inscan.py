"""-m gpu: f1, the in-scan pack (gcr_config.in_scan_pack): the
scan kernel writes every PRESENT page straight into the pinned image (mapped
memory) at offsets from per-CTA aggregates and K2's per-chunk base.  The image
must be byte-identical to the oracle's and to the staged pipeline's
(in_scan_pack = 0) -- for incremental checkpoints (the default path) and, with
in_scan_pack = 2, for full checkpoints at 100 % PRESENT (every page written
by the scan), over many chunks, K1 and K1g, pages cut across warps (2 MiB),
ragged tails and zero pages."""
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


def _state(G, P, chunk, seed):
    gcr, synth = G
    sizes = [3 * chunk + 5 * P + 4096 + 48, 2 * P + 512, 48, chunk + 3 * P, 7 * P + 4096]
    ts = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, seed, i, synth.RANDOM)
        ts.append(t)
    ts[0][P:2 * P].zero_()
    ts[3][0:P].zero_()
    torch.cuda.synchronize()
    return ts


CASES = [(4096, 1 << 20), (8192, 1 << 20), (65536, 1 << 20), (65536, 4 << 20), (2097152, 4 << 20)]


@pytest.mark.parametrize("P,chunk", CASES)
@pytest.mark.parametrize("isp", [1, 2])
def test_in_scan_pack_chain_equals_oracle(G, orc, P, chunk, isp):
    gcr, synth = G
    ts = _state(G, P, chunk, 31 + P)
    ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk, in_scan_pack=isp)
    try:
        reg = registry_of(ctx, ts)
        c0 = host_copies(ts)
        ctx.lock()
        full = ctx.checkpoint()
        got = full.stream()
        exp = oracle_stream(orc, P, reg, c0, generation=1)
        assert got == exp, first_diff(got, exp)
        ctx.unlock()
        rng = np.random.default_rng(P + isp)
        chain, cont = [full], c0
        for gen in (2, 3):
            for _ in range(int(rng.integers(5, 40))):  # dirty pages all over (every chunk)
                a = int(rng.integers(0, len(ts)))
                off = int(rng.integers(0, ts[a].numel() // 4)) * 4
                synth.gpu_xor_u32(ts[a].data_ptr() + off, int(rng.integers(1, 1 << 32)))
            torch.cuda.synchronize()
            prev = orc.parse(chain[-1].stream())["digests"]
            cont = host_copies(ts)
            ctx.lock()
            inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
            got = inc.stream()
            exp = oracle_stream(orc, P, reg, cont, mode=orc.INCREMENTAL, d_prev=prev, generation=gen,
                                parent_generation=gen - 1)
            assert got == exp, first_diff(got, exp)
            assert ctx.stats()["direct_bytes"] == 0
            ctx.unlock()
            chain.append(inc)
        for t in ts:
            t.fill_(0xA5)
        ctx.lock()
        ctx.restore(chain)
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 65536])
def test_in_scan_pack_matches_staged_pipeline_many_dirty(G, P):
    """25 % dirty pages over 9 chunks: in_scan_pack 1 and 0 give the same stream."""
    gcr, synth = G
    chunk = 1 << 20
    ts = _state(G, P, chunk, 77)
    streams = []
    for isp in (0, 1):
        for t, i in zip(ts, range(len(ts))):
            synth.gpu_fill(t.data_ptr(), t.numel(), 77, i, synth.RANDOM)
        torch.cuda.synchronize()
        ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk, in_scan_pack=isp)
        try:
            registry_of(ctx, ts)
            ctx.lock()
            ctx.checkpoint().free()
            ctx.unlock()
            rng = np.random.default_rng(5)
            n_pages = sum((t.numel() + P - 1) // P for t in ts)
            for _ in range(n_pages // 4):
                a = int(rng.integers(0, len(ts)))
                off = int(rng.integers(0, ts[a].numel() // 4)) * 4
                synth.gpu_xor_u32(ts[a].data_ptr() + off, 0x5A5A5A5A)
            torch.cuda.synchronize()
            ctx.lock()
            streams.append(ctx.checkpoint(gcr.GCR_INCREMENTAL).stream())
            ctx.unlock()
        finally:
            ctx.close()
    assert streams[0] == streams[1], first_diff(streams[0], streams[1])
