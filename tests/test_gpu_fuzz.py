"""-m gpu: seeded randomized configurations across the knobs that pick kernel
variants and pipeline layouts — page size (K1 / K1g), chunk size (many
chunks, slots reused), copy streams, direct-DMA threshold, f4 codec on/off,
K4 / K6 copy variant (GCR_TMA_COPY 0/1/2), restore region ring on/off
(GCR_RESTORE_RING), K1g immediate or IADD table base (GCR_GRP_IMM) — against
the oracle (gcr_oracle.c): the full and the incremental stream byte for byte,
then the chain [full, inc] and the full image alone restored into poison.
Sizes are random multiples of 16 (R-2), tiny ones included; pages are random,
constant, zero or training-state-shaped."""
import numpy as np
import pytest

from gpu_util import first_diff, host_copies, registry_of

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ALWAYS_STAGED = (1 << 64) - 1
N_CASES = 64


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    P = int(rng.choice([4096, 8192, 65536, 262144, 2097152]))
    unit = max(P, 65536)
    chunk = unit * int(rng.choice([1, 2, 3, 8, 64]))
    n_allocs = int(rng.integers(1, 7))
    sizes = []
    for _ in range(n_allocs):
        r = rng.random()
        if r < 0.15:
            sizes.append(16 * int(rng.integers(1, 64)))  # tiny
        else:
            pages = int(rng.integers(1, 12 if P >= 262144 else 40))
            tail = 16 * int(rng.integers(0, P // 16)) if rng.random() < 0.6 else 0
            sizes.append(max(16, (pages - 1) * P + (tail or P)))
    return dict(
        P=P, chunk=chunk, sizes=sizes, streams=int(rng.integers(1, 4)),
        direct_min=int(rng.choice([0, ALWAYS_STAGED, 256 << 10, 16 << 20])),
        compress=int(rng.integers(0, 2)), tma=str(int(rng.integers(0, 3))), ring=str(int(rng.integers(0, 2))),
        imm=str(int(rng.integers(0, 2))), kinds=[int(rng.integers(0, 7)) for _ in sizes],
        zero_frac=float(rng.choice([0.0, 0.1, 0.3])), dirty=int(rng.integers(1, 9)), rng=rng)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_randomized_configuration(G, orc, seed, monkeypatch):
    gcr, synth = G
    c = _case(seed)
    P, rng = c["P"], c["rng"]
    monkeypatch.setenv("GCR_TMA_COPY", c["tma"])
    monkeypatch.setenv("GCR_RESTORE_RING", c["ring"])
    monkeypatch.setenv("GCR_GRP_IMM", c["imm"])  # read by the K1g probe at context creation
    ts = []
    for i, (n, kind) in enumerate(zip(c["sizes"], c["kinds"])):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, 500 + seed, i, kind, synth.ONE_F32)
        for p in range((n + P - 1) // P):
            if rng.random() < c["zero_frac"]:
                t[p * P:min((p + 1) * P, n)].zero_()
        ts.append(t)
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P, chunk_bytes=c["chunk"], n_copy_streams=c["streams"],
                      direct_min_bytes=c["direct_min"], compress=c["compress"])
    try:
        reg = registry_of(ctx, ts)
        cont0 = host_copies(ts)
        comp = bool(c["compress"])
        ctx.lock()
        full = ctx.checkpoint(gcr.GCR_FULL)
        st, e0 = orc.checkpoint(P, reg, cont0, generation=1, compress=comp)
        assert st == orc.OK
        got = full.stream()
        assert got == e0, (c, first_diff(got, e0))
        ctx.unlock()
        # dirty a few random pages (one word each, XOR with a non-zero value)
        flat = [(a, p) for a, n in enumerate(c["sizes"]) for p in range((n + P - 1) // P)]
        for k in rng.choice(len(flat), min(c["dirty"], len(flat)), replace=False):
            a, p = flat[int(k)]
            ln = min(P, c["sizes"][a] - p * P)
            off = p * P + 4 * int(rng.integers(0, ln // 4))
            synth.gpu_xor_u32(ts[a].data_ptr() + off, int(rng.integers(1, 1 << 32)))
        torch.cuda.synchronize()
        cont1 = host_copies(ts)
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        dprev = orc.parse(e0)["digests"].copy()
        st, e1 = orc.checkpoint(P, reg, cont1, mode=orc.INCREMENTAL, d_prev=dprev, generation=2,
                                parent_generation=1, compress=comp)
        assert st == orc.OK
        got = inc.stream()
        assert got == e1, (c, first_diff(got, e1))
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([full, inc])
        assert ctx.stats()["verify_failures"] == 0
        for t, x in zip(ts, cont1):
            assert np.array_equal(t.cpu().numpy(), x), c
        for t in ts:
            t.fill_(0x5A)
        ctx.restore([full])
        assert ctx.stats()["verify_failures"] == 0
        for t, x in zip(ts, cont0):
            assert np.array_equal(t.cpu().numpy(), x), c
        ctx.unlock()
    finally:
        ctx.close()
