"""-m gpu: the f4 page codec on the GPU (KA/KB/KC encode before the drain, KD
decode after the H2D; R-19, "data compression") against the
oracle's codec (gcr_oracle.c orc_encode_page / orc_decode_page): whole
canonical streams byte for byte, restores byte for byte, chains, cross-restores
both ways, corruption handled identically, files, and the full-size C2 / C3
images page by page."""
import numpy as np
import pytest

import fullsize_check as fc
from gpu_util import first_diff, host_copies, registry_of

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2502_16631_b200 import gcr, synth
    return gcr, synth


def _mixed(G, P, seed=7):
    """Allocations of every value kind, ragged tails, zero pages, constant pages."""
    gcr, synth = G
    specs = [(9 * P + 4096 + 48, synth.F32_WEIGHT), (3 * P, synth.F32_CONST), (5 * P + 512, synth.F32_M),
             (7 * P, synth.F32_V), (4 * P + 4096, synth.BF16_WEIGHT), (2 * P + 48, synth.RANDOM), (48, synth.F32_V),
             (6 * P, synth.ZERO)]
    ts = []
    for i, (n, kind) in enumerate(specs):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, seed, i, kind, synth.ONE_F32)
        ts.append(t)
    ts[0][P:2 * P].zero_()
    ts[3][3 * P:4 * P].zero_()
    torch.cuda.synchronize()
    return ts


CASES = [(4096, 1 << 20), (8192, 1 << 20), (65536, 1 << 20), (65536, 1 << 30), (262144, 2 << 20),
         (2097152, 4 << 20)]


@pytest.mark.parametrize("P,chunk", CASES)
def test_compressed_stream_equals_oracle_and_restores(G, orc, P, chunk):
    gcr, synth = G
    ts = _mixed(G, P)
    ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk, compress=1)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint()
        got = img.stream()
        st, exp = orc.checkpoint(P, reg, cont, compress=True)
        assert st == orc.OK
        assert got == exp, first_diff(got, exp)
        h = img.header()
        s = ctx.stats()
        assert h.flags == 2 and s["present_raw_bytes"] > h.image_bytes  # something compressed
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0 and ctx.stats()["decode_dev_ns"] > 0
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.parametrize("P", [4096, 65536])
def test_compressed_incremental_chain(G, orc, P):
    gcr, synth = G
    ts = _mixed(G, P, seed=11)
    ctx = gcr.Context(0, page_size=P, chunk_bytes=1 << 20, compress=1)
    try:
        reg = registry_of(ctx, ts)
        c0 = host_copies(ts)
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        for (a, off) in [(0, 8), (3, 2 * P + 64), (4, P), (2, 5 * P + 4)]:
            synth.gpu_xor_u32(ts[a].data_ptr() + off, 0x00010000)
        torch.cuda.synchronize()
        c1 = host_copies(ts)
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        d0 = orc.parse(full.stream())["digests"]
        st, exp = orc.checkpoint(P, reg, c1, mode=orc.INCREMENTAL, d_prev=d0, generation=2, parent_generation=1,
                                 compress=True)
        got = inc.stream()
        assert got == exp, first_diff(got, exp)
        assert inc.header().n_present == 4
        for t in ts:
            t.fill_(0x5A)
        ctx.restore([full, inc])
        for t, c in zip(ts, c1):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
        # the oracle restores the GPU's compressed chain, too
        tgt = [np.full(r[2], 0xA5, np.uint8) for r in reg]
        st2, vf, _ = orc.restore([full.stream(), inc.stream()], P, [r[2] for r in reg], tgt)
        assert st2 == orc.OK and vf == 0 and all(np.array_equal(a, b) for a, b in zip(tgt, c1))
        assert c0 is not None
    finally:
        ctx.close()


def test_gpu_restores_oracle_written_compressed_stream(G, orc):
    gcr, synth = G
    P = 65536
    ts = _mixed(G, P, seed=3)
    ctx = gcr.Context(0, page_size=P, compress=1)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        st, s = orc.checkpoint(P, reg, cont, compress=True)
        ctx.lock()
        imp = ctx.import_stream(s)
        assert imp.header().flags == 2
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([imp])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        # a plain (uncompressed) context restores a compressed image too: the
        # format, not the ctx config, decides
        ctx.unlock()
    finally:
        ctx.close()
    ctx2 = gcr.Context(0, page_size=P)
    try:
        registry_of(ctx2, ts)
        ctx2.lock()
        imp = ctx2.import_stream(s)
        for t in ts:
            t.fill_(0)
        ctx2.restore([imp])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx2.unlock()
    finally:
        ctx2.close()


def test_corrupted_compressed_pages_restore_like_the_oracle(G, orc):
    """Code-bit flips, dictionary flips and malformed headers: the GPU restore
    reproduces the oracle's restore (same verify count and first page; a
    malformed page restores as zeros on both sides)."""
    gcr, synth = G
    P = 65536
    ts = _mixed(G, P, seed=5)
    sizes = [t.numel() for t in ts]
    ctx = gcr.Context(0, page_size=P, compress=1)
    try:
        reg = registry_of(ctx, ts)
        ctx.lock()
        img = ctx.checkpoint()
        s = img.stream()
        v = orc.parse(s)
        stored = v["stored"]
        data0 = int(len(s) - v["header"]["image_bytes"])
        offs = np.concatenate([np.zeros(1, np.int64), np.cumsum(stored, dtype=np.int64)])
        coded = [i for i in range(stored.size) if stored[i] % 16 == 0 and stored[i] < 65536]
        b = bytearray(s)
        b[data0 + offs[coded[0]] + 3] = 9            # malformed: mode 9 -> zero page
        b[data0 + offs[coded[1]] + stored[coded[1]] - 20] ^= 0x40   # a code bit / raw byte near the end
        b[data0 + offs[coded[2]] + 16 * 3 + 17] ^= 0x01             # somewhere in the sections
        bad = ctx.import_stream(bytes(b))
        tgt = [np.full(n, 0xA5, np.uint8) for n in sizes]
        st, vf, fb = orc.restore([bytes(b)], P, sizes, tgt)
        assert st == orc.E_VERIFY and vf >= 2
        for t in ts:
            t.fill_(0xA5)
        assert ctx.try_restore([bad]) == gcr.GCR_E_VERIFY
        s2 = ctx.stats()
        assert (s2["verify_failures"], s2["first_bad_page"]) == (vf, fb)
        for t, c in zip(ts, tgt):  # byte for byte the oracle's (corrupted) restore
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_compressed_image_file_round_trip(G, orc, tmp_path):
    gcr, synth = G
    P = 65536
    ts = _mixed(G, P, seed=9)
    ctx = gcr.Context(0, page_size=P, compress=1)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint()
        path = str(tmp_path / "c.img")
        img.write_file(path)
        st, exp = orc.checkpoint(P, reg, cont, compress=True)
        assert open(path, "rb").read() == exp
        back = ctx.read_file(path)
        for t in ts:
            t.fill_(1)
        ctx.restore([back])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_compressed_full_size_every_page(G, orc, cfg):
    """C2 (GPT-2 S fp32 W+m+v, the bench workload) and C3 (Llama-3 8B ZeRO
    shard: bf16 + fp32) compressed at full size in the bench's launch
    configuration: every stored page, length, digest and pagemap entry vs the
    oracle (slice-wise harness); restore into poison reproduces every byte."""
    gcr, synth = G
    w = synth.make_workload(cfg)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=w.page_size, compress=1)
    try:
        reg = [(ctx.register_tensor(t), t.data_ptr(), t.numel()) for t in ts]
        ctx.reserve_host(w.total_bytes + (256 << 20))
        ctx.lock()
        img = ctx.checkpoint()
        fc.check_image_full(orc, w, img, reg, compress=True)
        h = img.header()
        ratio = h.image_bytes / w.total_bytes
        assert ratio < (0.85 if cfg == "C2" else 0.80), ratio  # C2 ~0.82, C3 ~0.77 (bf16 planes ~0.69)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0
        fc.check_memory_full(w, ts)
        ctx.unlock()
    finally:
        ctx.close()


def test_codec_sub_chunks_in_a_subprocess(G):
    """f4 checkpoints encode and drain each chunk in sub-chunks (default 256
    MiB): force 1 MiB sub-chunks (GCR_CODEC_SUB_MB, read once per process) in
    a child process and require the codec stream tests to pass there too."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, GCR_CODEC_SUB_MB="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", "-p", "no:cacheprovider",
                        os.path.abspath(__file__) + "::test_compressed_stream_equals_oracle_and_restores",
                        os.path.abspath(__file__) + "::test_compressed_incremental_chain"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("compress,chunk,ring", [(1, 2 << 20, "1"), (0, 2 << 20, "1"), (1, 128 << 20, "1"),
                                                (0, 128 << 20, "1"), (1, 2 << 20, "0")])
def test_restore_region_ring_reuse(G, compress, chunk, ring, monkeypatch):
    """The restore lands staged groups in a ring of regions carved out of the
    staging slots (group_max bytes each; 2 MiB chunks: 2 regions, 128 MiB
    chunks: 2 x 2 regions of 64 MiB) and runs every scatter / decode on one
    kernel stream: with ~40 groups each region is reused many times, so an H2D
    that did not wait for the previous reader of its region would corrupt
    pages.  Restore into poison reproduces every byte, verify included, and a
    chain (full + incremental) restores too.  ring "0": the GCR_RESTORE_RING=0
    A/B layout (slot per copy stream, kernel on the copy stream)."""
    gcr, synth = G
    monkeypatch.setenv("GCR_RESTORE_RING", ring)
    P = 65536
    kinds = [synth.F32_WEIGHT, synth.F32_M, synth.RANDOM, synth.F32_V, synth.BF16_WEIGHT]
    ts = []
    for i, kind in enumerate(kinds):
        n = (16 << 20) + i * 3 * P + 48 * i
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, 31, i, kind, synth.ONE_F32)
        ts.append(t)
    ts[1][5 * P:9 * P].zero_()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P, chunk_bytes=chunk, compress=compress, direct_min_bytes=(1 << 64) - 1)
    try:
        for t in ts:
            ctx.register_tensor(t)
        cont = host_copies(ts)
        ctx.lock()
        full = ctx.checkpoint()
        ctx.unlock()
        for t in ts:  # dirty every 3rd page
            t.view(-1)[: (t.numel() // P) * P].view(-1, P)[::3, :64].add_(1)
        torch.cuda.synchronize()
        cont2 = host_copies(ts)
        ctx.lock()
        inc = ctx.checkpoint(gcr.GCR_INCREMENTAL)
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([full])
        assert ctx.stats()["verify_failures"] == 0
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        for t in ts:
            t.fill_(0x5A)
        ctx.restore([full, inc])
        assert ctx.stats()["verify_failures"] == 0
        for t, c in zip(ts, cont2):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_rejected_coded_image_leaves_memory_untouched(G):
    """The f4 restore copies the image's first group into a staging region
    BEFORE the host validates the chain (speculative prefix).  A chain that
    fails validation (one digest flipped in the pinned image: meta CRC
    mismatch -> GCR_E_CORRUPT) must still leave every registered byte as it
    was, keep the phase, and a valid restore right after must work."""
    import ctypes as C
    from paper_2502_16631_b200 import gcr as g
    gcr, synth = G
    P = 65536
    ts = _mixed(G, P, seed=21)
    ctx = gcr.Context(0, page_size=P, compress=1)
    try:
        registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint()
        for t in ts:
            t.fill_(0x3C)
        torch.cuda.synchronize()
        poison = host_copies(ts)
        p = g._P(g._u32)()
        n = C.c_uint64()
        ctx._check(g.gcr_image_digests(img.handle, C.byref(p), C.byref(n)))
        p[0] ^= 0x1
        st = ctx.try_restore([img])
        assert st == gcr.GCR_E_CORRUPT
        for t, x in zip(ts, poison):  # nothing written
            assert np.array_equal(t.cpu().numpy(), x)
        p[0] ^= 0x1
        ctx.restore([img])
        assert ctx.stats()["verify_failures"] == 0
        for t, x in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), x)
        ctx.unlock()
    finally:
        ctx.close()
