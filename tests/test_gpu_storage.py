"""-m gpu: the storage tier -- "Memory write time: the time
to save the memory state to persistent storage" and restore "from
storage".  An image file is exactly the canonical stream, so a
file written by the library equals the oracle's stream byte for byte, a file
holding the oracle's stream restores on the GPU, and every framing / meta CRC
check of gcr_image_import applies to files too."""
import os

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


def _state(synth, sizes, seed, P, zero_pages):
    ts = []
    for i, n in enumerate(sizes):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        synth.gpu_fill(t.data_ptr(), n, seed, i, synth.RANDOM)
        ts.append(t)
    for (a, p) in zero_pages:
        ts[a][p * P:min((p + 1) * P, sizes[a])].zero_()
    torch.cuda.synchronize()
    return ts


@pytest.mark.parametrize("threads", [1, 8])
def test_write_read_file_round_trip(G, orc, tmp_path, threads):
    gcr, synth = G
    P = 65536
    # > 64 MiB of data so the positional I/O splits into several units
    sizes = [80 * (1 << 20) + 4096, 3 * P + 48, 16]
    ts = _state(synth, sizes, 808, P, [(0, 7), (1, 1)])
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        cont = host_copies(ts)
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        path = str(tmp_path / "img.gcr")
        img.write_file(path, threads=threads)
        exp = oracle_stream(orc, P, reg, cont)
        with open(path, "rb") as f:
            on_disk = f.read()
        assert on_disk == exp, first_diff(on_disk, exp)
        img.free()
        back = ctx.read_file(path, threads=threads)
        assert back.stream() == exp
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([back])
        for t, c in zip(ts, cont):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_oracle_written_file_restores_on_gpu_and_chains(G, orc, tmp_path):
    """Files written outside the library (the oracle's streams) restore as a chain."""
    gcr, synth = G
    P = 4096
    sizes = [40 * P + 512, 9 * P]
    ts = _state(synth, sizes, 99, P, [(0, 3)])
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        c0 = host_copies(ts)
        e0 = oracle_stream(orc, P, reg, c0, generation=1)
        c1 = [c.copy() for c in c0]
        c1[0][5 * P + 8] ^= 0x5A
        c1[1][2 * P] ^= 0x01
        e1 = oracle_stream(orc, P, reg, c1, mode=orc.INCREMENTAL, d_prev=orc.parse(e0)["digests"].copy(),
                           generation=2, parent_generation=1)
        p0, p1 = str(tmp_path / "i0"), str(tmp_path / "i1")
        for p, e in ((p0, e0), (p1, e1)):
            with open(p, "wb") as f:
                f.write(e)
        i0, i1 = ctx.read_file(p0), ctx.read_file(p1)
        assert i1.header().n_present == 2
        ctx.lock()
        for t in ts:
            t.fill_(0xA5)
        ctx.restore([i0, i1])
        for t, c in zip(ts, c1):
            assert np.array_equal(t.cpu().numpy(), c)
        ctx.unlock()
    finally:
        ctx.close()


def test_corrupt_truncated_and_missing_files(G, orc, tmp_path):
    gcr, synth = G
    P = 65536
    ts = _state(synth, [5 * P + 16], 7, P, [])
    ctx = gcr.Context(0, page_size=P)
    try:
        reg = registry_of(ctx, ts)
        e = bytearray(oracle_stream(orc, P, reg, host_copies(ts)))
        path = str(tmp_path / "x")
        for off in (0, 12, 40, 96 + 3, 96 + 24 + 5, len(e) - 5 * P - 16 - 4 * 6 + 1):  # header, allocs, pagemap, digests
            b = bytearray(e)
            b[off] ^= 0x10
            with open(path, "wb") as f:
                f.write(b)
            with pytest.raises(gcr.GcrError) as ei:
                ctx.read_file(path)
            assert ei.value.status == gcr.GCR_E_CORRUPT, off
        with open(path, "wb") as f:
            f.write(bytes(e[:-1]))  # truncated data
        with pytest.raises(gcr.GcrError) as ei:
            ctx.read_file(path)
        assert ei.value.status == gcr.GCR_E_CORRUPT
        with pytest.raises(gcr.GcrError) as ei:
            ctx.read_file(str(tmp_path / "missing"))
        assert ei.value.status == gcr.GCR_E_IO
        ctx.lock()
        img = ctx.checkpoint(gcr.GCR_FULL)
        with pytest.raises(gcr.GcrError) as ei:
            img.write_file(str(tmp_path / "no_such_dir" / "f"))
        assert ei.value.status == gcr.GCR_E_IO
        ctx.unlock()
    finally:
        ctx.close()
