"""CPU checks of the full-size parity harness (tests/fullsize_check.py): the
slice-wise oracle comparison must accept the whole-registry oracle stream of the
same input and reject a stream with any one kind of defect.  Pins the harness
itself, so a green full-size GPU test means what it says."""
import numpy as np
import pytest

import fullsize_check as fc  # noqa: E402
from paper_2502_16631_b200 import synth


class StreamImage:
    """An image-like view of a canonical stream (what the GPU Image exposes)."""

    def __init__(self, s: bytes):
        from paper_2502_16631_b200 import gcr
        self.s = bytearray(s)
        self.h, self.pm, self.dg, self.st, self.data = fc.parse_stream(self.s, with_stored=True)
        self._hdr = gcr.gcr_image_hdr.from_buffer_copy(bytes(self.s[:96]))

    def header(self):
        return self._hdr

    def digests(self):
        return self.dg.copy()

    def pagemap_array(self):
        return self.pm

    def data_view(self):
        return self.data

    def stored(self):
        return None if self.st is None else self.st.copy()


def small_workload(P):
    w = synth.Workload("T", P, 0xBEEF, [
        synth.AllocSpec("a", 5 * P + 4096 + 48, synth.F32_WEIGHT, key=0),
        synth.AllocSpec("b", 3 * P, synth.RANDOM, key=1),
        synth.AllocSpec("c", 48, synth.RANDOM, key=2),
        synth.AllocSpec("d", 9 * P + 512, synth.BF16_WEIGHT, key=3)])
    w.zero_ranges = [(0, P, 2 * P), (1, 0, 3 * P), (3, 4 * P, P), (3, 9 * P, 512)]
    return w


def registry(w):
    return [(i + 1, 0x7F0000000000 + (i << 28), s.nbytes) for i, s in enumerate(w.allocs)]


@pytest.mark.parametrize("P", [4096, 65536])
@pytest.mark.parametrize("slice_pages", [1, 3, 64])
@pytest.mark.parametrize("compress", [False, True])
def test_harness_accepts_whole_oracle_stream(orc, P, slice_pages, compress):
    w = small_workload(P)
    reg = registry(w)
    cont = [w.cpu_bytes(a) for a in range(len(reg))]
    st, s = orc.checkpoint(P, reg, cont, generation=1, compress=compress)
    assert st == 0
    d0 = fc.check_image_full(orc, w, StreamImage(s), reg, slice_bytes=slice_pages * P, threads=3, compress=compress)
    assert np.array_equal(d0, fc.parse_stream(s)[2])
    # incremental over a mutated state
    w.mutations = [(0, 4 * P + 8, 0x1234), (3, 2 * P, 0xFFFF0000)]
    cont = [w.cpu_bytes(a) for a in range(len(reg))]
    st, s2 = orc.checkpoint(P, reg, cont, mode=1, d_prev=d0, generation=2, parent_generation=1, compress=compress)
    assert st == 0
    fc.check_image_full(orc, w, StreamImage(s2), reg, mode=1, d_prev=d0, generation=2, parent_generation=1,
                        slice_bytes=slice_pages * P, threads=2, compress=compress)


@pytest.mark.parametrize("defect", ["digest", "data", "pagemap", "header", "generation", "stored"])
def test_harness_rejects_defects(orc, defect):
    P = 4096
    w = small_workload(P)
    reg = registry(w)
    cont = [w.cpu_bytes(a) for a in range(len(reg))]
    st, s = orc.checkpoint(P, reg, cont, generation=1, compress=True)
    im = StreamImage(s)
    gen = 1
    if defect == "digest":
        im.dg[7] ^= 1
    elif defect == "data":
        im.data[im.data.size // 2] ^= 0x80
    elif defect == "pagemap":
        pm = im.pm.copy()
        i = int(np.flatnonzero(pm["flags"] == 4)[0])
        pm["flags"][i] = 8
        im.pm = pm
    elif defect == "header":
        im._hdr.meta_crc32c ^= 1
    elif defect == "stored":
        st2 = im.st.copy()
        i, j = 0, int(np.flatnonzero(st2 != st2[0])[0])
        st2[i], st2[j] = st2[j], st2[i]  # same total, wrong per-page lengths
        im.st = st2
    else:
        gen = 2
    with pytest.raises(AssertionError):
        fc.check_image_full(orc, w, im, reg, generation=gen, slice_bytes=2 * P, threads=2, compress=True)
