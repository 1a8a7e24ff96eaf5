"""CPU pins of the oracle's f4 page codec (gcr_oracle.c orc_encode_page /
orc_decode_page; reading R-19, the byte-plane dictionary code for
the paper's "data compression").

What pins it, independently of the oracle's own loops:
* hand-derived golden pages (the coded bytes worked out by hand from R-19);
* a second implementation of R-19 from numpy library routines (np.unique for
  the dictionary, np.searchsorted for the ranks, np.packbits(bitorder="little")
  for the LSB-first fields) compared byte for byte on random pages;
* decode(encode(x)) == x on every alphabet size 1..256 and ragged lengths;
* malformed headers decode to zero pages, out-of-range codes to byte 0;
* stream level: the data section is the concatenation of the stored forms,
  image_bytes = sum of the stored lengths, restore reproduces the registry, a
  flipped data byte is caught by the verify at exactly that page.
"""
import numpy as np
import pytest


def pad16(x):
    return (x + 15) // 16 * 16


def np_encode(page: np.ndarray) -> bytes:
    """R-19 from numpy primitives (independent of gcr_oracle.c)."""
    L = page.size
    n = L // 4
    planes = page.reshape(n, 4).T  # plane k = byte k of every LE word
    hdr = np.zeros(16, np.uint8)
    secs = []
    for k in range(4):
        D, codes = np.unique(planes[k], return_inverse=True)
        d = D.size
        b = int(np.ceil(np.log2(d))) if d > 1 else 0
        sp, sr = pad16(d) + pad16((n * b + 7) // 8), pad16(n)
        if d <= 128 and sp < sr:
            hdr[k], hdr[4 + k] = b, d - 1
            dict_ = np.zeros(pad16(d), np.uint8)
            dict_[:d] = D
            bits = ((codes[:, None] >> np.arange(b)) & 1).astype(np.uint8).reshape(-1)  # field i at bits i*b..
            packed = np.packbits(bits, bitorder="little") if b else np.zeros(0, np.uint8)
            sec = np.zeros(pad16((n * b + 7) // 8), np.uint8)
            sec[:packed.size] = packed
            secs += [dict_, sec]
        else:
            hdr[k] = 8
            raw = np.zeros(sr, np.uint8)
            raw[:n] = planes[k]
            secs.append(raw)
    coded = np.concatenate([hdr] + secs)
    return coded.tobytes() if coded.size < L else page.tobytes()


def random_page(rng, L, alphabets):
    """Page whose plane k draws from `alphabets[k]` distinct random byte values."""
    n = L // 4
    cols = []
    for a in alphabets:
        vals = rng.choice(256, a, replace=False).astype(np.uint8)
        cols.append(vals[rng.integers(0, a, n)])
    return np.stack(cols, axis=1).reshape(-1).copy()


def test_golden_constant_page(orc):
    """4 KiB of 0x3F800000 (1.0f): every plane has one value -> mode 0 (no
    code bits), dictionaries 00, 00, 80, 3F -> 16 + 4 x 16 = 80 bytes."""
    page = np.full(1024, 0x3F800000, np.uint32).view(np.uint8)
    e = orc.encode_page(page)
    exp = bytes(16) + bytes([0x00]) + bytes(15) + bytes([0x00]) + bytes(15) + bytes([0x80]) + bytes(15) + \
        bytes([0x3F]) + bytes(15)
    assert e == exp
    assert np.array_equal(orc.decode_page(e, 4096), page)


def test_golden_sign_alternating_page(orc):
    """4 KiB of +1.0f, -1.0f, +1.0f, ...: plane 3 = 3F, BF, 3F, ... -> d = 2,
    b = 1, dictionary [3F, BF], code(i) = i & 1 -> bytes 0b10101010 = 0xAA;
    section = 16 (dict) + 128 (1024 one-bit codes); header modes 0,0,0,1 and
    d-1 = 0,0,0,1 -> 16 + 16 + 16 + 16 + 144 = 208 bytes."""
    w = np.where(np.arange(1024) % 2 == 0, 0x3F800000, 0xBF800000).astype(np.uint32)
    page = w.view(np.uint8)
    e = orc.encode_page(page)
    hdr = bytes([0, 0, 0, 1, 0, 0, 0, 1]) + bytes(8)
    exp = hdr + bytes(16) + bytes(16) + bytes([0x80]) + bytes(15) + bytes([0x3F, 0xBF]) + bytes(14) + b"\xAA" * 128
    assert len(e) == 208 and e == exp
    assert np.array_equal(orc.decode_page(e, 4096), page)


def test_golden_three_symbol_plane(orc):
    """Plane 0 cycles 9, 5, 7 (D = [5, 7, 9], ranks 2, 0, 1; d = 3 -> b = 2):
    the code stream is 2,0,1, 2,0,1, ... as 2-bit LSB-first fields, so the
    first byte is 2 | 0<<2 | 1<<4 | 2<<6 = 0x92, the second 0 | 1<<2 | 2<<4 |
    0<<6 = 0x24, the third 1 | 2<<2 | 0<<4 | 1<<6 = 0x49 (period 3 bytes)."""
    n = 1024
    w = np.array([9, 5, 7] * (n // 3) + [9], np.uint32)[:n] | np.uint32(0x11223300)
    e = orc.encode_page(w.view(np.uint8))
    assert e[:8] == bytes([2, 0, 0, 0, 2, 0, 0, 0])
    sec0 = e[16:16 + 16 + 256]
    assert sec0[:3] == bytes([5, 7, 9]) and sec0[3:16] == bytes(13)
    assert sec0[16:19] == bytes([0x92, 0x24, 0x49]) and sec0[19:22] == bytes([0x92, 0x24, 0x49])
    assert np.array_equal(orc.decode_page(e, 4096), w.view(np.uint8))


def test_random_and_tiny_pages_stay_raw(orc):
    rng = np.random.default_rng(1)
    page = rng.integers(0, 256, 65536, dtype=np.uint8)
    assert orc.encode_page(page) == page.tobytes()  # 4 full planes: coded > raw
    tiny = np.full(16, 7, np.uint8)                   # n = 4: S_p = 16 is not < S_r = 16
    assert orc.encode_page(tiny) == tiny.tobytes()


@pytest.mark.parametrize("L", [16, 64, 4096, 4096 + 48, 65536, 65536 - 16])
def test_matches_numpy_formulation_and_round_trips(orc, L):
    rng = np.random.default_rng(L)
    sizes = [1, 2, 3, 4, 5, 8, 9, 16, 17, 64, 127, 128, 129, 200, 256]
    for t in range(24):
        al = [int(rng.choice(sizes)) for _ in range(4)]
        al = [min(a, L // 4) for a in al]
        page = random_page(rng, L, al)
        e = orc.encode_page(page)
        assert e == np_encode(page), (L, al)
        assert len(e) == L or (len(e) % 16 == 0 and len(e) < L)
        assert np.array_equal(orc.decode_page(e, L), page), (L, al)


def test_fp32_training_state_ratio(orc):
    """fp32 weights with |w| in [2^-9, 2^-5) (synth F32_WEIGHT): the top byte
    (sign + 7 exponent bits) takes 4 values -> 2-bit codes; the other planes
    stay raw: 16 + 3 x 16384 + (16 + 4096) = 53,280 of 65,536 bytes."""
    from paper_2502_16631_b200 import synth
    page = synth.gen_words(123, 4, 0, 8192, synth.F32_WEIGHT).view(np.uint8)
    e = orc.encode_page(page)
    assert len(e) == 53280 and e[:8] == bytes([8, 8, 8, 2, 0, 0, 0, 3])


def test_malformed_headers_decode_to_zero_pages(orc):
    page = np.full(1024, 0x3F800000, np.uint32).view(np.uint8)
    e = bytearray(orc.encode_page(page))
    for off, val in [(0, 9), (3, 8), (4, 1), (9, 1), (15, 0xFF)]:
        b = bytearray(e)
        b[off] = val
        assert not orc.decode_page(bytes(b), 4096).any(), off
    assert not orc.decode_page(bytes(e[:64]), 4096).any()  # sections do not sum to the stored length
    # a code >= d restores byte 0: plane 3 of the alternating page, dictionary cut to one value
    w = np.where(np.arange(1024) % 2 == 0, 0x3F800000, 0xBF800000).astype(np.uint32).view(np.uint8)
    b = bytearray(orc.encode_page(w))
    b[3], b[7] = 1, 0  # d = 1 with b = 1 is malformed (ceil(log2 1) = 0)
    assert not orc.decode_page(bytes(b), 4096).any()


def test_compressed_stream_round_trip_and_layout(orc):
    from paper_2502_16631_b200 import synth
    P = 65536
    w = synth.Workload("T", P, 77, [synth.AllocSpec("w", 5 * P + 4096, synth.F32_WEIGHT, key=0),
                                     synth.AllocSpec("g", 2 * P, synth.F32_CONST, synth.ONE_F32, key=1),
                                     synth.AllocSpec("r", 3 * P + 48, synth.RANDOM, key=2),
                                     synth.AllocSpec("v", 4 * P, synth.F32_V, key=3)])
    w.zero_ranges = [(0, P, P), (3, 2 * P, P)]
    reg = [(i + 1, 0x7F0000000000 + (i << 30), s.nbytes) for i, s in enumerate(w.allocs)]
    cont = [w.cpu_bytes(a) for a in range(len(reg))]
    st, s = orc.checkpoint(P, reg, cont, compress=True)
    assert st == orc.OK
    v = orc.parse(s)
    h = v["header"]
    assert h["flags"] == 2 and v["stored"].size == h["n_present"]
    # data = concatenation of the stored forms of the PRESENT pages, in page order
    exp, stored = [], []
    for a, c in enumerate(cont):
        for p in range(0, c.size, P):
            pg = c[p:p + P]
            if pg.any():
                exp.append(orc.encode_page(pg))
                stored.append(len(exp[-1]))
    assert v["data"] == b"".join(exp) and list(v["stored"]) == stored and h["image_bytes"] == sum(stored)
    # uncompressed stream: same digests / pagemap; compressed data strictly smaller here
    st0, s0 = orc.checkpoint(P, reg, cont)
    v0 = orc.parse(s0)
    assert np.array_equal(v0["digests"], v["digests"]) and v0["entries"] == v["entries"]
    assert h["image_bytes"] < v0["header"]["image_bytes"]
    tgt = [np.full(r[2], 0xA5, np.uint8) for r in reg]
    st2, vf, _ = orc.restore([s], P, [r[2] for r in reg], tgt)
    assert st2 == orc.OK and vf == 0
    assert all(np.array_equal(t, c) for t, c in zip(tgt, cont))
    # a flipped data byte inside the 3rd stored page -> exactly that page fails the verify
    b = bytearray(s)
    data0 = len(s) - h["image_bytes"]
    b[data0 + stored[0] + stored[1] + 20] ^= 0x01
    tgt = [np.full(r[2], 0xA5, np.uint8) for r in reg]
    st3, vf3, fb3 = orc.restore([bytes(b)], P, [r[2] for r in reg], tgt)
    present_pages = [g for g, (a, p) in enumerate((a, p) for a, c in enumerate(cont) for p in range(0, c.size, P))
                     if cont[a][p:p + P].any()]
    assert st3 == orc.E_VERIFY and vf3 == 1 and fb3 == present_pages[2]


def test_unknown_flag_bits_are_rejected(orc):
    P = 65536
    c = np.ones(P, np.uint8)
    st, s = orc.checkpoint(P, [(1, 1 << 40, P)], [c], compress=True)
    b = bytearray(s)
    b[36] |= 4  # unknown flag bit; re-seal the meta CRC so only the flag is wrong
    meta = len(b) - orc.parse(bytes(b))["header"]["image_bytes"]
    b[88:92] = bytes(4)
    b[88:92] = int(orc.crc32c(bytes(b[:meta]))).to_bytes(4, "little")
    st2, _, _ = orc.restore([bytes(b)], P, [P], [np.zeros(P, np.uint8)])
    assert st2 == orc.E_VERSION
