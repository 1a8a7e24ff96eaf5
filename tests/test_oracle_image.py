"""Pins for the oracle's checkpoint/restore:
brute force on tiny registries, constructed special cases with exact counts,
and invariants (round trip, chains, corruption, cross-page-size identity).
Independent helpers: tests/helpers/hwcrc.c (SSE4.2) and tests/gf2.py."""
import itertools

import numpy as np
import pytest

import gf2

P4K = 4096


def _rand(rng, n):
    a = rng.integers(0, 256, n, dtype=np.uint8)
    if n >= 16:  # guarantee non-zero
        a[0] |= 1
    return a


def _pages(nbytes, P):
    return [(p * P, min(P, nbytes - p * P)) for p in range((nbytes + P - 1) // P)]


def _naive_expect(registry, contents, P, classes_of_page, hwcrc):
    """Naive formulation: one record per page, then merge adjacent equal
    flags inside an allocation; data = concat of PRESENT pages."""
    flag = {0: 4, 1: 8, 2: 1}
    recs, data, digests = [], [], []
    g = 0
    for (aid, va, nb), c in zip(registry, contents):
        per = []
        for (off, ln) in _pages(nb, P):
            cls = classes_of_page[g]
            per.append([va + off, 1, flag[cls]])
            digests.append(hwcrc(c[off:off + ln]))
            if cls == 0:
                data.append(c[off:off + ln].tobytes())
            g += 1
        merged = []
        for r in per:
            if merged and merged[-1][2] == r[2]:
                merged[-1][1] += 1
            else:
                merged.append(r)
        recs += [tuple(m) for m in merged]
    return recs, b"".join(data), digests


def test_header_and_sections_full(orc, hwcrc):
    rng = np.random.default_rng(1)
    sizes = [3 * P4K, 2 * P4K + 1024, 4096]
    reg = [(7 + i, 0x7F0000000000 + i * 0x100000, s) for i, s in enumerate(sizes)]
    cont = [_rand(rng, s) for s in sizes]
    cont[0][P4K:2 * P4K] = 0          # one ZERO page in the middle
    st, s = orc.checkpoint(P4K, reg, cont, generation=5)
    assert st == orc.OK
    p = orc.parse(s)
    h = p["header"]
    assert h["magic"] == b"GCRIMG\x00\x01" and h["version"] == 1 and h["page_size"] == P4K
    assert h["generation"] == 5 and h["parent_generation"] == 0 and h["flags"] == 0
    assert h["n_pages"] == 3 + 3 + 1 and h["n_zero"] == 1 and h["n_parent"] == 0 and h["n_present"] == 6
    assert h["image_bytes"] == sum(sizes) - P4K
    assert p["allocs"] == [(va, nb, aid) for (aid, va, nb) in reg]
    # meta crc recomputed with the independent hardware CRC
    meta_len = 96 + 24 * 3 + 16 * h["n_entries"] + 4 * h["n_pages"]
    hdr = bytearray(s[:96]); hdr[88:92] = b"\0\0\0\0"
    assert hwcrc(bytes(hdr) + s[96:meta_len]) == h["meta_crc32c"]
    assert len(s) == meta_len + h["image_bytes"]


@pytest.mark.parametrize("sizes", [[1], [2], [3], [6], [1, 1], [2, 3], [1, 2, 3], [3, 1, 2]])
def test_pagemap_and_pack_brute_force(orc, hwcrc, sizes):
    """Every class pattern over tiny registries (pages of 4 KiB; the last page
    of each allocation short when possible) vs the naive formulation."""
    rng = np.random.default_rng(sum(sizes) * 31 + len(sizes))
    n = sum(sizes)
    nbytes = [k * P4K - (1024 if k > 1 else 0) for k in sizes]
    reg = [(i, 0x10000000 + i * 0x200000, nb) for i, nb in enumerate(nbytes)]
    base = [_rand(rng, nb) for nb in nbytes]
    # ensure every non-zero page is non-zero
    for c in base:
        c[::512] |= 1
    pats = list(itertools.product([0, 1, 2], repeat=n))
    if len(pats) > 243:
        pats = [pats[i] for i in rng.choice(len(pats), 243, replace=False)]
    for pat in pats:
        cont = [c.copy() for c in base]
        g = 0
        dprev = []
        for a, nb in enumerate(nbytes):
            for (off, ln) in _pages(nb, P4K):
                if pat[g] == 1:
                    cont[a][off:off + ln] = 0
                dig = hwcrc(cont[a][off:off + ln])
                # PARENT: previous digest equals the page's digest; else differs
                dprev.append(dig if pat[g] == 2 else dig ^ 0x5A5A5A5A)
                g += 1
        st, s = orc.checkpoint(P4K, reg, cont, mode=orc.INCREMENTAL, d_prev=np.array(dprev, np.uint32),
                               generation=9, parent_generation=8)
        assert st == orc.OK
        p = orc.parse(s)
        recs, data, digests = _naive_expect(reg, cont, P4K, pat, hwcrc)
        assert p["entries"] == recs, pat
        assert p["data"] == data
        assert list(p["digests"]) == digests
        h = p["header"]
        assert sum(e[1] for e in p["entries"]) == n
        assert (h["n_present"], h["n_zero"], h["n_parent"]) == (pat.count(0), pat.count(1), pat.count(2))
        assert h["flags"] == 1 and h["parent_generation"] == 8


def test_c1_constructed_counts(orc, hwcrc):
    """C1: one 64 MiB region registered as 4 contiguous 16 MiB
    allocations, 64 KiB pages, exactly 256 zero pages -> n_present 768,
    image_bytes 50,331,648, every ZERO digest 0x72C0C4A4, runs break at the
    allocation borders although the VAs are contiguous."""
    P = 65536
    rng = np.random.default_rng(0xC0FFEE)
    region = rng.integers(0, 256, 64 << 20, dtype=np.uint8)
    region[::4096] |= 1
    zero = rng.choice(1024, 256, replace=False)
    for z in zero:
        region[z * P:(z + 1) * P] = 0
    base = 0x7F1200000000
    reg = [(a, base + a * (16 << 20), 16 << 20) for a in range(4)]
    cont = [region[a * (16 << 20):(a + 1) * (16 << 20)] for a in range(4)]
    st, s = orc.checkpoint(P, reg, cont)
    assert st == orc.OK
    p = orc.parse(s)
    h = p["header"]
    assert h["n_pages"] == 1024 and h["n_zero"] == 256 and h["n_present"] == 768
    assert h["image_bytes"] == 50_331_648
    dg = p["digests"]
    assert all(dg[z] == 0x72C0C4A4 for z in zero)
    # runs never cross allocation borders
    for (va, nr, fl) in p["entries"]:
        a = (va - base) // (16 << 20)
        assert va + nr * P <= base + (a + 1) * (16 << 20)
    # border pages start entries even if the class continues
    starts = {va for (va, nr, fl) in p["entries"]}
    for a in range(4):
        assert base + a * (16 << 20) in starts
    # spot-check digests against the hardware CRC
    for g in rng.choice(1024, 40, replace=False):
        assert dg[g] == hwcrc(region[g * P:(g + 1) * P])


def test_image_data_folds_to_present_digests(orc):
    """CRC32C(whole image data) == fold of PRESENT digests with combine (c.4)."""
    rng = np.random.default_rng(3)
    P = 8192
    sizes = [5 * P + 4096, 3 * P, 7 * P + 16]
    reg = [(i, 0x1000000 * (i + 1), s) for i, s in enumerate(sizes)]
    cont = [_rand(rng, s) for s in sizes]
    cont[1][P:2 * P] = 0
    st, s = orc.checkpoint(P, reg, cont)
    p = orc.parse(s)
    # walk entries in order, folding PRESENT page digests with their lengths
    g = 0
    a_pages = [(nb, _pages(nb, P)) for nb in sizes]
    flat = [ln for nb, pg in a_pages for (_, ln) in pg]
    acc = None
    for (va, nr, fl) in p["entries"]:
        for k in range(nr):
            if fl == orc.PE_PRESENT:
                d = int(p["digests"][g])
                acc = d if acc is None else gf2.combine(acc, d, flat[g])
            g += 1
    assert acc == orc.crc32c(np.frombuffer(p["data"], np.uint8))


def _mk_state(rng, sizes, zero_frac=0.25, P=P4K):
    cont = [_rand(rng, s) for s in sizes]
    for c in cont:
        c[::256] |= 1
        for (off, ln) in _pages(c.size, P):
            if rng.random() < zero_frac:
                c[off:off + ln] = 0
    return cont


def test_round_trip_into_poison(orc):
    rng = np.random.default_rng(5)
    sizes = [9 * P4K + 2048, P4K, 33 * P4K]
    reg = [(i, 0x2000000 * (i + 1), s) for i, s in enumerate(sizes)]
    cont = _mk_state(rng, sizes)
    st, s = orc.checkpoint(P4K, reg, cont)
    tgt = [np.full(sz, 0xA5, np.uint8) for sz in sizes]
    st, vf, fb = orc.restore([s], P4K, sizes, tgt)
    assert (st, vf) == (orc.OK, 0)
    for a, b in zip(cont, tgt):
        assert np.array_equal(a, b)


def test_chain_restore_and_counts(orc):
    """restore(I0, I1, I2) == state at I2; exact dirty counts from mutations
    that XOR one non-zero 32-bit word (guaranteed dirty)."""
    rng = np.random.default_rng(6)
    P = P4K
    sizes = [40 * P, 17 * P + 512]
    reg = [(i, 0x40000000 * (i + 1), s) for i, s in enumerate(sizes)]
    cont = _mk_state(rng, sizes, zero_frac=0.0)
    n = sum((s + P - 1) // P for s in sizes)
    st, s0 = orc.checkpoint(P, reg, cont, generation=1)
    d0 = orc.parse(s0)["digests"].copy()
    states = [[c.copy() for c in cont]]
    streams = [s0]
    dprev, gen = d0, 1
    for step, j in enumerate([5, 11]):
        flat_pages = [(a, off, ln) for a, nb in enumerate(sizes) for (off, ln) in _pages(nb, P)]
        pick = rng.choice(n, j, replace=False)
        for g in pick:
            a, off, ln = flat_pages[g]
            w = int(rng.integers(0, ln // 4))
            x = np.uint32(int(rng.integers(1, 1 << 32)))
            v = cont[a][off + 4 * w: off + 4 * w + 4].view(np.uint32)
            v ^= x
        st, si = orc.checkpoint(P, reg, cont, mode=orc.INCREMENTAL, d_prev=dprev, generation=gen + 1,
                                parent_generation=gen)
        assert st == orc.OK
        h = orc.parse(si)["header"]
        assert (h["n_present"], h["n_parent"], h["n_zero"]) == (j, n - j, 0)
        dprev = orc.parse(si)["digests"].copy()
        gen += 1
        streams.append(si)
        states.append([c.copy() for c in cont])
    for k in range(1, 4):
        tgt = [np.full(sz, 0xA5, np.uint8) for sz in sizes]
        st, vf, fb = orc.restore(streams[:k], P, sizes, tgt)
        assert (st, vf) == (orc.OK, 0)
        for a, b in zip(states[k - 1], tgt):
            assert np.array_equal(a, b)


def test_zero_wins_over_parent_and_negative_zero_is_not_zero(orc):
    P = P4K
    reg = [(0, 0x10000, 2 * P)]
    c = np.zeros(2 * P, np.uint8)
    c[P:].view(np.float32)[:] = -0.0          # 0x80000000 words: not zero (R-4)
    z = orc.crc32c(np.zeros(P, np.uint8))
    dn = orc.crc32c(c[P:])
    st, s = orc.checkpoint(P, reg, [c], mode=orc.INCREMENTAL, d_prev=np.array([z, dn ^ 1], np.uint32),
                           generation=2, parent_generation=1)
    p = orc.parse(s)
    assert p["entries"] == [(0x10000, 1, orc.PE_ZERO), (0x10000 + P, 1, orc.PE_PRESENT)]


def test_corruption_and_validation_errors(orc):
    rng = np.random.default_rng(8)
    P = P4K
    sizes = [6 * P, 3 * P + 2048]
    reg = [(i, 0x3000000 * (i + 1), s) for i, s in enumerate(sizes)]
    cont = _mk_state(rng, sizes, zero_frac=0.3)
    st, s = orc.checkpoint(P, reg, cont)
    h = orc.parse(s)["header"]
    meta = 96 + 24 * 2 + 16 * h["n_entries"] + 4 * h["n_pages"]
    # every metadata byte flip -> CORRUPT
    for off in list(range(0, meta)):
        b = bytearray(s)
        b[off] ^= 0x40
        st2, _, _ = orc.restore([bytes(b)], P, sizes, [np.zeros(x, np.uint8) for x in sizes])
        assert st2 == orc.E_CORRUPT, off
    # a data byte flip -> exactly one verify failure at that page
    data_off = meta
    b = bytearray(s)
    b[data_off + 5] ^= 1
    tgt = [np.zeros(x, np.uint8) for x in sizes]
    st2, vf, fb = orc.restore([bytes(b)], P, sizes, tgt)
    first_present = 0
    g = 0
    for (va, nr, fl) in orc.parse(s)["entries"]:
        if fl == orc.PE_PRESENT:
            first_present = g
            break
        g += nr
    assert (st2, vf, fb) == (orc.E_VERIFY, 1, first_present)
    # truncated stream -> CORRUPT
    assert orc.restore([s[:-1]], P, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.E_CORRUPT
    # layout mismatches
    assert orc.restore([s], P * 2, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.E_LAYOUT
    assert orc.restore([s], P, [sizes[0], sizes[1] + 16], [np.zeros(sizes[0], np.uint8), np.zeros(sizes[1] + 16, np.uint8)])[0] == orc.E_LAYOUT
    assert orc.restore([s], P, sizes[:1], [np.zeros(sizes[0], np.uint8)])[0] == orc.E_LAYOUT
    # chain: an incremental first -> CHAIN; a broken parent link -> CHAIN
    d0 = orc.parse(s)["digests"].copy()
    st, si = orc.checkpoint(P, reg, cont, mode=orc.INCREMENTAL, d_prev=d0, generation=2, parent_generation=1)
    assert orc.restore([si], P, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.E_CHAIN
    st, sbad = orc.checkpoint(P, reg, cont, mode=orc.INCREMENTAL, d_prev=d0, generation=3, parent_generation=7)
    assert orc.restore([s, sbad], P, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.E_CHAIN
    assert orc.restore([s, si], P, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.OK
    # unknown version with a valid meta CRC -> VERSION
    b = bytearray(s)
    b[8:12] = (2).to_bytes(4, "little")
    b[88:92] = b"\0\0\0\0"
    crc = orc.crc32c(bytes(b[:meta]))
    b[88:92] = crc.to_bytes(4, "little")
    assert orc.restore([bytes(b)], P, sizes, [np.zeros(x, np.uint8) for x in sizes])[0] == orc.E_VERSION


def test_incremental_requires_parent(orc):
    reg = [(0, 0x10000, P4K)]
    st, s = orc.checkpoint(P4K, reg, [np.ones(P4K, np.uint8)], mode=orc.INCREMENTAL, d_prev=None)
    assert st == orc.E_CHAIN


def test_invalid_registry(orc):
    one = [np.ones(P4K, np.uint8)]
    assert orc.checkpoint(P4K, [(0, 0x10008, P4K)], one)[0] == orc.E_INVAL      # misaligned vaddr
    assert orc.checkpoint(P4K, [(0, 0x10000, P4K - 8)], [np.ones(P4K - 8, np.uint8)])[0] == orc.E_INVAL
    assert orc.checkpoint(3000, [(0, 0x10000, P4K)], one)[0] == orc.E_INVAL     # not a power of two
    assert orc.checkpoint(2048, [(0, 0x10000, P4K)], one)[0] == orc.E_INVAL     # below 4 KiB


def test_cross_page_size_identity(orc):
    """With no tail pages: D_2P[k] = adv_P(D_P[2k]) ^ D_P[2k+1]; a page is ZERO
    at 2P iff both halves are ZERO at P (c.4)."""
    rng = np.random.default_rng(10)
    P = P4K
    sizes = [16 * P, 8 * P]
    reg = [(i, 0x5000000 * (i + 1), s) for i, s in enumerate(sizes)]
    cont = _mk_state(rng, sizes, zero_frac=0.4)
    _, s1 = orc.checkpoint(P, reg, cont)
    _, s2 = orc.checkpoint(2 * P, reg, cont)
    d1, d2 = orc.parse(s1)["digests"], orc.parse(s2)["digests"]
    for k in range(len(d2)):
        assert d2[k] == gf2.combine(int(d1[2 * k]), int(d1[2 * k + 1]), P)
    z1 = gf2.zero_digest(P)
    z2 = gf2.zero_digest(2 * P)
    for k in range(len(d2)):
        assert (d2[k] == z2) == (d1[2 * k] == z1 and d1[2 * k + 1] == z1)
