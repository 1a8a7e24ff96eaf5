"""Pins for the oracle's CRC32C (SURVEY.md §8(c) c.4 rows 'CRC32C',
'CRC32C, independent', 'Zero-page digest', 'Linearity').  Reading R-10."""
import os

import numpy as np
import pytest

import gf2

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "crc32c_vectors.txt")


def _decode(spec: str) -> bytes:
    kind, _, arg = spec.partition(":")
    if kind == "ascii":
        return arg.encode()
    n = int(arg)
    if kind == "zeros":
        return bytes(n)
    if kind == "ones":
        return b"\xff" * n
    if kind == "incr":
        return bytes(range(n))
    if kind == "decr":
        return bytes(range(n - 1, -1, -1))
    raise ValueError(spec)


def _vectors():
    out = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) == 2:          # empty ascii payload
            name, exp = parts
            spec = "ascii:"
        else:
            name, spec, exp = parts
        out.append((name, _decode(spec), int(exp, 16)))
    return out


@pytest.mark.parametrize("name,data,expected", _vectors(), ids=[v[0] for v in _vectors()])
def test_published_vectors(orc, name, data, expected):
    assert orc.crc32c(data) == expected


@pytest.mark.parametrize("name,data,expected", _vectors(), ids=[v[0] for v in _vectors()])
def test_hw_helper_matches_published_vectors(hwcrc, name, data, expected):
    # the independent implementation is itself pinned to the same vectors
    assert hwcrc(data) == expected


def test_oracle_vs_sse42_random(orc, hwcrc):
    rng = np.random.default_rng(20250216)
    for i in range(3000):
        n = int(rng.integers(0, 9000)) if i % 10 else int(rng.integers(0, 70000))
        buf = rng.integers(0, 256, n, dtype=np.uint8)
        assert orc.crc32c(buf) == hwcrc(buf), n


@pytest.mark.parametrize("log2p", range(12, 22))
def test_zero_page_digest_closed_form(orc, hwcrc, log2p):
    P = 1 << log2p
    z = np.zeros(P, dtype=np.uint8)
    d, cls = orc.page_record(z)
    assert d == gf2.zero_digest(P) == hwcrc(z)
    assert cls == orc.CLASS_ZERO


def test_zero_digest_64k_matches_survey_constant(orc):
    # SURVEY.md §8(d) C1 states every ZERO digest at 64 KiB is 0x72C0C4A4
    assert orc.crc32c(np.zeros(65536, np.uint8)) == 0x72C0C4A4 == gf2.zero_digest(65536)


def test_linearity_combine(orc):
    rng = np.random.default_rng(7)
    for _ in range(200):
        a = rng.integers(0, 256, int(rng.integers(0, 3000)), dtype=np.uint8)
        b = rng.integers(0, 256, int(rng.integers(0, 3000)), dtype=np.uint8)
        ab = np.concatenate([a, b])
        assert orc.crc32c(ab) == gf2.combine(orc.crc32c(a), orc.crc32c(b), b.size)


def test_single_bit_and_burst_changes_flip_digest(orc):
    # H8 / R-6: any error burst of <= 32 bits changes a CRC-32
    rng = np.random.default_rng(11)
    page = rng.integers(0, 256, 4096, dtype=np.uint8)
    d0 = orc.crc32c(page)
    for _ in range(500):
        p = page.copy()
        bit = int(rng.integers(0, 4096 * 8 - 32))
        burst = int(rng.integers(1, 1 << 32)) | 1  # non-zero burst starting at `bit`
        for j in range(32):
            if (burst >> j) & 1:
                q = bit + j
                p[q // 8] ^= np.uint8(1 << (q % 8))
        assert orc.crc32c(p) != d0
