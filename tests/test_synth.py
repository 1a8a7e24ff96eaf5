"""CPU pins of the seeded input generator's CPU twin (synth.py): every kind
against a scalar, one-word-at-a-time restatement of the formulas written in
include/gcr_synth.h.  The GPU fill is compared with the CPU twin on the GPU
(test_gpu_parity.py::test_gpu_generator_matches_cpu_twin)."""
import numpy as np
import pytest

from paper_2502_16631_b200 import synth

M64 = (1 << 64) - 1


def sm64(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def word(seed, key, i, kind, const_bits=0):
    if kind == synth.ZERO:
        return 0
    if kind == synth.F32_CONST:
        return const_bits | (const_bits << 32)
    r = sm64(seed ^ (key << 40) ^ i)
    if kind == synth.RANDOM:
        return r
    if kind in (synth.F32_WEIGHT, synth.F32_M, synth.F32_V):
        e0, sg = {synth.F32_WEIGHT: (118, 1), synth.F32_M: (113, 1), synth.F32_V: (103, 0)}[kind]
        out = 0
        for half in range(2):
            b = (r >> (32 * half)) & 0xFFFFFFFF
            v = ((e0 + ((b >> 23) & 3)) << 23) | (b & 0x7FFFFF) | ((b & 0x80000000) if sg else 0)
            out |= v << (32 * half)
        return out
    if kind == synth.BF16_WEIGHT:
        out = 0
        for q in range(4):
            h = (r >> (16 * q)) & 0xFFFF
            v = (h & 0x8000) | ((118 + ((h >> 7) & 3)) << 7) | (h & 0x7F)
            out |= v << (16 * q)
        return out
    raise ValueError(kind)


@pytest.mark.parametrize("kind", [synth.RANDOM, synth.F32_WEIGHT, synth.F32_CONST, synth.ZERO, synth.F32_M,
                                  synth.F32_V, synth.BF16_WEIGHT])
def test_cpu_twin_matches_scalar_formula(kind):
    seed, key = synth.seed_for(3, 1), 7
    start, n = 123_456_789, 257
    got = synth.gen_words(seed, key, start, n, kind, synth.ONE_F32)
    exp = np.array([word(seed, key, start + i, kind, synth.ONE_F32) for i in range(n)], dtype=np.uint64)
    assert np.array_equal(got, exp)


def test_splitmix64_known_value():
    # splitmix64 of 0: the first output of the reference generator seeded with 0
    assert int(synth.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    assert sm64(0) == 0xE220A8397B1DCDAF


def test_cpu_bytes_overlays():
    w = synth.make_workload("C5", gib=1, page_size=65536)
    za, zo, zn = next(z for z in w.zero_ranges if z[1] >= 64 and z[1] + z[2] + 64 <= (1 << 30)
                      and not any(y[0] == z[0] and y[1] in (z[1] - z[2], z[1] + z[2]) for y in w.zero_ranges))
    b = w.cpu_bytes(za, zo - 64, zn + 128)
    assert not b[64:64 + zn].any() and b[:64].any() and b[64 + zn:].any()
    w.mutations = [(0, 4096, 0xDEADBEEF)]
    x = w.cpu_bytes(0, 0, 8192)
    w.mutations = []
    y = w.cpu_bytes(0, 0, 8192)
    assert int((x[4096:4100].view(np.uint32) ^ y[4096:4100].view(np.uint32))[0]) == 0xDEADBEEF
    assert np.array_equal(x[:4096], y[:4096]) and np.array_equal(x[4100:], y[4100:])
