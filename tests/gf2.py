"""GF(2) helpers for tests: the CRC32C register advance adv_n as a 32x32
bit-matrix power (zlib crc32_combine style).  Written independently of
oracle/ (which uses a Sarwate byte table) and of the product; used only to
state closed forms and invariants."""

POLY = 0x82F63B78  # reflected Castagnoli polynomial (R-10)


def _mat_times(mat, vec):
    s = 0
    i = 0
    while vec:
        if vec & 1:
            s ^= mat[i]
        vec >>= 1
        i += 1
    return s


def _mat_square(mat):
    return [_mat_times(mat, mat[n]) for n in range(32)]


def _one_zero_bit():
    # operator for one zero bit in the reflected register
    return [POLY] + [1 << (n - 1) for n in range(1, 32)]


def adv(nbytes: int, state: int) -> int:
    """Register after feeding nbytes zero bytes from `state` (s (x) x^(8n) mod P)."""
    if nbytes == 0:
        return state
    odd = _one_zero_bit()
    even = _mat_square(odd)      # 2 zero bits
    odd = _mat_square(even)      # 4 zero bits
    n = nbytes
    while True:
        even = _mat_square(odd)  # 8, 32, ... bits: first iteration = 1 byte
        if n & 1:
            state = _mat_times(even, state)
        n >>= 1
        if n == 0:
            break
        odd = _mat_square(even)
        if n & 1:
            state = _mat_times(odd, state)
        n >>= 1
        if n == 0:
            break
    return state


def zero_digest(n: int) -> int:
    """Z(n) = CRC32C of n zero bytes = adv_n(0xFFFFFFFF) ^ 0xFFFFFFFF (c.4)."""
    return adv(n, 0xFFFFFFFF) ^ 0xFFFFFFFF


def combine(crc_a: int, crc_b: int, len_b: int) -> int:
    """crc(A||B) = adv_{|B|}(crc(A)) ^ crc(B) (c.4 linearity)."""
    return adv(len_b, crc_a) ^ crc_b
