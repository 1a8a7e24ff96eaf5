// crc_host.cpp -- host-side CRC32C math for libgcr (product code; shares
// nothing with oracle/).
//
// CRC32C parameters (reading R-10): reflected Castagnoli polynomial
// 0x82F63B78, init and xorout 0xFFFFFFFF.  Everything the kernels need is a
// GF(2)-linear map "advance the register by d zero bytes", adv_d(v) =
// v * x^(8d) mod P, represented as a 32x32 bit matrix (one column per input
// bit) and raised to the d-th power by repeated squaring; byte tables are
// then read off by linearity: tab[k][e] = adv_d(e << 8k).
#include <algorithm>
#include <cstring>
#include <nmmintrin.h>

#include "gcr_internal.h"

namespace gcr {
namespace {

constexpr uint32_t kPoly = 0x82F63B78u;

struct Mat {
    uint32_t col[32];  // col[i] = image of bit i
};

uint32_t mat_vec(const Mat &m, uint32_t v) {
    uint32_t r = 0;
    for (int i = 0; v; i++, v >>= 1)
        if (v & 1u) r ^= m.col[i];
    return r;
}

Mat mat_mul(const Mat &a, const Mat &b) {  // a * b (apply b first)
    Mat r;
    for (int i = 0; i < 32; i++) r.col[i] = mat_vec(a, b.col[i]);
    return r;
}

Mat identity() {
    Mat m;
    for (int i = 0; i < 32; i++) m.col[i] = 1u << i;
    return m;
}

// one zero BIT through the reflected register: v -> (v >> 1) ^ (v & 1 ? P : 0)
Mat zero_bit() {
    Mat m;
    m.col[0] = kPoly;
    for (int i = 1; i < 32; i++) m.col[i] = 1u << (i - 1);
    return m;
}

Mat zero_byte() {
    Mat b = zero_bit();
    Mat m = mat_mul(b, b);   // 2 bits
    m = mat_mul(m, m);       // 4
    return mat_mul(m, m);    // 8
}

Mat adv_matrix(uint64_t nbytes) {
    Mat r = identity(), p = zero_byte();
    while (nbytes) {
        if (nbytes & 1) r = mat_mul(p, r);
        p = mat_mul(p, p);
        nbytes >>= 1;
    }
    return r;
}

void fill_table(uint32_t tab[4][256], uint64_t d) {
    Mat m = adv_matrix(d);
    for (int k = 0; k < 4; k++)
        for (uint32_t e = 0; e < 256; e++) tab[k][e] = mat_vec(m, e << (8 * k));
}

uint32_t apply4(const uint32_t tab[4][256], uint32_t v) {
    return tab[0][v & 255] ^ tab[1][(v >> 8) & 255] ^ tab[2][(v >> 16) & 255] ^ tab[3][v >> 24];
}

}  // namespace

void build_tables(CrcTables *t) {
    fill_table(t->braid, kRowBytes);
    fill_table(t->t4, 4);
    fill_table(t->a16, 16);
    fill_table(t->a32, 32);
    fill_table(t->a64, 64);
    fill_table(t->a128, 128);
    fill_table(t->a256, 256);
    // fold_m[d] = adv_{512 d}(x^0): x^0 is bit 31 of the reflected register
    uint32_t row[4][256];
    fill_table(row, kRowBytes);
    t->fold_m[0] = 0x80000000u;
    for (int d = 1; d < 4096; d++) t->fold_m[d] = apply4(row, t->fold_m[d - 1]);
}

void table_basis(const uint32_t (&tab)[4][256], uint32_t *basis32) {
    for (int k = 0; k < 4; k++)
        for (int i = 0; i < 8; i++) basis32[8 * k + i] = tab[k][1u << i];
}

// The reflected GF(2) product K1 evaluates lane-parallel (lane k: v * x^k).
static uint32_t mulmod(uint32_t m, uint32_t v) {
    uint32_t r = 0;
    for (int k = 0; k < 32; k++) {
        if ((m >> (31 - k)) & 1u) r ^= v;
        v = (v >> 1) ^ ((v & 1u) ? kPoly : 0u);
    }
    return r;
}

uint32_t crc_shift(uint32_t reg, uint64_t nbytes) { return mat_vec(adv_matrix(nbytes), reg); }

uint32_t zero_digest(uint64_t n) { return mat_vec(adv_matrix(n), 0xFFFFFFFFu) ^ 0xFFFFFFFFu; }

// Raw register update over host bytes for image metadata (meta_crc32c).  The
// x86 SSE4.2 crc32 instruction implements exactly this register update for
// the Castagnoli polynomial; a table path covers CPUs without it.
constexpr uint64_t kCrcSplitMin = 64 * 1024;  // below this one chain is as fast as the join

uint32_t host_crc32c_update(uint32_t state, const void *p, uint64_t n) {
    const uint8_t *b = static_cast<const uint8_t *>(p);
    static const bool have_sse42 = __builtin_cpu_supports("sse4.2");
    if (have_sse42 && n >= kCrcSplitMin) {
        // three independent crc32 chains (the instruction has 3-cycle latency
        // and 1-cycle throughput), joined by linearity:
        // reg(s, A|B|C) = adv_k(adv_k(reg(s, A)) ^ reg(0, B)) ^ reg(0, C)
        const uint64_t k = (n / 3) & ~7ull;
        const uint8_t *b1 = b + k, *b2 = b + 2 * k;
        uint64_t s0 = state, s1 = 0, s2 = 0;
        for (uint64_t i = 0; i < k; i += 8) {
            uint64_t w0, w1, w2;
            std::memcpy(&w0, b + i, 8);
            std::memcpy(&w1, b1 + i, 8);
            std::memcpy(&w2, b2 + i, 8);
            s0 = _mm_crc32_u64(s0, w0);
            s1 = _mm_crc32_u64(s1, w1);
            s2 = _mm_crc32_u64(s2, w2);
        }
        // (the shift matrix is cached: a drain CRCs equal-sized digest batches)
        thread_local uint64_t mk = 0;
        thread_local Mat m;
        if (mk != k) {
            m = adv_matrix(k);
            mk = k;
        }
        const uint32_t joined = mat_vec(m, mat_vec(m, (uint32_t)s0) ^ (uint32_t)s1) ^ (uint32_t)s2;
        return host_crc32c_update(joined, b + 3 * k, n - 3 * k);
    }
    if (have_sse42) {
        uint64_t s = state;
        while (n >= 8) {
            uint64_t w;
            std::memcpy(&w, b, 8);
            s = _mm_crc32_u64(s, w);
            b += 8;
            n -= 8;
        }
        uint32_t s32 = static_cast<uint32_t>(s);
        while (n--) s32 = _mm_crc32_u8(s32, *b++);
        return s32;
    }
    static uint32_t t1[256];
    static bool init = false;
    if (!init) {
        Mat m = zero_byte();
        for (uint32_t e = 0; e < 256; e++) t1[e] = mat_vec(m, e);
        init = true;
    }
    while (n--) state = (state >> 8) ^ t1[(state ^ *b++) & 255u];
    return state;
}

bool crc_self_test() {
    // "123456789" -> 0xE3069283 through the word-step tables (slicing-by-4
    // form the kernels use) and through host_crc32c_update.
    CrcTables *t = new CrcTables;
    build_tables(t);
    const char *s = "123456789";
    uint32_t st = 0xFFFFFFFFu;
    int i = 0;
    for (; i + 4 <= 9; i += 4) {
        uint32_t w;
        std::memcpy(&w, s + i, 4);
        st = apply4(t->t4, st ^ w);
    }
    uint32_t a = host_crc32c_update(st, s + i, 9 - i) ^ 0xFFFFFFFFu;
    uint32_t b = host_crc32c_update(0xFFFFFFFFu, s, 9) ^ 0xFFFFFFFFu;
    // braid table consistency: adv_512 == (adv_4)^128 on a probe value
    uint32_t v = 0x12345678u, w = v;
    for (int k = 0; k < 128; k++) w = apply4(t->t4, w);
    // the 3-chain split path against the one-chain path on a long buffer
    {
        const uint64_t n = 3 * kCrcSplitMin + 40;
        uint8_t *buf = new uint8_t[n];
        for (uint64_t j = 0; j < n; j++) buf[j] = (uint8_t)(j * 2654435761u >> 13);
        uint32_t one = 0xFFFFFFFFu;
        for (uint64_t j = 0; j < n; j += 4096) one = host_crc32c_update(one, buf + j, std::min<uint64_t>(4096, n - j));
        const bool split_ok = host_crc32c_update(0xFFFFFFFFu, buf, n) == one;
        delete[] buf;
        if (!split_ok) {
            delete t;
            return false;
        }
    }
    // fold products: fold_m[d] (*) v == adv_{512 d}(v) by an independent matrix power
    bool ok = a == 0xE3069283u && b == 0xE3069283u && apply4(t->braid, v) == w &&
              zero_digest(65536) == 0x72C0C4A4u && mulmod(t->fold_m[1], v) == w;
    for (uint32_t d : {0u, 2u, 3u, 127u, 128u, 1000u, 4095u}) ok = ok && mulmod(t->fold_m[d], v) == mat_vec(adv_matrix(512ull * d), v);
    delete t;
    return ok;
}

}  // namespace gcr
