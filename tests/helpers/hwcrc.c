/* Independent CRC32C for tests: the x86 SSE4.2 `crc32` instruction computes
 * CRC32C (Castagnoli) in hardware (Intel SDM Vol. 2A, "CRC32 -- Accumulate
 * CRC32 Value": polynomial 11EDC6F41H).  Shares nothing with oracle/ or the
 * product; used only to pin the oracle (tests/test_oracle_crc.py). */
#include <stdint.h>
#include <nmmintrin.h>
uint32_t hw_crc32c_update(uint32_t state, const uint8_t *p, uint64_t n) {
    uint64_t s = state;
    while (n >= 8) { uint64_t w; __builtin_memcpy(&w, p, 8); s = _mm_crc32_u64(s, w); p += 8; n -= 8; }
    uint32_t s32 = (uint32_t)s;
    while (n--) s32 = _mm_crc32_u8(s32, *p++);
    return s32;
}
uint32_t hw_crc32c(const uint8_t *p, uint64_t n) { return hw_crc32c_update(0xFFFFFFFFu, p, n) ^ 0xFFFFFFFFu; }
