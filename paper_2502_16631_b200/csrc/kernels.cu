// kernels.cu -- sm_100a kernels of the device-memory snapshot path
// (SURVEY.md §8(a) rows A1-A9).
//
//  K0  build_page_table  A1: page -> allocation, tile -> allocation maps
//  K1  scan              A2+A3+A4 (+A9 in verify mode): per-page CRC32C,
//                        all-zero test, dirty diff, class, tile counters
//  K1g scan_grp<G>       the same for 4 / 8 KiB pages: G pages per 16 KiB group
//  K2  tile_scan         A5: chunk-local exclusive scan of PRESENT bytes per
//                        tile (the pack's destination offsets) and chunk totals
//  K3  pagemap_*         A5: maximal runs -> CRIU-style pagemap entries
//  K4  pack              A6: stream-compaction of PRESENT pages into staging
//                        (16-B vector copy; k_pack_tma: the TMA ring, GCR_TMA_COPY=2)
//  K6  scatter_tma       A8: staged image pieces -> allocation pages through a
//                        TMA bulk-copy ring (k_scatter: vector copy, GCR_TMA_COPY=0)
//  K7  zero_fill         A8: ZERO runs (TMA bulk stores)
//
// CRC32C arithmetic.  raw(x) is the register after x from 0
// (GF(2)-linear); crc(x) = raw(x) ^ Z(|x|).  A warp streams 512-byte rows;
// lane l owns words 4l..4l+3 of every row ("braids", the zlib braided-CRC
// idea).  Braid register x_b evolves as x_b <- adv_512(x_b) ^ w_b per row;
// after the last row of a page the 512-byte block Y = (x_0..x_127) satisfies
// raw(page) = raw(Y).  Each lane folds its 16 bytes of Y (raw16) and a 5-level
// shuffle tree combines the lanes (distances 16..256 B).  A short (tail) page
// is processed as if front-padded with zeros to the full page -- leading
// zeros leave raw() unchanged -- so every page uses the same geometry.
//
// adv_512 is evaluated with four 256-entry tables held LANE-PRIVATE in shared
// memory (entry e of table k for lane l at byte (k>>1)*64K + e*256 +
// (k&1)*128 + l*4, so the bank always equals the lane: conflict-free).  The
// byte index is extracted and scaled in ONE prmt: prmt(x, l*4, 0x55k4) =
// (byte_k(x) << 8) | l*4.  Per 4 data bytes: 4 PRMT + 4 LDS + 4 IMAD.IADD
// (FMA pipe) + 2 LOP3.
//
// Work split: the chunk's REAL rows (the virtual padding of short pages is not
// counted) are divided into equal contiguous ranges, one per warp, so every
// warp streams the same bytes whatever the page or chunk size (no wave
// quantization) and every page event is warp-uniform (no divergence).  A warp
// streams its range continuously across page and allocation boundaries with
// the next block of rows always in flight: a LOAD cursor walks contiguous
// address runs, a PROCESS cursor finalizes pages.  A page cut by range
// boundaries is folded in K1 itself: each piece is advanced to the page end
// (one GF(2) product with fold_m[d], lane-parallel) and XORed into the page's
// owner slot; the piece that completes the page's rows finalizes it.
#include <cstdio>
#include <cstdlib>

#include "gcr_internal.h"

namespace gcr {

namespace {

constexpr uint32_t kBraidSmem = 4u * 256u * 32u * 4u;  // 128 KiB
constexpr uint32_t kSmallTables = 6;                   // t4 a16 a32 a64 a128 a256
constexpr uint32_t kNibWords = 7u * 4u * 2u * 16u;  // nibble tables of the 7 tables (staging scratch)
constexpr uint32_t kScanSmem = kBraidSmem + kSmallTables * 4096u + kNibWords * 4u;
// K1g option (ScanParams::t4rep): the raw16 table t4 replicated 8x, entry e of
// sub-table k for lane-group c = lane & 7 at word (256k + e) * 8 + c: bank =
// (8e + c) mod 32, so only the 4 lanes sharing c can collide (the unreplicated
// table puts 32 random lookups on 32 banks: ~3.5-way conflicts).
constexpr uint32_t kT4RepBytes = 8u * 1024u * 4u;

__device__ __forceinline__ uint32_t apply_t4rep(const uint32_t *t, uint32_t v, uint32_t c) {
    return t[((v & 255u) << 3) + c] ^ t[((256u + ((v >> 8) & 255u)) << 3) + c] ^
           t[((512u + ((v >> 16) & 255u)) << 3) + c] ^ t[((768u + (v >> 24)) << 3) + c];
}
constexpr uint32_t kLog2Row = 9;
#ifndef GCR_SCAN_THREADS
#define GCR_SCAN_THREADS 640
#endif
constexpr int kScanThreads = GCR_SCAN_THREADS;
#ifndef GCR_SCAN_UNROLL
#define GCR_SCAN_UNROLL 5
#endif
constexpr int kScanUnroll = GCR_SCAN_UNROLL;
constexpr unsigned kFull = 0xFFFFFFFFu;
#ifndef GCR_SCAN_PREFETCH_DEFAULT
#define GCR_SCAN_PREFETCH_DEFAULT 4096
#endif
constexpr uint32_t kScanPrefetchDefault = GCR_SCAN_PREFETCH_DEFAULT;

enum : uint32_t { kT4 = 0, kA16 = 1, kA32 = 2, kA64 = 3, kA128 = 4, kA256 = 5 };
// GCR_SCAN_TIMES stamps per warp: entry, tables staged, first rows loaded (chunk 0), chunk 0 done, exit
constexpr uint32_t kStamps = kScanStamps;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// 16-byte streaming load that does not allocate in L1 (every byte is read once).
__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

// Request [p, p + bytes) into L2 (one bulk async prefetch; no completion to wait on).
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int kOff>
__device__ __forceinline__ uint32_t lds_imm(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(saddr), "n"(kOff));
    return v;
}

// x -> adv_512(x) through the lane-private braid tables (shared address sb =
// table base).  prmt(x, l*4, 0x55k4) = byte_k(x) << 8 | l*4 builds the scaled
// index in one instruction; the table number lives in the ld.shared
// immediate.  The base add runs on the FMA pipe (IMAD.IADD), which the
// lookups leave idle.  (A 64 KiB-aligned table base would fold it into the
// prmt but costs ~63 KiB of L1, which the streaming loads need in flight.)
__device__ __forceinline__ uint32_t braid(uint32_t x, uint32_t lane4, uint32_t sb) {
    const uint32_t i0 = prmt(x, lane4, 0x5504u) + sb;
    const uint32_t i1 = prmt(x, lane4, 0x5514u) + sb;
    const uint32_t i2 = prmt(x, lane4, 0x5524u) + sb;
    const uint32_t i3 = prmt(x, lane4, 0x5534u) + sb;
    return lds_imm<0>(i0) ^ lds_imm<128>(i1) ^ lds_imm<65536>(i2) ^ lds_imm<65536 + 128>(i3);
}

// v -> adv_d(v) through an unreplicated 4x256 table (used once per page).
__device__ __forceinline__ uint32_t apply_tab(const uint32_t *tb, uint32_t v) {
    return tb[v & 255u] ^ tb[256u + ((v >> 8) & 255u)] ^ tb[512u + ((v >> 16) & 255u)] ^
           tb[768u + (v >> 24)];
}

// The same step with the table base folded into the PRMT and the ld.shared
// immediate: lb = lane*4 | (sb & 0xFFFF0000) and prmt(x, lb, 0x76k4) = lb with
// byte 1 replaced by byte_k(x), so entry = that + ((sb & 0xFFFF) + table
// offset).  kSbLo is the compile-time guess of sb & 0xFFFF, checked per
// device by scan_probe() (the kernel's static shared layout fixes it): no
// per-lookup IADD.  ptxas folds the base into a uniform register for K1 but
// not for K1g (IMAD.IADD per lookup: 16 of ~60 instructions per row, ncu
// r2zb), which is where this is used.
template <uint32_t kSbLo>
__device__ __forceinline__ uint32_t braid_imm(uint32_t x, uint32_t lb) {
    return lds_imm<kSbLo>(prmt(x, lb, 0x7604u)) ^ lds_imm<kSbLo + 128>(prmt(x, lb, 0x7614u)) ^
           lds_imm<kSbLo + 65536>(prmt(x, lb, 0x7624u)) ^ lds_imm<kSbLo + 65536 + 128>(prmt(x, lb, 0x7634u));
}

template <uint32_t kSbLo>
__device__ __forceinline__ void row_step_imm(uint32_t lb, uint32_t (&x)[4], uint32_t &acc, const uint4 &w) {
    acc |= w.x | w.y | w.z | w.w;
    x[0] = braid_imm<kSbLo>(x[0], lb) ^ w.x;
    x[1] = braid_imm<kSbLo>(x[1], lb) ^ w.y;
    x[2] = braid_imm<kSbLo>(x[2], lb) ^ w.z;
    x[3] = braid_imm<kSbLo>(x[3], lb) ^ w.w;
}

__device__ __forceinline__ void row_step(uint32_t lane4, uint32_t sb, uint32_t (&x)[4], uint32_t &acc,
                                         const uint4 &w) {
    acc |= w.x | w.y | w.z | w.w;
    x[0] = braid(x[0], lane4, sb) ^ w.x;
    x[1] = braid(x[1], lane4, sb) ^ w.y;
    x[2] = braid(x[2], lane4, sb) ^ w.z;
    x[3] = braid(x[3], lane4, sb) ^ w.w;
}

// raw() of the warp's 512-byte Y block; valid in lane 0.  Tree level j only
// needs the lanes that are multiples of 2^(j+1): the others skip the lookups,
// which also thins the bank conflicts of these unreplicated tables (this
// per-page cost is what small pages pay on top of the braid lookups).
__device__ __forceinline__ uint32_t warp_raw(const uint32_t *small, const uint32_t (&x)[4], uint32_t lane) {
    const uint32_t *t4 = small + kT4 * 1024u;
    uint32_t v = apply_tab(t4, x[0]);
    v = apply_tab(t4, v ^ x[1]);
    v = apply_tab(t4, v ^ x[2]);
    v = apply_tab(t4, v ^ x[3]);
#pragma unroll
    for (int j = 0; j < 5; j++) {
        const uint32_t o = __shfl_down_sync(kFull, v, 1 << j);
        if ((lane & ((2u << j) - 1u)) == 0u) v = apply_tab(small + (kA16 + j) * 1024u, v) ^ o;
    }
    return v;
}

// Tile that anchors page pi of an allocation for compaction/pack: the tile
// holding it (P <= 64 KiB) or its first 64 KiB slice (P > 64 KiB).
__device__ __forceinline__ uint64_t tile_of_page(uint64_t tile0, uint64_t pi, uint32_t P, uint32_t lg) {
    return P <= kTileBytes ? tile0 + (pi >> (kLog2Tile - lg)) : tile0 + (pi << (lg - kLog2Tile));
}

// c.1 steps 3-5 for one page given its raw register and non-zero flag (or
// the A9 verify comparison), plus the per-tile compaction counters that K2
// turns into image offsets and chunk totals.  Executed by one lane.
__device__ __forceinline__ bool finalize_page(const ScanParams &p, uint64_t g, uint64_t tile, bool alloc_start,
                                              uint32_t len, uint32_t zlen, uint32_t raw, bool nz) {
    const uint32_t d = raw ^ zlen;
    if (p.mode == kScanVerify) {
        if (d != __ldg(p.d_ref + g)) {
            atomicAdd(p.verify_count, 1ull);
            atomicMin(p.first_bad, (unsigned long long)g);
        }
        return false;
    }
    uint8_t c;
    uint32_t inc;
    if (!nz) {
        c = kClsZero;
        inc = 1u << 10;
    } else if (p.mode == kScanIncremental && __ldg(p.d_ref + g) == d) {
        c = kClsParent;
        inc = 1u << 20;
    } else {
        c = kClsPresent;
        inc = 1u;
        atomicAdd(&p.tile_info[tile].present_bytes, len);
    }
    atomicAdd(&p.tile_info[tile].counts, inc);
    p.d_out[g] = d;
    p.cls[g] = c | (alloc_start ? kClsAllocStart : 0);
    return c == kClsPresent;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- f1 in-scan pack (InScanPack, gcr_internal.h) ---------------------------
__device__ __forceinline__ uint32_t *isp_list(const ScanParams &p, uint32_t par, uint64_t wid) {
    return p.isp.list + (par * p.workers + wid) * (uint64_t)p.isp.cap;
}

__device__ __forceinline__ uint64_t isp_tag(uint32_t epoch, uint32_t ch) {
    return ((uint64_t)(epoch & 0xFFFFu) << 48) | ((uint64_t)(ch & 0xFFFFu) << 32);
}

// Per-CTA shared state of the in-scan pack (two chunk parities).
struct IspShared {
    unsigned long long wagg[2][32];  // PRESENT bytes each warp finalized
    unsigned long long wpfx[2][32];  // exclusive prefix of those inside the CTA
    uint32_t wn[2][32];              // pages in each warp's list
    uint32_t cnt[2];                 // warps of the CTA done with the chunk
    uint32_t ready[2];               // ch + 1 once wpfx of the chunk is written
    uint32_t wdone;                  // chunk write-outs finished by the CTA's warps (monotonic)
    uint32_t par[32];                // each warp's current chunk parity
    uint32_t pad[27];
};

// One per CTA of K1 / K1g (file scope: the device functions below reach it
// without a parameter, so the scan's hot loop carries no f1 state in
// registers -- an earlier version kept an accumulator in the chunk context
// and the compiler scheduled the row loop's lookups with less latency slack).
__shared__ __align__(128) IspShared g_isp;

__device__ __forceinline__ void isp_init() {
    if (threadIdx.x < 2) {
        g_isp.cnt[threadIdx.x] = 0;
        g_isp.ready[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) g_isp.wdone = 0;
}

// Start of chunk ch for this warp: its counters of the chunk's parity.
__device__ __forceinline__ void isp_chunk_begin(uint32_t ch, uint32_t lane) {
    if (lane == 0) {
        const uint32_t wib = threadIdx.x >> 5, par = ch & 1u;
        g_isp.wagg[par][wib] = 0;
        g_isp.wn[par][wib] = 0;
        g_isp.par[wib] = par;
    }
    __syncwarp();
}

// One finalized PRESENT page (K1: lane 0, the only lane that finalizes).
__device__ __forceinline__ void isp_note(const ScanParams &p, uint64_t g, uint32_t len) {
    const uint32_t wib = threadIdx.x >> 5, par = g_isp.par[wib], n = g_isp.wn[par][wib];
    if (n < p.isp.cap) isp_list(p, par, (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib)[n] = (uint32_t)g;
    else atomicCAS(p.isp.err, 0ull, 4ull);  // list overflow
    g_isp.wn[par][wib] = n + 1;
    g_isp.wagg[par][wib] += len;
}

// Before a warp records pages of chunk ch (ch >= 2) into the list slot of
// chunk ch - 2 (two parities), every warp of the CTA must be done writing
// chunk ch - 2 out: the write-out of a chunk is shared by the CTA's warps and
// reads all of their lists.  Bounded; a timeout is reported like the others.
__device__ __forceinline__ void isp_lists_free(const ScanParams &p, IspShared &ss, uint32_t ch) {
    if (ch < 2) return;
    const uint32_t need = (blockDim.x >> 5) * (ch - 1);
    const uint64_t t0 = globaltimer_ns();
    while (*reinterpret_cast<volatile uint32_t *>(&ss.wdone) < need)
        if (globaltimer_ns() - t0 > p.isp.wait_ns) {
            if ((threadIdx.x & 31u) == 0) atomicCAS(p.isp.err, 0ull, 5ull | (uint64_t)ch << 8);
            break;
        }
}

// End of chunk ch for this warp: publish its aggregate in the CTA; the CTA's
// last warp writes the in-CTA prefixes and the CTA aggregate (global).
__device__ __forceinline__ void isp_chunk_end(const ScanParams &p, IspShared &ss, uint32_t ch, uint32_t lane) {
    const uint32_t par = ch & 1u, nw = blockDim.x >> 5;
    uint32_t arrived = 0;
    if (lane == 0) {  // the warp's counters are final (isp_note, in this warp)
        __threadfence_block();
        arrived = atomicAdd(&ss.cnt[par], 1u);
    }
    arrived = __shfl_sync(kFull, arrived, 0);
    if (arrived == nw - 1) {  // the CTA's last warp for this chunk
        __threadfence_block();
        const unsigned long long v = lane < nw ? *reinterpret_cast<volatile unsigned long long *>(&ss.wagg[par][lane]) : 0ull;
        unsigned long long inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, inc, d);
            if (lane >= (uint32_t)d) inc += o;
        }
        if (lane < nw) ss.wpfx[par][lane] = inc - v;
        const unsigned long long tot = __shfl_sync(kFull, inc, nw - 1);
        if (lane == 0) {
            ss.cnt[par] = 0;
            p.isp.cta_agg[(uint64_t)ch * gridDim.x + blockIdx.x] = isp_tag(p.epoch, ch) | tot;
            __threadfence();
            __threadfence_block();
            *reinterpret_cast<volatile uint32_t *>(&ss.ready[par]) = ch + 1;
        }
    }
}

// Write chunk ch's PRESENT pages finalized by this warp into the image.
__device__ __forceinline__ void isp_write(const ScanParams &p, IspShared &ss, uint32_t ch, uint64_t wid,
                                          uint32_t lane) {
    const uint32_t par = ch & 1u, wib = threadIdx.x >> 5;
    const uint64_t t0 = globaltimer_ns(), lim = p.isp.wait_ns;
    uint32_t why = 0;  // which wait timed out (error word: why | chunk << 8 | CTA << 32)
    // the in-CTA prefix of this chunk
    while (*reinterpret_cast<volatile uint32_t *>(&ss.ready[par]) != ch + 1u)
        if (globaltimer_ns() - t0 > lim) { why = 1; break; }
    // PRESENT bytes of the earlier CTAs (their aggregates carry this chunk's tag)
    unsigned long long before = 0;
    const uint64_t tag = isp_tag(p.epoch, ch);
    for (uint32_t b = lane; !why && b < blockIdx.x; b += 32u) {
        unsigned long long v;
        while (((v = *reinterpret_cast<volatile unsigned long long *>(p.isp.cta_agg + (uint64_t)ch * gridDim.x + b)) >> 32) !=
               tag >> 32)
            if (globaltimer_ns() - t0 > lim) { why = 2; break; }
        before += v & 0xFFFFFFFFull;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) before += __shfl_xor_sync(kFull, before, d);
    // the chunk's image offset, from K2 of the previous chunk
    if (ch != 0 && !why)
        while (*reinterpret_cast<volatile uint32_t *>(p.isp.base_ready + ch) != p.epoch)
            if (globaltimer_ns() - t0 > lim) { why = 3; break; }
    why = __reduce_max_sync(kFull, why);
    if (why) {
        if (lane == 0) {
            atomicCAS(p.isp.err, 0ull, (unsigned long long)why | (uint64_t)ch << 8 | (uint64_t)blockIdx.x << 32);
            atomicAdd(&ss.wdone, 1u);
        }
        return;
    }
    __threadfence();
    // The CTA's chunk-ch pages (its warps' lists in warp order) cover image
    // bytes [cta0, cta0 + T); warp wib writes the 512-B-aligned share
    // [s0, s1) of them, so one CTA's pages are written by all its warps
    // (a single warp writing a few 64 KiB pages over PCIe would otherwise
    // trail the chunk by tens of microseconds).
    const uint32_t nw = blockDim.x >> 5;
    const unsigned long long cta0 = (ch ? *reinterpret_cast<volatile unsigned long long *>(p.isp.base + ch) : 0ull) + before;
    const unsigned long long T = ss.wpfx[par][nw - 1] + ss.wagg[par][nw - 1];
    const unsigned long long s0 = (T * wib / nw) & ~511ull, s1 = wib + 1 == nw ? T : (T * (wib + 1) / nw) & ~511ull;
    const uint32_t P = p.page_size, lg = p.log2_page;
    for (uint32_t v = 0; v < nw && s0 < s1; v++) {
        unsigned long long r = ss.wpfx[par][v];
        if (r >= s1) break;
        if (r + ss.wagg[par][v] <= s0) continue;
        const uint32_t n = min(ss.wn[par][v], p.isp.cap);
        const uint32_t *list = isp_list(p, par, (uint64_t)blockIdx.x * nw + v);
        for (uint32_t k = 0; k < n && r < s1; k++) {
            const uint64_t g = __ldcg(list + k);  // written in this launch: not the read-only path
            const AllocDev *al = p.allocs + __ldg(p.isp_page_alloc + g);
            const uint64_t pi = g - __ldg(&al->page0);
            const uint32_t len = pi == (uint64_t)__ldg(&al->n_pages) - 1 ? __ldg(&al->tail_len) : P;
            const unsigned long long a = max(r, s0), b = min(r + len, s1);
            if (a < b) {
                const uint8_t *src = reinterpret_cast<const uint8_t *>(__ldg(&al->base) + (pi << lg)) + (a - r);
                uint8_t *dst = p.isp.img + cta0 + a;
                const uint32_t m = (uint32_t)(b - a);
                uint32_t o = lane * 16u;
                for (; o + 3 * 512u < m; o += 4 * 512u) {
                    uint4 x[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) x[u] = ldg_stream(src + o + u * 512u);
#pragma unroll
                    for (int u = 0; u < 4; u++) *reinterpret_cast<uint4 *>(dst + o + u * 512u) = x[u];
                }
                for (; o < m; o += 512u) *reinterpret_cast<uint4 *>(dst + o) = ldg_stream(src + o);
            }
            r += len;
        }
    }
    __syncwarp();
    if (lane == 0) atomicAdd(&ss.wdone, 1u);  // this warp is done with the CTA's lists of chunk ch
}

// GF(2) product m (*) v mod P in the reflected representation (bit 31 = x^0):
// the sum over the set bits 31-k of m of v * x^k.  Lane k forms v * x^k (k
// single-bit register steps, predicated so the loop is warp-uniform), and a
// 5-level XOR butterfly sums the lanes.  All lanes return the product.
__device__ __forceinline__ uint32_t warp_mulmod(uint32_t m, uint32_t v, uint32_t lane) {
    constexpr uint32_t kPoly = 0x82F63B78u;
#pragma unroll 1
    for (uint32_t s = 0; s < 31; s++)
        if (s < lane) v = (v >> 1) ^ ((v & 1u) ? kPoly : 0u);
    uint32_t t = (m >> (31u - lane)) & 1u ? v : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) t ^= __shfl_xor_sync(kFull, t, o);
    return t;
}

// The chunk a warp is scanning: its real rows and its fold slots.
struct ChunkCtx {
    uint64_t rb, rows;  // first global real row, real rows
    unsigned long long *fs;  // fold slots of this chunk (one per warp)
};

// A piece of a cut page arrives at the page's owner slot (executed by one
// lane).  The piece's contribution is already advanced to the page end.  One
// 64-bit CAS folds {XOR contribution, + rows, + non-zero} (FoldSlots); the
// arrival that completes the page's Rp - r0 real rows finalizes it from its
// own CAS result.
template <bool kIsp>
__device__ __forceinline__ void fold_arrive(const ScanParams &p, ChunkCtx &cc, uint64_t g, uint32_t a,
                                            uint32_t pi, uint32_t r0, uint32_t rows, uint32_t contrib, bool nz) {
    const uint32_t P = p.page_size, lg = p.log2_page, Rp = P >> kLog2Row;
    const AllocDev *al = p.allocs + a;
    // owner: the last warp whose range starts at or before the page's first
    // real row; ranges are [rows*w/W, rows*(w+1)/W) relative to the chunk
    const uint64_t x = __ldg(&al->row0) + (uint64_t)pi * Rp - cc.rb;
    const uint64_t owner = ((x + 1) * p.workers - 1) / cc.rows;
    unsigned long long *slot = cc.fs + owner;
    const unsigned long long add = ((unsigned long long)rows << 32) | (nz ? 1ull << 48 : 0ull);
    unsigned long long old = 0ull, nv;
    for (;;) {  // first guess: the slot is empty
        nv = (old ^ contrib) + add;  // contrib < 2^32: the XOR only touches the low word
        const unsigned long long seen = atomicCAS(slot, old, nv);
        if (seen == old) break;
        old = seen;
    }
    if (((nv >> 32) & 0xFFFFull) != Rp - r0) return;
    *slot = 0ull;  // every piece arrived: the slot is free for the next launch
    const uint32_t n_pages = __ldg(&al->n_pages);
    const bool tail = pi == n_pages - 1;
    const uint32_t len = tail ? __ldg(&al->tail_len) : P;
    if (finalize_page(p, g, tile_of_page(__ldg(&al->tile0), pi, P, lg), pi == 0, len,
                      tail ? __ldg(&al->z_tail) : p.z_page, (uint32_t)nv, (nv >> 48) != 0ull) &&
        (kIsp && p.isp.img))
        isp_note(p, g, len);
}

// Block-wide exclusive scan of one u64 per thread (blockDim.x <= 1024).
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long *total) {
    __shared__ unsigned long long warp_sums[32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(kFull, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x >> 5;
        unsigned long long s = lane < nw ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, s, d);
            if (lane >= (uint32_t)d) s += o;
        }
        if (lane < nw) warp_sums[lane] = s;  // inclusive
    }
    __syncthreads();
    const unsigned long long before = warp == 0 ? 0ull : warp_sums[warp - 1];
    const unsigned long long res = before + inc - v;
    if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return res;
}

// K2: chunk-local exclusive scan of PRESENT bytes over the chunk's tiles;
// re-zeroes the tile counters; writes the chunk totals and the NON-EMPTY
// tiles, compacted, into mapped pinned host memory ({tile, present bytes,
// image offset}; count in rec_count) so the host plans the drain from ~d*T
// records instead of T.  One CTA: the chunk's counters are staged in shared
// memory with coalesced loads, each thread then scans a contiguous run of
// tiles.  Enqueued ahead on the post stream; it first waits until the
// persistent K1 publishes the chunk (chunk_done[chunk] == epoch), bounded by
// kChunkWaitNs (a timeout reports image_bytes = ~0 and the checkpoint fails).
constexpr int kTileScanThreads = 1024;
constexpr uint64_t kChunkWaitNs = 30ull * 1000000000ull;


__global__ void __launch_bounds__(kTileScanThreads) k_tile_scan(TileInfo *ti, uint64_t tb, uint64_t te,
                                                                const uint32_t *chunk_done, uint32_t chunk,
                                                                uint32_t epoch, TileRec *host_rec,
                                                                unsigned long long *rec_count,
                                                                ChunkTotals *totals_host,
                                                                unsigned long long *isp_base, uint32_t *isp_ready) {
    extern __shared__ uint32_t pb[];  // present bytes per tile of the chunk
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
        const uint64_t t0 = globaltimer_ns();
        int to = 0;
        while (*reinterpret_cast<const volatile uint32_t *>(chunk_done + chunk) != epoch) {
            if (globaltimer_ns() - t0 > kChunkWaitNs) {
                to = 1;
                break;
            }
            __nanosleep(200);
        }
        __threadfence();
        timed_out = to;
    }
    __syncthreads();
    if (timed_out) {
        if (threadIdx.x == 0) {
            reinterpret_cast<volatile unsigned long long *>(totals_host)[0] = ~0ull;
            *reinterpret_cast<volatile unsigned long long *>(rec_count) = 0ull;
            __threadfence_system();
        }
        return;
    }
    const uint32_t n = (uint32_t)(te - tb);
    unsigned long long np = 0, nz = 0, npa = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        // written by the concurrently running K1 (atomics at L2): bypass L1
        const uint2 v = __ldcg(reinterpret_cast<const uint2 *>(ti + tb + i));
        const TileInfo x{v.x, v.y};
        pb[i] = x.present_bytes;
        np += x.counts & 1023u;
        nz += (x.counts >> 10) & 1023u;
        npa += (x.counts >> 20) & 1023u;
        ti[tb + i] = TileInfo{0u, 0u};
    }
    __syncthreads();
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(n, per * threadIdx.x), hi = min(n, lo + per);
    unsigned long long s = 0, cnt = 0;
    for (uint32_t i = lo; i < hi; i++) {
        s += pb[i];
        cnt += pb[i] != 0u;
    }
    unsigned long long tot_b, tot_c, tp, tz, tpa;
    unsigned long long off = block_exclusive_scan(s, &tot_b);
    unsigned long long k = block_exclusive_scan(cnt, &tot_c);
    block_exclusive_scan(np, &tp);
    block_exclusive_scan(nz, &tz);
    block_exclusive_scan(npa, &tpa);
    for (uint32_t i = lo; i < hi; i++) {
        if (pb[i]) {
            TileRec *r = host_rec + k;
            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(r), "r"(i), "r"(pb[i]),
                         "r"((uint32_t)off), "r"(0u)
                         : "memory");
            k++;
        }
        off += pb[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned long long *h = reinterpret_cast<volatile unsigned long long *>(totals_host);
        h[0] = tot_b;
        h[1] = tp;
        h[2] = tz;
        h[3] = tpa;
        *reinterpret_cast<volatile unsigned long long *>(rec_count) = tot_c;
        if (isp_base) {  // f1: the next chunk's image offset for the in-scan pack (K2s run in chunk order)
            const unsigned long long b = chunk ? *reinterpret_cast<volatile unsigned long long *>(isp_base + chunk) : 0ull;
            *reinterpret_cast<volatile unsigned long long *>(isp_base + chunk + 1) = b + tot_b;
            __threadfence();
            *reinterpret_cast<volatile uint32_t *>(isp_ready + chunk + 1) = epoch;
        }
        __threadfence_system();
    }
}

// Allocation holding global real row r: 32-ary search by the warp (each round
// every lane probes one row0; one ballot narrows the range 32x).
__device__ __forceinline__ uint32_t alloc_of_row(const AllocDev *al, uint32_t n, uint64_t r, uint32_t lane) {
    uint32_t lo = 0, hi = n;  // al[lo].row0 <= r < al[hi].row0 (al[n] = +inf)
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t probe = lo + lane * step;
        const bool le = probe < hi && __ldg(&al[probe].row0) <= r;
        const uint32_t qm = 31 - __clz(__ballot_sync(kFull, le));  // lane 0 (probe = lo) always qualifies
        lo = lo + qm * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// Cached fields of one allocation (warp-uniform registers).
struct AllocView {
    uint64_t base, page0, tile0;
    uint32_t n_pages, tail_len, z_tail, nfull;  // nfull: pages of length P
};

__device__ __forceinline__ AllocView load_alloc(const AllocDev *al, uint32_t P) {
    AllocView v;
    v.base = __ldg(&al->base);
    v.page0 = __ldg(&al->page0);
    v.tile0 = __ldg(&al->tile0);
    v.n_pages = __ldg(&al->n_pages);
    v.tail_len = __ldg(&al->tail_len);
    v.z_tail = __ldg(&al->z_tail);
    v.nfull = v.n_pages - (v.tail_len < P ? 1u : 0u);
    return v;
}

// Both cursors walk the same sequence of PAGES; a block is the next
// cnt = min(U, Rp - vr, rows left) rows, so a block never crosses a page (and
// hence never an allocation or a short-page boundary): loads are U predicated
// independent LDG.128 from one base, and a page ends only after a block.

// LOAD cursor: this lane's pointer to the next row of its current page.
struct LoadCursor {
    const char *addr;
    uint32_t a, pi, vr;
    uint64_t base, end;  // the current allocation's [base, end)
    uint32_t n_pages, tail_len;
    bool mask;  // next row is the first row of a short page and this lane's 16 B lie in its padding
};

__device__ __forceinline__ void lc_next_page(LoadCursor &lc, const AllocDev *allocs, uint32_t P, uint32_t lg,
                                          uint32_t lane) {
    if (++lc.pi == lc.n_pages) {
        const AllocDev *al = allocs + (++lc.a);
        lc.base = __ldg(&al->base);
        lc.end = lc.base + __ldg(&al->bytes);
        lc.n_pages = __ldg(&al->n_pages);
        lc.tail_len = __ldg(&al->tail_len);
        lc.pi = 0;
    }
    const bool tail = lc.pi == lc.n_pages - 1 && lc.tail_len < P;
    const uint32_t pad = tail ? P - lc.tail_len : 0u;
    lc.vr = pad >> kLog2Row;
    lc.addr = reinterpret_cast<const char *>(lc.base + ((uint64_t)lc.pi << lg)) - pad + (lc.vr << kLog2Row) +
              lane * 16u;
    lc.mask = (lc.vr << kLog2Row) + lane * 16u < pad;
}

template <int U>
__device__ __forceinline__ void load_rows(uint4 (&w)[U], int &left, LoadCursor &lc, const AllocDev *allocs,
                                          uint32_t P, uint32_t lg, uint32_t lane, uint32_t pf) {
    const uint32_t Rp = P >> kLog2Row;
    if (lc.vr == Rp) lc_next_page(lc, allocs, P, lg, lane);
    const int cnt = min(min(U, left), (int)(Rp - lc.vr));
    // keep the stream requested pf bytes ahead: the block pf bytes past this
    // one, if it still lies in this warp's range and in this allocation (the
    // real rows of an allocation are contiguous in memory)
    if (pf != 0u && lane == 0u) {
        const uint64_t a = reinterpret_cast<uint64_t>(lc.addr) + pf;
        if ((uint64_t)left * kRowBytes >= pf + U * kRowBytes && a >= lc.base && a + U * kRowBytes <= lc.end)
            prefetch_l2(reinterpret_cast<const void *>(a), U * kRowBytes);
    }
    if (cnt == U && !lc.mask) {
#pragma unroll
        for (int u = 0; u < U; u++) w[u] = ldg_stream(lc.addr + (u << kLog2Row));
    } else {
#pragma unroll
        for (int u = 0; u < U; u++)
            if (u < cnt) w[u] = (u == 0 && lc.mask) ? make_uint4(0, 0, 0, 0) : ldg_stream(lc.addr + (u << kLog2Row));
    }
    lc.addr += cnt << kLog2Row;
    lc.vr += cnt;
    lc.mask = false;
    left -= cnt;
}

// PROCESS cursor: the page being digested and where this warp's part of it
// started (vstart == r0: the warp saw the whole page).
struct ProcCursor {
    AllocView al;
    uint32_t a, pi, vr, vstart, r0;
};

__device__ __forceinline__ void pc_set_page(ProcCursor &pc, uint32_t P) {
    const bool tail = pc.pi == pc.al.n_pages - 1 && pc.al.tail_len < P;
    pc.r0 = tail ? (P - pc.al.tail_len) >> kLog2Row : 0u;
    pc.vr = pc.r0;
    pc.vstart = pc.r0;
}

// Page complete (vr == Rp): digest it (or leave a piece) and move on.
template <bool kIsp>
__device__ __forceinline__ void page_end(const ScanParams &p, ChunkCtx &cc, ProcCursor &pc, uint32_t (&x)[4],
                                         uint32_t &acc, const uint32_t *small, uint32_t lane) {
    const uint32_t P = p.page_size, lg = p.log2_page;
    const uint32_t raw = warp_raw(small, x, lane);
    const bool nz = __any_sync(kFull, acc != 0);
    const bool whole = pc.vstart == pc.r0;
    if (lane == 0) {
        const uint64_t g = pc.al.page0 + pc.pi;
        if (whole) {
            const bool tail = pc.pi == pc.al.n_pages - 1;
            const uint32_t len = tail ? pc.al.tail_len : P;
            if (finalize_page(p, g, tile_of_page(pc.al.tile0, pc.pi, P, lg), pc.pi == 0, len,
                              tail ? pc.al.z_tail : p.z_page, raw, nz) &&
                (kIsp && p.isp.img))
                isp_note(p, g, len);
        } else {  // the page's last piece: nothing left to advance over
            fold_arrive<kIsp>(p, cc, g, pc.a, pc.pi, pc.r0, (P >> kLog2Row) - pc.vstart, raw, nz);
        }
    }
    x[0] = x[1] = x[2] = x[3] = 0u;
    acc = 0u;
    if (++pc.pi == pc.al.n_pages) {
        if (++pc.a < p.n_allocs) pc.al = load_alloc(p.allocs + pc.a, P);
        pc.pi = 0;
    }
    pc_set_page(pc, P);
}

// Digest the next block (the same cnt rows load_rows fetched into w).
template <int U, bool kIsp>
__device__ __forceinline__ void process_rows(const ScanParams &p, ChunkCtx &cc, ProcCursor &pc, const uint4 (&w)[U],
                                             int &left, uint32_t (&x)[4], uint32_t &acc, const uint32_t *small,
                                             uint32_t lane4, uint32_t sb, uint32_t lane) {
    const uint32_t Rp = p.page_size >> kLog2Row;
    const int cnt = min(min(U, left), (int)(Rp - pc.vr));
    if (cnt == U) {
#pragma unroll
        for (int u = 0; u < U; u++) row_step(lane4, sb, x, acc, w[u]);
    } else {
#pragma unroll
        for (int u = 0; u < U; u++)
            if (u < cnt) row_step(lane4, sb, x, acc, w[u]);
    }
    pc.vr += cnt;
    left -= cnt;
    if (pc.vr == Rp) page_end<kIsp>(p, cc, pc, x, acc, small, lane);
}

// Build the tables in shared memory from the launch's basis vectors
// (ScanParams::basis, constant bank): entry e of table k = XOR of basis[8k + i]
// over the set bits i of e.  The braid table goes into all 32 lane-private
// replicas (word (k>>1)*16384 + e*64 + (k&1)*32 + l), the small tables (t4,
// a16 .. a256) once.  Every warp works on one k at a time (k is warp-uniform),
// so the basis reads are constant-bank broadcasts.
__device__ __forceinline__ uint32_t tab_entry(const uint32_t *b32, uint32_t k, uint32_t e) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 4; i++)
        if ((e >> i) & 1u) v ^= b32[8 * k + i];
    return v;
}

// Two phases.  (1) The 7 tables' NIBBLE tables -- entry n of half h of byte
// position k of table t = XOR of basis[t][8k + 4h + i] over the set bits i of
// n -- into a 3.5 KiB scratch at the end of the dynamic smem (896 entries,
// one or two per thread, from the constant bank).  (2) Every table entry =
// lo-nibble entry ^ hi-nibble entry (two broadcast LDS): the braid table into
// all 32 lane-private replicas -- 8 threads write one entry's 128 contiguous
// replica bytes, one conflict-free STS.128 phase -- and the small tables
// (t4, a16 .. a256) once.  (One thread per replicated entry, 8 stores each,
// put every lane of a store phase on the same 4 banks: 8-way conflicts, ~4 us
// per launch; building every entry straight from the 8 basis values cost
// ~700 instructions per thread.)
__device__ __forceinline__ void stage_tables(uint32_t *sm, const ScanParams &p) {
    uint32_t *nib = sm + (kBraidSmem + kSmallTables * 4096u) / 4;
    for (uint32_t i = threadIdx.x; i < kNibWords; i += kScanThreads) {
        const uint32_t t = i >> 7, k = (i >> 5) & 3u, h = (i >> 4) & 1u, n = i & 15u;
        nib[i] = tab_entry(p.basis[t] + 4 * h, k, n);  // basis words 8k + 4h + (0..3)
    }
    __syncthreads();
    constexpr uint32_t kGroups = kScanThreads / 8;
    const uint32_t sub = threadIdx.x & 7u;
    for (uint32_t ke = threadIdx.x >> 3; ke < 1024u; ke += kGroups) {
        const uint32_t k = ke >> 8, e = ke & 255u;
        const uint32_t v = nib[k * 32 + (e & 15u)] ^ nib[k * 32 + 16 + (e >> 4)];
        uint4 *dst = reinterpret_cast<uint4 *>(sm + (k >> 1) * 16384u + e * 64u + (k & 1u) * 32u) + sub;
        *dst = make_uint4(v, v, v, v);
    }
    uint32_t *ss = sm + kBraidSmem / 4;
    for (uint32_t i = threadIdx.x; i < kSmallTables * 1024u; i += kScanThreads) {
        const uint32_t t = 1 + (i >> 10), k = (i >> 8) & 3u, e = i & 255u;
        ss[i] = nib[t * 128 + k * 32 + (e & 15u)] ^ nib[t * 128 + k * 32 + 16 + (e >> 4)];
    }
    if (p.t4rep) {  // K1g: t4 x 8 after the nibble scratch; two 16-B stores per entry, contiguous per warp
        uint32_t *tr = sm + kScanSmem / 4;
        for (uint32_t h = threadIdx.x; h < 2048u; h += kScanThreads) {
            const uint32_t i = h >> 1, k = i >> 8, e = i & 255u;
            const uint32_t v = nib[128 + k * 32 + (e & 15u)] ^ nib[128 + k * 32 + 16 + (e >> 4)];
            *reinterpret_cast<uint4 *>(tr + i * 8u + (h & 1u) * 4u) = make_uint4(v, v, v, v);
        }
    }
}

// K1.
// kIsp = false (K1 scans without the f1 in-scan pack): the f1 hooks compiled
// out -- same box, alternating (profiles/r2zq_*, r2zr_*): the incremental K1
// 5.35 -> 5.51 TB/s, the full K1 +1 % with them gone.
template <bool kIsp>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan(const ScanParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);  // braid tables at the dynamic smem base
    const uint32_t *small = sm + kBraidSmem / 4;
    if (kIsp && p.isp.img) isp_init();

    const uint64_t t_entry = p.warp_times ? globaltimer_ns() : 0ull;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lane4 = lane * 4u;
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    stage_tables(sm, p);
    __syncthreads();
    if (wid >= p.workers) return;
    if (p.warp_times && lane == 0) {
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        p.warp_times[kStamps * wid] = t_entry;
        p.warp_times[kStamps * wid + 1] = globaltimer_ns();  // tables staged
        p.warp_times[kStamps * wid + 5] = smid;
    }
    const uint32_t P = p.page_size, lg = p.log2_page;
    const uint32_t Rp = P >> kLog2Row;
    for (uint32_t ch = 0; ch < p.n_chunks; ch++) {
        // chunks merge_from .. n_chunks-1 form ONE range split over the warps
        // (full checkpoints: see ScanParams::merge_from); published together
        const uint32_t ch_end = p.merge_from && ch == p.merge_from ? p.n_chunks : ch + 1;
        ChunkCtx cc;
        cc.rb = p.chunk_rows[ch];
        cc.rows = p.chunk_rows[ch_end] - cc.rb;
        cc.fs = p.fold.s + (uint64_t)ch * p.workers;
        if (kIsp && p.isp.img) {
            isp_lists_free(p, g_isp, ch);
            isp_chunk_begin(ch, lane);
        }
        const uint64_t r = cc.rb + cc.rows * wid / p.workers;
        const uint64_t rend = cc.rb + cc.rows * (wid + 1) / p.workers;
        if (r < rend) {
            const uint32_t a = alloc_of_row(p.allocs, p.n_allocs, r, lane);
            // position of row r: a full page, or the short tail page
            ProcCursor pc;
            pc.a = a;
            pc.al = load_alloc(p.allocs + a, P);
            const uint64_t lr = r - __ldg(&p.allocs[a].row0);
            uint32_t pad0 = 0;  // padding of the first page (non-zero only for a short tail page)
            if (lr < ((uint64_t)pc.al.nfull << (lg - kLog2Row))) {
                pc.pi = (uint32_t)(lr >> (lg - kLog2Row));
                pc.r0 = 0;
                pc.vr = (uint32_t)(lr & (Rp - 1));
            } else {
                pc.pi = pc.al.n_pages - 1;
                pad0 = P - pc.al.tail_len;
                pc.r0 = pad0 >> kLog2Row;
                pc.vr = (uint32_t)(lr - ((uint64_t)pc.al.nfull << (lg - kLog2Row))) + pc.r0;
            }
            pc.vstart = pc.vr;
            LoadCursor lc;
            lc.a = a;
            lc.pi = pc.pi;
            lc.vr = pc.vr;
            lc.base = pc.al.base;
            lc.end = pc.al.base + __ldg(&p.allocs[a].bytes);
            lc.n_pages = pc.al.n_pages;
            lc.tail_len = pc.al.tail_len;
            lc.addr = reinterpret_cast<const char *>(pc.al.base + ((uint64_t)pc.pi << lg)) - pad0 +
                      (pc.vr << kLog2Row) + lane * 16u;
            lc.mask = pc.vr == pc.r0 && (pc.r0 << kLog2Row) + lane * 16u < pad0;

            constexpr int U = kScanUnroll;
            int to_load = (int)(rend - r), to_proc = to_load;
            if (p.prefetch != 0u && lane == 0u) {  // the range's first pf bytes (clamped to the allocation)
                const uint64_t a0 = max(reinterpret_cast<uint64_t>(lc.addr), lc.base);  // a short page's row may start before it
                const uint64_t e = min(min(a0 + p.prefetch, lc.end), a0 + (uint64_t)to_load * kRowBytes);
                if (e > a0) prefetch_l2(reinterpret_cast<const void *>(a0), (uint32_t)(e - a0));
            }
            uint32_t x[4] = {0u, 0u, 0u, 0u}, acc = 0u;
            uint4 wa[U], wb[U];
            load_rows<U>(wa, to_load, lc, p.allocs, P, lg, lane, p.prefetch);
            if (p.warp_times && ch == 0) {  // first rows in registers: the range's first HBM round trip
                uint32_t dep = wa[0].x;
                asm volatile("mov.b32 %0, %0;" : "+r"(dep));  // wait for the load before the stamp
                const uint64_t t = globaltimer_ns();
                if (lane == 0) p.warp_times[kStamps * wid + 2] = t;
                wa[0].x = dep;
            }
            while (to_proc > 0) {
                if (to_load > 0) load_rows<U>(wb, to_load, lc, p.allocs, P, lg, lane, p.prefetch);
                process_rows<U, kIsp>(p, cc, pc, wa, to_proc, x, acc, small, lane4, sb, lane);
                if (to_proc <= 0) break;
                if (to_load > 0) load_rows<U>(wa, to_load, lc, p.allocs, P, lg, lane, p.prefetch);
                process_rows<U, kIsp>(p, cc, pc, wb, to_proc, x, acc, small, lane4, sb, lane);
            }
            // the range ended inside a page: advance the piece to the page end
            // (d = Rp - vr rows) and arrive at the page's owner slot
            if (pc.vr != pc.vstart) {
                const uint32_t raw = __shfl_sync(kFull, warp_raw(small, x, lane), 0);
                const bool nz = __any_sync(kFull, acc != 0);
                const uint32_t contrib = warp_mulmod(__ldg(&p.tables->fold_m[Rp - pc.vr]), raw, lane);
                if (lane == 0)
                    fold_arrive<kIsp>(p, cc, pc.al.page0 + pc.pi, pc.a, pc.pi, pc.r0, pc.vr - pc.vstart, contrib, nz);
            }
        }
        if (kIsp && p.isp.img) isp_chunk_end(p, g_isp, ch, lane);  // f1: the warp's aggregate
        // this warp is done with chunk ch (.. ch_end - 1); the last one publishes it for K2
        if (lane == 0) {
            __threadfence();
            if (atomicAdd(p.chunk_arrive + ch, 1u) == (uint32_t)p.workers - 1u) {
                atomicExch(p.chunk_arrive + ch, 0u);
                __threadfence();
                for (uint32_t c2 = ch; c2 < ch_end; c2++) atomicExch(p.chunk_done + c2, p.epoch);
            }
        }
        __syncwarp();
        if (p.warp_times && lane == 0 && ch == 0) p.warp_times[kStamps * wid + 3] = globaltimer_ns();
        // f1: write the previous chunk's PRESENT pages (every aggregate of it is
        // published by now, normally without waiting)
        if (kIsp && p.isp.img && ch >= 1) isp_write(p, g_isp, ch - 1, wid, lane);
        if (ch_end == p.n_chunks) break;
    }
    if (kIsp && p.isp.img && p.n_chunks) isp_write(p, g_isp, p.n_chunks - 1, wid, lane);
    if (p.warp_times && lane == 0) p.warp_times[kStamps * wid + 4] = globaltimer_ns();
}

// ---------------------------------------------------------------------------
// K1g: the scan for small pages (P = 4 KiB: G = 4; 8 KiB: G = 2).  At 4 KiB
// K1 finalizes a page every 8 rows and the per-page raw16 + lane tree (through
// unreplicated, bank-conflicting tables) costs as much as the page's braid
// lookups.  K1g streams a GROUP of G consecutive pages of one allocation (16
// KiB) as 32 rows of 512 bytes in which lanes [q*QL, (q+1)*QL) (QL = 32/G) read
// page q's next 512/G bytes: the braid step is adv_{512/G} (the a128 / a256
// table, staged lane-private), each page's 512/G-byte Y block sits in its own
// lane group, and ONE raw16 + log2(QL)-level tree finalizes all G pages.
// Warps take whole groups (equal split of the chunk's groups), so no page is
// ever cut between warps: no fold.  Loads stay full 128-byte lines.  A short
// tail page is front-padded with zeros as in K1; a last group with fewer than
// G pages masks the missing pages' lanes.
template <int G>
struct GroupLane {  // this lane's page in the current group
    const char *ptr;  // address of row 0 for this lane (front padding included)
    uint32_t pad;     // front padding bytes of a short tail page (0 otherwise)
    uint32_t pi;      // page index in the allocation
    bool valid;       // the page exists (partial last group)
};

template <int G>
__device__ __forceinline__ GroupLane<G> group_lane(const AllocView &al, uint64_t gi, uint32_t P, uint32_t lg,
                                                   uint32_t q, uint32_t m) {
    GroupLane<G> gl;
    gl.pi = (uint32_t)(gi * G + q);
    gl.valid = gl.pi < al.n_pages;
    const bool tail = gl.valid && gl.pi == al.n_pages - 1 && al.tail_len < P;
    gl.pad = tail ? P - al.tail_len : 0u;
    gl.ptr = reinterpret_cast<const char *>(al.base + ((uint64_t)gl.pi << lg)) - gl.pad + m * 16u;
    return gl;
}

__device__ __forceinline__ uint32_t alloc_of_group(const AllocDev *al, uint32_t n, uint64_t g, uint32_t lane) {
    uint32_t lo = 0, hi = n;  // al[lo].grp0 <= g < al[hi].grp0
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t probe = lo + lane * step;
        const bool le = probe < hi && __ldg(&al[probe].grp0) <= g;
        const uint32_t qm = 31 - __clz(__ballot_sync(kFull, le));
        lo = lo + qm * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// K1g's dynamic shared-memory base, low 16 bits, as laid out by this build
// (1 KiB reserved + the f1 state in static shared memory); verified per device
// by scan_probe(), which falls back to the IADD variant on a mismatch.
// Two immediate-base instances: with the f1 hooks (the f1 state in static
// shared memory moves the dynamic base to 0xA00) and without them (0x400).
#ifndef GCR_GRP_SB_LO
#define GCR_GRP_SB_LO 0xA00
#endif
#ifndef GCR_GRP_SB_LO_PLAIN
#define GCR_GRP_SB_LO_PLAIN 0x400
#endif
constexpr uint32_t kGrpSbLo = GCR_GRP_SB_LO, kGrpSbLoPlain = GCR_GRP_SB_LO_PLAIN;

// kImm: table base in the PRMT + immediate (else the IADD per lookup);
// kHooks: the f1 in-scan-pack hooks compiled in (K1 measured 3 % slower with
// them, profiles/r2zq_*; scans without f1 run a hook-free instance).
template <int G, bool kImm, bool kHooks>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan_grp(const ScanParams p) {
    constexpr uint32_t QL = 32 / G, Wr = kRowBytes / G, Rg = 32, U = 4, NB = Rg / U;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    if (p.sb_probe) {  // scan_probe(): report the base, do nothing else
        if (threadIdx.x == 0 && blockIdx.x == 0) *p.sb_probe = sb;
        return;
    }
    if (kHooks && p.isp.img) isp_init();
    const uint32_t *small = sm + kBraidSmem / 4;
    const uint64_t t_entry = p.warp_times ? globaltimer_ns() : 0ull;
    const uint32_t lane = threadIdx.x & 31u, lane4 = lane * 4u, q = lane / QL, m = lane % QL;
    const uint32_t lbase = lane4 | (sb & 0xFFFF0000u);  // braid_imm's PRMT operand
    const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    stage_tables(sm, p);  // the host put adv_{512/G} (a128 / a256) in basis[0]
    __syncthreads();
    if (wid >= p.workers) return;
    if (p.warp_times && lane == 0) {
        p.warp_times[kStamps * wid] = t_entry;
        p.warp_times[kStamps * wid + 1] = globaltimer_ns();
    }
    const uint32_t P = p.page_size, lg = p.log2_page;
    for (uint32_t ch = 0; ch < p.n_chunks; ch++) {
        if (kHooks && p.isp.img) {
            isp_lists_free(p, g_isp, ch);
            isp_chunk_begin(ch, lane);
        }
        const uint32_t ch_end = p.merge_from && ch == p.merge_from ? p.n_chunks : ch + 1;  // see k_scan
        const uint64_t cb = p.chunk_groups[ch], n = p.chunk_groups[ch_end] - cb;
        const uint64_t g0 = cb + n * wid / p.workers, g1 = cb + n * (wid + 1) / p.workers;
        if (g0 < g1) {
            // load cursor (group gl_g, block lb) runs one block ahead of the process cursor
            uint32_t la = alloc_of_group(p.allocs, p.n_allocs, g0, lane);
            AllocView lal = load_alloc(p.allocs + la, P);
            uint64_t lgi = g0 - __ldg(&p.allocs[la].grp0), lgg = g0;
            GroupLane<G> lgl = group_lane<G>(lal, lgi, P, lg, q, m);
            uint32_t lb = 0;
            uint32_t pa = la;
            AllocView pal = lal;
            GroupLane<G> pgl = lgl;
            const uint64_t ngr = g1 - g0;
            uint64_t done = 0;  // groups finalized
            auto load_block = [&](uint4 (&w)[U]) {
                if (lb == p.grp_pf_block && p.prefetch != 0u && lane == 0u && lgg + 1 < g1 &&
                    lgi + 1 < (lal.n_pages + G - 1) / G) {  // the next group of this allocation
                    const uint64_t nx = lal.base + ((lgi + 1) * G << lg);
                    const uint64_t e = min(nx + (uint64_t)G * P, lal.base + __ldg(&p.allocs[la].bytes));
                    if (e > nx) prefetch_l2(reinterpret_cast<const void *>(nx), (uint32_t)(e - nx));
                }
#pragma unroll
                for (uint32_t u = 0; u < U; u++) {
                    const uint32_t off = (lb * U + u) * Wr;
                    w[u] = lgl.valid && off + m * 16u >= lgl.pad ? ldg_stream(lgl.ptr + off) : make_uint4(0, 0, 0, 0);
                }
                if (++lb == NB) {  // next group
                    lb = 0;
                    lgg++;
                    if (lgg < g1) {
                        if (++lgi == (lal.n_pages + G - 1) / G) {
                            la++;
                            lal = load_alloc(p.allocs + la, P);
                            lgi = 0;
                        }
                        lgl = group_lane<G>(lal, lgi, P, lg, q, m);
                    }
                }
            };
            uint32_t x[4] = {0u, 0u, 0u, 0u}, acc = 0u, pb = 0;
            auto process_block = [&](const uint4 (&w)[U]) {
                if constexpr (kImm) {
#pragma unroll
                    for (uint32_t u = 0; u < U; u++) row_step_imm<kHooks ? kGrpSbLo : kGrpSbLoPlain>(lbase, x, acc, w[u]);
                } else {
#pragma unroll
                    for (uint32_t u = 0; u < U; u++) row_step(lane4, sb, x, acc, w[u]);
                }
                if (++pb < NB) return;
                // group complete: one raw16 + tree for all G pages
                uint32_t v;
                if (p.t4rep) {
                    const uint32_t *tr = sm + kScanSmem / 4, c = lane & 7u;
                    v = apply_t4rep(tr, x[0], c);
                    v = apply_t4rep(tr, v ^ x[1], c);
                    v = apply_t4rep(tr, v ^ x[2], c);
                    v = apply_t4rep(tr, v ^ x[3], c);
                } else {
                    const uint32_t *t4 = small + kT4 * 1024u;
                    v = apply_tab(t4, x[0]);
                    v = apply_tab(t4, v ^ x[1]);
                    v = apply_tab(t4, v ^ x[2]);
                    v = apply_tab(t4, v ^ x[3]);
                }
#pragma unroll
                for (uint32_t j = 0; (1u << j) < QL; j++) {
                    const uint32_t o = __shfl_down_sync(kFull, v, 1u << j);
                    if ((m & ((2u << j) - 1u)) == 0u) v = apply_tab(small + (kA16 + j) * 1024u, v) ^ o;
                }
                const uint32_t bal = __ballot_sync(kFull, acc != 0u);
                const uint32_t nzq = QL == 32 ? bal : (bal >> (q * QL)) & ((1u << QL) - 1u);
                bool pres = false;
                uint32_t plen = 0;
                if (m == 0u && pgl.valid) {
                    const bool tail = pgl.pi == pal.n_pages - 1;
                    plen = tail ? pal.tail_len : P;
                    pres = finalize_page(p, pal.page0 + pgl.pi, tile_of_page(pal.tile0, pgl.pi, P, lg), pgl.pi == 0,
                                         plen, tail ? pal.z_tail : p.z_page, v, nzq != 0u);
                }
                if (kHooks && p.isp.img) {  // f1: the group's PRESENT pages, in lane (= page) order
                    const uint32_t bal2 = __ballot_sync(kFull, pres);
                    const uint32_t wib = threadIdx.x >> 5, par = ch & 1u, n0 = g_isp.wn[par][wib];
                    const uint32_t bytes = __reduce_add_sync(kFull, pres ? plen : 0u);
                    if (pres) {
                        const uint32_t k = n0 + __popc(bal2 & ((1u << lane) - 1u));
                        if (k < p.isp.cap) isp_list(p, par, wid)[k] = (uint32_t)(pal.page0 + pgl.pi);
                        else atomicCAS(p.isp.err, 0ull, 4ull);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        g_isp.wn[par][wib] = n0 + __popc(bal2);
                        g_isp.wagg[par][wib] += bytes;
                    }
                    __syncwarp();
                }
                x[0] = x[1] = x[2] = x[3] = 0u;
                acc = 0u;
                pb = 0;
                if (++done < ngr) {
                    const uint64_t pgi = (uint64_t)pgl.pi / G + 1;
                    if (pgi == (pal.n_pages + G - 1) / G) {
                        pa++;
                        pal = load_alloc(p.allocs + pa, P);
                        pgl = group_lane<G>(pal, 0, P, lg, q, m);
                    } else {
                        pgl = group_lane<G>(pal, pgi, P, lg, q, m);
                    }
                }
            };
            const uint64_t nblk = ngr * NB;
            uint4 wa[U], wb[U];
            load_block(wa);
            for (uint64_t bk = 0; bk < nblk; bk += 2) {
                if (bk + 1 < nblk) load_block(wb);
                process_block(wa);
                if (bk + 1 >= nblk) break;
                if (bk + 2 < nblk) load_block(wa);
                process_block(wb);
            }
        }
        if (kHooks && p.isp.img) isp_chunk_end(p, g_isp, ch, lane);  // f1: the warp's aggregate
        // every leader lane's page results visible before lane 0 publishes
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            if (atomicAdd(p.chunk_arrive + ch, 1u) == (uint32_t)p.workers - 1u) {
                atomicExch(p.chunk_arrive + ch, 0u);
                __threadfence();
                for (uint32_t c2 = ch; c2 < ch_end; c2++) atomicExch(p.chunk_done + c2, p.epoch);
            }
        }
        __syncwarp();
        if (p.warp_times && lane == 0 && ch == 0) p.warp_times[kStamps * wid + 3] = globaltimer_ns();
        if (kHooks && p.isp.img && ch >= 1) isp_write(p, g_isp, ch - 1, wid, lane);
        if (ch_end == p.n_chunks) break;
    }
    if (kHooks && p.isp.img && p.n_chunks) isp_write(p, g_isp, p.n_chunks - 1, wid, lane);
    if (p.warp_times && lane == 0) p.warp_times[kStamps * wid + 4] = globaltimer_ns();
}

// K0: page -> allocation and tile -> allocation (A1).  One CTA per allocation.
__global__ void k_build_page_table(const AllocDev *allocs, uint32_t *page_alloc, uint32_t *tile_alloc) {
    const uint32_t a = blockIdx.x;
    const uint64_t page0 = allocs[a].page0, tile0 = allocs[a].tile0;
    const uint32_t np = allocs[a].n_pages, nt = allocs[a].n_tiles;
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) page_alloc[page0 + i] = a;
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) tile_alloc[tile0 + i] = a;
}

// Warp-cooperative 16-byte-vector copy of `bytes` (multiple of 16).

// K1 leaves kFreeSMs SMs unoccupied so that K2/K4 (and the restore's K6)
// start the moment they are enqueued instead of waiting
// for the persistent scan to release an SM (measured: a pack queued behind
// two scan launches delayed its chunk's drain by ~0.5 ms).
constexpr int kFreeSMsDefault = 10;  // = pack CTAs (8) + K2 (1) + 1 spare
// GCR_FREE_SMS overrides (>= 3): pack CTAs = free - 2
static int free_sms() {
    static const int v = [] {
        const char *e = std::getenv("GCR_FREE_SMS");
        const int f = e ? std::atoi(e) : kFreeSMsDefault;
        return f < 3 ? 3 : f;
    }();
    return v;
}

// K4: gather the PRESENT bytes of the chunk's staged tiles into the staging
// slot.  The host lists the staged tiles, each with the slot offset of its
// first PRESENT byte (from K2's records), in MAPPED pinned memory: no H2D sits
// in a copy-engine queue behind the drain.  A CTA stages a batch of items in
// shared memory with coalesced PCIe reads; a warp unit is one 4 KiB slice of
// a tile (8 rows of 512 B: every load in flight at once), so the work spreads
// evenly over all warps whatever the dirty pattern.  Within a row every byte
// lies in one page (pages are >= 4 KiB and row aligned): the row's page j and
// the PRESENT bytes before it in the tile come from a lane-parallel scan of
// the tile's page classes.
constexpr int kPackThreads = 1024;
constexpr uint32_t kPackBatch = 1024;                     // items staged per CTA round
constexpr uint32_t kPackSlice = 4096, kPackSliceRows = kPackSlice >> kLog2Row;
constexpr uint32_t kSlicesPerTile = kTileBytes / kPackSlice;  // 16

__global__ void __launch_bounds__(kPackThreads) k_pack(const AllocDev *allocs, const uint32_t *tile_alloc,
                                                       const uint8_t *cls, uint64_t tb, uint32_t P, uint32_t lg,
                                                       uint8_t *slot, const StageItem *items, uint32_t n_items,
                                                       const uint32_t *scan_done, uint32_t epoch,
                                                       uint32_t *decision, uint32_t pack_ctas) {
    __shared__ StageItem si[kPackBatch];
    __shared__ uint32_t s_wide;
    // Launched wide; while the persistent scan still runs (its last chunk not
    // yet published) only the first pack_ctas CTAs work -- the SMs K1 leaves
    // free -- and the rest exit at once.  Decided when the pack RUNS (packs
    // are enqueued long before their slot frees up), ONCE per launch: the
    // first CTA to get here publishes its reading in this chunk's decision
    // word (tagged with the epoch) and every CTA uses that one -- CTAs reading
    // scan_done on their own could straddle the scan's end and split the items
    // with different grid widths (some packed twice, some never).
    if (threadIdx.x == 0) {
        uint32_t w = 1u;
        if (scan_done != nullptr) {
            const uint32_t tag = (epoch & 0x7FFFFFFFu) << 1;
            const uint32_t cur = *reinterpret_cast<volatile uint32_t *>(decision);
            if ((cur & ~1u) == tag) {
                w = cur & 1u;
            } else {
                const uint32_t mine = *reinterpret_cast<const volatile uint32_t *>(scan_done) == epoch ? 1u : 0u;
                const uint32_t prev = atomicCAS(decision, cur, tag | mine);
                w = prev == cur ? mine : (prev & 1u);  // lost the race: the winner's reading
            }
        }
        s_wide = w;
    }
    __syncthreads();
    const uint32_t G = s_wide ? gridDim.x : min(gridDim.x, pack_ctas);
    if (blockIdx.x >= G) return;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t i0 = (uint32_t)((uint64_t)n_items * blockIdx.x / G);
    const uint32_t i1 = (uint32_t)((uint64_t)n_items * (blockIdx.x + 1) / G);
    for (uint32_t b0 = i0; b0 < i1; b0 += kPackBatch) {
        const uint32_t nb = min(kPackBatch, i1 - b0);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
            const uint2 v = __ldcv(reinterpret_cast<const uint2 *>(items + b0 + i));  // host-written: never cached
            si[i] = StageItem{v.x, v.y};
        }
        __syncthreads();
        for (uint32_t u = warp; u < nb * kSlicesPerTile; u += nw) {
            const StageItem it = si[u / kSlicesPerTile];
            const uint32_t so = (u % kSlicesPerTile) * kPackSlice;  // slice offset in the tile
            const uint64_t t = tb + it.tile;
            const AllocDev *al = allocs + __ldg(tile_alloc + t);
            const uint64_t base = __ldg(&al->base), page0 = __ldg(&al->page0), lt = t - __ldg(&al->tile0);
            const uint32_t n_pages = __ldg(&al->n_pages), tail_len = __ldg(&al->tail_len);
            const uint8_t *src;
            uint8_t *dst;
            uint32_t plen, pref;  // lane j: PRESENT length of the tile's page j, PRESENT bytes before it
            uint32_t rlg = lg;    // row offset -> page-in-tile shift
            if (P <= kTileBytes) {
                const uint32_t ppt = kTileBytes >> lg;
                const uint64_t pi = lt * ppt + lane;
                plen = 0;
                if (lane < ppt && pi < n_pages && (cls[page0 + pi] & 3u) == kClsPresent)
                    plen = pi == (uint64_t)n_pages - 1 ? tail_len : P;
                uint32_t inc = plen;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(kFull, inc, d);
                    if (lane >= (uint32_t)d) inc += o;
                }
                pref = inc - plen;
                src = reinterpret_cast<const uint8_t *>(base + (lt << kLog2Tile));
                dst = slot + it.dst;
            } else {  // one 64 KiB slice of a page; the item's dst is the slice's own offset
                const uint32_t tpp = P >> kLog2Tile;
                const uint64_t pi = lt / tpp;
                const uint32_t s = (uint32_t)(lt % tpp);
                const uint32_t len = pi == (uint64_t)n_pages - 1 ? tail_len : P;
                const bool present = (cls[page0 + pi] & 3u) == kClsPresent;
                plen = present && s * kTileBytes < len ? min(len - s * kTileBytes, kTileBytes) : 0u;
                plen = __shfl_sync(kFull, plen, 0);
                pref = 0;
                src = reinterpret_cast<const uint8_t *>(base + (pi << lg) + (uint64_t)s * kTileBytes);
                dst = slot + it.dst;
                rlg = kLog2Tile;  // the slice is the tile's only "page"
            }
            uint4 v[kPackSliceRows];
            uint32_t doff[kPackSliceRows];  // slot offset of this lane's 16 B, ~0 = not PRESENT
#pragma unroll
            for (uint32_t r = 0; r < kPackSliceRows; r++) {
                const uint32_t off = so + r * kRowBytes;  // row offset in the tile
                const uint32_t j = off >> rlg;
                const uint32_t pl = __shfl_sync(kFull, plen, j), pr = __shfl_sync(kFull, pref, j);
                const uint32_t w = off - (j << rlg) + lane * 16u;  // byte offset in page j
                doff[r] = w < pl ? pr + w : ~0u;
                if (doff[r] != ~0u) v[r] = ldg_stream(src + off + lane * 16u);
            }
#pragma unroll
            for (uint32_t r = 0; r < kPackSliceRows; r++)
                if (doff[r] != ~0u) *reinterpret_cast<uint4 *>(dst + doff[r]) = v[r];
        }
    }
}

// K3 phase 1: run-start counts per block of 4096 pages.
__device__ __forceinline__ uint32_t run_starts4(const uint8_t *cls, uint64_t g0, uint64_t n, uint32_t &mask) {
    uint32_t cnt = 0;
    mask = 0;
    for (int i = 0; i < 4; i++) {
        const uint64_t g = g0 + i;
        if (g >= n) break;
        const uint8_t c = cls[g];
        const bool st = (c & kClsAllocStart) || g == 0 || ((c & 3u) != (cls[g - 1] & 3u));
        if (st) {
            cnt++;
            mask |= 1u << i;
        }
    }
    return cnt;
}

__global__ void __launch_bounds__(1024) k_pm_count(const uint8_t *cls, uint64_t n, uint32_t *blk_cnt) {
    const uint64_t g0 = (uint64_t)blockIdx.x * 4096u + threadIdx.x * 4u;
    uint32_t m;
    const uint32_t c = run_starts4(cls, g0, n, m);
    const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, c);
    __shared__ uint32_t ws[32];
    if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, ws[threadIdx.x]);
        if (threadIdx.x == 0) blk_cnt[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(1024) k_pm_scan(const uint32_t *blk_cnt, uint32_t *blk_off, uint64_t nblk,
                                                  unsigned long long *n_entries) {
    const uint64_t per = (nblk + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = per * threadIdx.x, hi = min(nblk, lo + per);
    unsigned long long s = 0;
    for (uint64_t b = lo; b < hi; b++) s += blk_cnt[b];
    unsigned long long total;
    unsigned long long off = block_exclusive_scan(s, &total);
    for (uint64_t b = lo; b < hi; b++) {
        blk_off[b] = (uint32_t)off;
        off += blk_cnt[b];
    }
    if (threadIdx.x == 0) {
        *reinterpret_cast<volatile unsigned long long *>(n_entries) = total;  // mapped pinned
        __threadfence_system();
    }
}

__global__ void __launch_bounds__(1024) k_pm_starts(const uint8_t *cls, uint64_t n, const uint32_t *blk_off,
                                                    uint32_t *run_start) {
    const uint64_t g0 = (uint64_t)blockIdx.x * 4096u + threadIdx.x * 4u;
    uint32_t m;
    const uint32_t c = run_starts4(cls, g0, n, m);
    unsigned long long tot;
    uint32_t e = blk_off[blockIdx.x] + (uint32_t)block_exclusive_scan(c, &tot);
    for (int i = 0; i < 4; i++)
        if (m & (1u << i)) run_start[e++] = (uint32_t)(g0 + i);
}

struct PmEntry {
    unsigned long long vaddr;
    uint32_t nr_pages, flags;
};

__global__ void k_pm_entries(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls,
                             uint64_t n, uint32_t lg, const uint32_t *run_start, uint64_t ne, PmEntry *out) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = run_start[e];
        const uint64_t gn = e + 1 < ne ? run_start[e + 1] : n;
        const uint32_t a = page_alloc[g];
        const uint64_t va = allocs[a].base + ((g - allocs[a].page0) << lg);
        const uint32_t c = cls[g] & 3u;
        const uint32_t fl = c == kClsZero ? (1u << 3) : c == kClsParent ? (1u << 0) : (1u << 2);
        out[e] = PmEntry{va, (uint32_t)(gn - g), fl};
    }
}

// ---- TMA bulk stores (cp.async.bulk shared -> global: SASS UBLKCP) ---------
// Driven by one thread, completion tracked by bulk groups.  Every size and
// address is a multiple of 16 (R-2).
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// K6: staged image pieces -> allocation pages.  Descriptors are at most
// kScatterDescMax (1 MiB: the restore planner's piece size), so work piece u
// of a launch is the 64 KiB piece u mod 16 of descriptor u / 16 (pieces past a
// short descriptor's end are empty): CTAs grid-stride over pieces, not
// descriptors, so a 64 MiB group (64 descriptors) still spreads over every SM.
// 256 threads x 4 x 16 B per step, loads before stores.  (One CTA per
// descriptor left a 64 MiB group on 64 CTAs: 0.25 TB/s.  A TMA ring -- one
// issuing thread per CTA, bulk load -> mbarrier -> bulk store -- measured
// 0.41-0.47 TB/s: profiles/r2m_bench_staged.json, r2n_bench_staged.json.)
constexpr uint32_t kTmaStage = 16384;
constexpr uint64_t kScatterDescMax = 1ull << 20, kScatterPiece = 65536;
constexpr uint64_t kPiecesPerDesc = kScatterDescMax / kScatterPiece;

__global__ void __launch_bounds__(256) k_scatter(const ScatterDesc *desc, uint64_t n, const uint8_t *slot) {
    const uint64_t total = n * kPiecesPerDesc;
    for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
        const ScatterDesc dd = desc[u / kPiecesPerDesc];
        const uint64_t p0 = (u % kPiecesPerDesc) * kScatterPiece;
        if (p0 >= dd.bytes) continue;
        const uint64_t by = min(dd.bytes - p0, kScatterPiece);
        const uint8_t *src = slot + dd.src_off + p0;
        uint8_t *d = reinterpret_cast<uint8_t *>(dd.dst) + p0;
        constexpr int U = 4;
        uint64_t off = (uint64_t)threadIdx.x * 16u;
        const uint32_t stride = blockDim.x * 16u;
        for (; off + (U - 1) * stride < by; off += U * stride) {
            uint4 v[U];
#pragma unroll
            for (int w = 0; w < U; w++) v[w] = ldg_stream(src + off + w * stride);
#pragma unroll
            for (int w = 0; w < U; w++) *reinterpret_cast<uint4 *>(d + off + w * stride) = v[w];
        }
        for (; off < by; off += stride) *reinterpret_cast<uint4 *>(d + off) = ldg_stream(src + off);
    }
}

// K7: zero fill of ZERO runs: bulk stores from one zeroed 32 KiB smem buffer.
__global__ void __launch_bounds__(128) k_zero_fill(const ZeroDesc *desc, uint64_t n) {
    __shared__ __align__(128) uint4 zero[2 * kTmaStage / 16];
    for (uint32_t i = threadIdx.x; i < 2 * kTmaStage / 16; i += blockDim.x) zero[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy zeros visible to the bulk copies
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t groups = 0;
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        uint8_t *d = reinterpret_cast<uint8_t *>(desc[i].dst);
        const uint64_t by = desc[i].bytes;
        for (uint64_t off = 0; off < by; off += 2 * kTmaStage) {
            bulk_store(d + off, zero, (uint32_t)(by - off < 2 * kTmaStage ? by - off : 2 * kTmaStage));
            if (++groups % 8 == 0) bulk_commit();
        }
    }
    bulk_commit();
    bulk_wait_all();
}

// ---- TMA bulk-copy ring (K4 pack and K6 scatter) ---------------------------
// One issuing lane per warp streams (src, dst, len <= kTStg) pieces through a
// ring of kTStages shared-memory stages: cp.async.bulk global -> shared
// (mbarrier complete_tx), then cp.async.bulk shared -> global (bulk_group).
// A stage is reloaded only once the store that read it has finished reading
// (cp.async.bulk.wait_group.read): at most kTStages - 1 loads and the stores
// behind them in flight per warp.  3 warps x 4 x 16 KiB = 192 KiB per CTA,
// one CTA per SM.  Measured on 64 KiB pieces (tools/tma_copy, r2v): 6.10-6.17
// TB/s of copy (read + write) against 5.88-5.98 for the 16-B vector copy and
// 6.62 for a contiguous cudaMemcpyAsync D2D.
constexpr uint32_t kTStg = 16384, kTStages = 4, kTWarps = 3;
constexpr uint32_t kTSmem = kTWarps * kTStages * kTStg + kTWarps * kTStages * 8 + kTWarps * kTStages * 16 +
                            kTWarps * 32 * 24;

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra MW_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

struct TRing {  // lane 0 of a warp only
    uint8_t *buf;
    uint64_t *bar;
    unsigned long long *sdst;  // per stage: destination of the loaded piece
    uint32_t *slen;            // per stage: its length
    uint32_t nload, nstore;

    __device__ __forceinline__ void init(uint8_t *b, uint64_t *br, unsigned long long *sd, uint32_t *sl) {
        buf = b;
        bar = br;
        sdst = sd;
        slen = sl;
        nload = nstore = 0;
        for (uint32_t s = 0; s < kTStages; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __device__ __forceinline__ void pop() {  // oldest loaded piece -> its destination
        const uint32_t s = nstore % kTStages;
        mbar_wait(&bar[s], (nstore / kTStages) & 1u);
        bulk_store(reinterpret_cast<void *>(sdst[s]), buf + s * kTStg, slen[s]);
        bulk_commit();
        nstore++;
    }
    __device__ __forceinline__ void push(const uint8_t *src, uint8_t *dst, uint32_t len) {
        while (nload - nstore >= kTStages - 1) pop();
        const uint32_t s = nload % kTStages;
        // the last store out of stage s is store nload - kTStages; >= 1 store was
        // committed after it (nstore >= nload - kTStages + 2), so read<1> covers it
        if (nload >= kTStages) bulk_wait_read<1>();
        sdst[s] = reinterpret_cast<unsigned long long>(dst);
        slen[s] = len;
        mbar_expect_tx(&bar[s], len);
        bulk_load(buf + s * kTStg, src, len, &bar[s]);
        nload++;
    }
    __device__ __forceinline__ void push_run(const uint8_t *src, uint8_t *dst, uint64_t len) {
        for (uint64_t o = 0; o < len; o += kTStg) push(src + o, dst + o, (uint32_t)(len - o < kTStg ? len - o : (uint64_t)kTStg));
    }
    __device__ __forceinline__ void drain() {
        while (nstore < nload) pop();
        bulk_wait_all();  // every store performed before the kernel ends (the D2H / verify read them next)
    }
};

// Per-warp pieces of the CTA's shared memory: stages, barriers, stage metadata, item table.
struct TWarpSmem {
    uint8_t *buf;
    uint64_t *bar;
    unsigned long long *sdst;
    uint32_t *slen;
    unsigned long long *item;  // 32 x 3 u64 per warp
};
__device__ __forceinline__ TWarpSmem twarp_smem(uint8_t *sm, uint32_t w) {
    TWarpSmem t;
    t.buf = sm + (size_t)w * kTStages * kTStg;
    uint8_t *p = sm + (size_t)kTWarps * kTStages * kTStg;
    t.bar = reinterpret_cast<uint64_t *>(p) + w * kTStages;
    p += kTWarps * kTStages * 8;
    t.sdst = reinterpret_cast<unsigned long long *>(p) + w * kTStages;
    p += kTWarps * kTStages * 8;
    t.slen = reinterpret_cast<uint32_t *>(p) + w * kTStages * 2;
    p += kTWarps * kTStages * 8;
    t.item = reinterpret_cast<unsigned long long *>(p) + w * 32 * 3;
    return t;
}

// K4 (TMA): the same items and image layout as k_pack.  Each lane of a
// working warp describes one item (interleaved over the warps) as
// (source base, destination base, PRESENT-unit mask | unit size | short last
// unit) in shared memory, then lane 0 streams the PRESENT units of the
// warp's 32 items -- maximal runs of consecutive units, each run contiguous in
// the allocation and at its image offset in the slot -- through the TMA ring.
// A unit is a page (P <= 64 KiB) or the item's 64 KiB slice of a page (P > 64
// KiB).  (A first version gave each warp 32 CONSECUTIVE items: a 1 %-dirty
// chunk's ~160 items then ran on 6 warps, 56 GB/s; r2x.)
__global__ void __launch_bounds__(kTWarps * 32, 1) k_pack_tma(const AllocDev *allocs, const uint32_t *tile_alloc,
                                                             const uint8_t *cls, uint64_t tb, uint32_t P, uint32_t lg,
                                                             uint8_t *slot, const StageItem *items, uint32_t n_items,
                                                             const uint32_t *scan_done, uint32_t epoch,
                                                             uint32_t *decision, uint32_t pack_ctas) {
    extern __shared__ __align__(128) uint8_t tsm[];
    __shared__ uint32_t s_wide;
    if (threadIdx.x == 0) {  // the launch's one width decision, as in k_pack
        uint32_t wd = 1u;
        if (scan_done != nullptr) {
            const uint32_t tag = (epoch & 0x7FFFFFFFu) << 1;
            const uint32_t cur = *reinterpret_cast<volatile uint32_t *>(decision);
            if ((cur & ~1u) == tag) {
                wd = cur & 1u;
            } else {
                const uint32_t mine = *reinterpret_cast<const volatile uint32_t *>(scan_done) == epoch ? 1u : 0u;
                const uint32_t prev = atomicCAS(decision, cur, tag | mine);
                wd = prev == cur ? mine : (prev & 1u);
            }
        }
        s_wide = wd;
    }
    __syncthreads();
    const uint32_t G = s_wide ? gridDim.x : min(gridDim.x, pack_ctas);
    if (blockIdx.x >= G) return;
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const TWarpSmem ws = twarp_smem(tsm, w);
    TRing ring;
    if (lane == 0) ring.init(ws.buf, ws.bar, ws.sdst, ws.slen);
    const uint64_t W = (uint64_t)G * kTWarps, me = (uint64_t)blockIdx.x * kTWarps + w;
    // lane i of warp me takes item (k * 32 + i) * W + me: a chunk's few items
    // (1 % dirty: ~160) still spread over every working warp
    for (uint64_t k = 0; me + k * 32 * W < n_items; k++) {
        const uint64_t i = (k * 32 + lane) * W + me;
        // desc: PRESENT-unit mask (bits 0-15) | log2 unit (16-23) | index of a short
        // last unit (24-31, 0xFF: none) | its length (32-63)
        unsigned long long src = 0, dst = 0, desc = 0xFFull << 24;
        if (i < n_items) {
            const uint2 v = __ldcv(reinterpret_cast<const uint2 *>(items + i));  // host-written: never cached
            const uint64_t t = tb + v.x;
            const AllocDev *al = allocs + __ldg(tile_alloc + t);
            const uint64_t base = __ldg(&al->base), page0 = __ldg(&al->page0), lt = t - __ldg(&al->tile0);
            const uint32_t n_pages = __ldg(&al->n_pages), tail_len = __ldg(&al->tail_len);
            dst = reinterpret_cast<unsigned long long>(slot) + v.y;
            if (P <= kTileBytes) {
                const uint32_t ppt = kTileBytes >> lg;
                const uint64_t pi0 = lt * ppt;
                uint32_t mask = 0;
                for (uint32_t j = 0; j < ppt && pi0 + j < n_pages; j++)
                    if ((cls[page0 + pi0 + j] & 3u) == kClsPresent) mask |= 1u << j;
                src = base + (lt << kLog2Tile);
                desc = mask | (unsigned long long)lg << 16;
                if (pi0 + ppt >= n_pages)  // the tile holds the allocation's last page
                    desc |= (unsigned long long)(n_pages - 1 - pi0) << 24 | (unsigned long long)tail_len << 32;
                else
                    desc |= 0xFFull << 24;
            } else {
                const uint32_t tpp = P >> kLog2Tile;
                const uint64_t pi = lt / tpp;
                const uint32_t s = (uint32_t)(lt % tpp);
                const uint32_t len = pi == (uint64_t)n_pages - 1 ? tail_len : P;
                const bool present = (cls[page0 + pi] & 3u) == kClsPresent && s * kTileBytes < len;
                src = base + (pi << lg) + (uint64_t)s * kTileBytes;
                desc = (present ? 1ull : 0ull) | (unsigned long long)kLog2Tile << 16 |
                       (unsigned long long)(present ? min(len - s * kTileBytes, kTileBytes) : 0u) << 32;
            }
        }
        ws.item[lane * 3] = src;
        ws.item[lane * 3 + 1] = dst;
        ws.item[lane * 3 + 2] = desc;
        __syncwarp();
        if (lane == 0) {
            for (uint32_t q = 0; q < 32; q++) {
                const uint64_t s0 = ws.item[q * 3], d = ws.item[q * 3 + 2];
                uint8_t *dp = reinterpret_cast<uint8_t *>(ws.item[q * 3 + 1]);
                uint32_t mask = (uint32_t)d & 0xFFFFu;
                const uint32_t ulg = (uint32_t)(d >> 16) & 0xFFu, jt = (uint32_t)(d >> 24) & 0xFFu;
                const uint32_t short_len = (uint32_t)(d >> 32);
                while (mask) {  // maximal runs of consecutive PRESENT units: contiguous in memory and in the image
                    const uint32_t j = __ffs(mask) - 1u;
                    const uint32_t r = __ffs(~(mask >> j)) - 1u;  // mask < 2^16: a zero bit above the run
                    uint64_t len = (uint64_t)r << ulg;
                    if (jt == j + r - 1u) len -= (1ull << ulg) - short_len;  // ends on the short last unit
                    ring.push_run(reinterpret_cast<const uint8_t *>(s0 + ((uint64_t)j << ulg)), dp, len);
                    dp += len;
                    mask &= ~(((1u << r) - 1u) << j);
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0) ring.drain();
}

// K6 (TMA): staged image pieces -> allocation pages.  Piece u of the launch is
// the kTStg-sized piece u mod M of descriptor u / M (M = kScatterDescMax /
// kTStg; pieces past a short descriptor's end are empty).  Lane i of warp me
// describes pieces (k * 32 + i) * W + me (W warps in the grid), so adjacent
// warps take adjacent pieces and a 64 MiB group spreads over every SM; lane 0
// streams the non-empty ones through the TMA ring.
constexpr uint64_t kTPiecesPerDesc = kScatterDescMax / kTStg;

__global__ void __launch_bounds__(kTWarps * 32, 1) k_scatter_tma(const ScatterDesc *desc, uint64_t n,
                                                                const uint8_t *slot) {
    extern __shared__ __align__(128) uint8_t tsm[];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const TWarpSmem ws = twarp_smem(tsm, w);
    TRing ring;
    if (lane == 0) ring.init(ws.buf, ws.bar, ws.sdst, ws.slen);
    const uint64_t W = (uint64_t)gridDim.x * kTWarps, me = (uint64_t)blockIdx.x * kTWarps + w;
    const uint64_t total = n * kTPiecesPerDesc;
    for (uint64_t k = 0; me + k * 32 * W < total; k++) {
        const uint64_t u = (k * 32 + lane) * W + me;
        unsigned long long src = 0, dst = 0, len = 0;
        if (u < total) {
            const ScatterDesc *dd = desc + u / kTPiecesPerDesc;
            const uint64_t p0 = (u % kTPiecesPerDesc) * kTStg, by = __ldg(&dd->bytes);
            if (p0 < by) {
                src = reinterpret_cast<unsigned long long>(slot) + __ldg(&dd->src_off) + p0;
                dst = __ldg(&dd->dst) + p0;
                len = by - p0 < kTStg ? by - p0 : (uint64_t)kTStg;
            }
        }
        ws.item[lane * 3] = src;
        ws.item[lane * 3 + 1] = dst;
        ws.item[lane * 3 + 2] = len;
        __syncwarp();
        if (lane == 0)
            for (uint32_t j = 0; j < 32; j++)
                if (ws.item[j * 3 + 2])
                    ring.push(reinterpret_cast<const uint8_t *>(ws.item[j * 3]),
                              reinterpret_cast<uint8_t *>(ws.item[j * 3 + 1]), (uint32_t)ws.item[j * 3 + 2]);
        __syncwarp();
    }
    if (lane == 0) ring.drain();
}

}  // namespace

size_t scan_smem_bytes() { return kScanSmem; }
uint64_t scan_warps_per_cta() { return kScanThreads / 32; }

static int launched(int n) { return cudaPeekAtLastError() == cudaSuccess ? n : -1; }

int launch_build_page_table(const AllocDev *allocs, uint32_t n_allocs, uint32_t *page_alloc,
                            uint32_t *tile_alloc, uint32_t, uint32_t, cudaStream_t st) {
    k_build_page_table<<<n_allocs, 256, 0, st>>>(allocs, page_alloc, tile_alloc);
    return launched(1);
}


// SMs K1 leaves free: an incremental checkpoint (scan about as long as the
// drain) keeps K2 + 8 pack CTAs running beside it; a full checkpoint (drain
// ~100x the scan) keeps only K2's SM, so the scan runs ~7 % faster and the
// packs simply queue behind it (they start when it ends, wide); the verify
// takes every SM.
int scan_free_sms(bool incremental) { return incremental ? free_sms() : 1; }

uint64_t scan_workers(int n_sms, int free) {
    return (uint64_t)(free > 0 && n_sms > 4 * free ? n_sms - free : n_sms) * (kScanThreads / 32);
}

// K1 keeps each warp's stream requested into L2 this many bytes ahead of its
// register loads (cp.async.bulk.prefetch.L2: no registers, no shared memory),
// so the ~50 KiB of register double buffers per SM only have to cover L2
// latency, not HBM latency.  GCR_SCAN_PREFETCH overrides (0 = off).
// K1g requests the next group (16 KiB) into L2 when it loads block
// GCR_GRP_PF_BLOCK (default 4, i.e. ~8 KiB ahead) of the current one.  At
// block 0 (16 KiB ahead) 4-9 % of the prefetched lines were evicted before use
// and re-read from DRAM (ncu: 1.56-1.62 GB read for 1.49 GB); at block 4 the
// reads are 1.0010x the algorithmic bytes (profiles/r1n_grp_prefetch.jsonl).
// K1g: replicate t4 8x for the per-group raw16 (GCR_GRP_T4REP=1).  Off by
// default: same-box A/B at 4 KiB pages (profiles/r2l_t4rep_ab.jsonl) showed no
// gain -- ncu: bank conflicts 3.95 M -> 3.63 M of 54 M shared wavefronts; the
// 32 KiB it takes comes out of L1.
bool grp_t4rep() {
    const char *e = std::getenv("GCR_GRP_T4REP");  // read per checkpoint (A/B in one process)
    return e && e[0] == '1';
}

uint32_t grp_prefetch_block() {
    static const uint32_t v = [] {
        const char *e = std::getenv("GCR_GRP_PF_BLOCK");
        return e ? (uint32_t)std::strtoul(e, nullptr, 0) % 8u : 4u;
    }();
    return v;
}

uint32_t scan_prefetch_bytes() {
    static const uint32_t v = [] {
        const char *e = std::getenv("GCR_SCAN_PREFETCH");
        return e ? (uint32_t)std::strtoul(e, nullptr, 0) & ~15u : kScanPrefetchDefault;
    }();
    return v;
}

// GCR_TMA_COPY (read per launch; tests flip it): unset / 1 = K6 scatter
// through the TMA ring, K4 pack as the 16-B vector copy (default); 2 = both
// through the TMA ring; 0 = both vector copies.  K4 stays a vector copy by
// default: on C4 1 % the TMA pack made the step 0.1-0.4 ms SLOWER (same box,
// alternating, r2x / r2y: 9.39-9.76 vs 9.28-9.37 ms, drain 47.7-49.7 vs
// 49.8-50.2 GB/s) and its wide launch measured 387 vs 361 us per 1 GiB
// fully staged chunk in ncu; the TMA scatter is 3-4 % faster than the vector
// one (1.13-1.14 vs 1.17 ms per all-staged C2 restore).
static int tma_mode() {
    const char *e = std::getenv("GCR_TMA_COPY");
    return e ? std::atoi(e) : 1;
}

// the ring kernels' shared-memory opt-in, once per device and kernel (setting
// an attribute can serialise with work in flight)
static bool tma_attr(const void *fn) {
    static bool done[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int k = fn == reinterpret_cast<const void *>(k_pack_tma) ? 0 : 1;
    if (dev < 64 && done[dev][k]) return true;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTSmem) != cudaSuccess) return false;
    if (dev < 64) done[dev][k] = true;
    return true;
}

// K1g for 4 KiB / 8 KiB pages unless GCR_SMALL_GROUPS=0
bool scan_uses_groups(uint32_t page_size) {
    const char *e = std::getenv("GCR_SMALL_GROUPS");  // read per layout build (tests flip it)
    return !(e && e[0] == '0') && (page_size == kGroupBytes / 4 || page_size == kGroupBytes / 2);
}

static bool g_grp_imm[64] = {};        // per device: K1g immediate-base instance with the f1 hooks verified
static bool g_grp_imm_plain[64] = {};  // ... and the hook-free one

// GCR_K1_HOOKS=1: K1 / K8 always through the instance with the f1 hooks (A/B)
static bool k1_hooks_always() {
    const char *e = std::getenv("GCR_K1_HOOKS");
    return e && e[0] == '1';
}  // per device: K1g's immediate-base variant verified by scan_probe()

static int scan_attrs() {
    const int big = (int)(kScanSmem + kT4RepBytes);
    if (cudaFuncSetAttribute(k_scan<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<4, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<4, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<4, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<2, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess ||
        cudaFuncSetAttribute(k_scan_grp<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big) != cudaSuccess)
        return -1;
    return 0;
}

// GCR_GRP_IMM=0 forces the IADD variant (A/B knob).
int scan_probe() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return -1;
    const char *e = std::getenv("GCR_GRP_IMM");
    if (scan_attrs() != 0) return -1;
    uint32_t *d = nullptr, h[4] = {~0u, ~0u, ~0u, ~0u};
    if (cudaMalloc(&d, 16) != cudaSuccess) return -1;
    ScanParams p{};
    for (int v = 0; v < 4; v++) {
        p.sb_probe = d + v;
        if (v == 0) k_scan_grp<4, true, true><<<1, kScanThreads, kScanSmem>>>(p);
        else if (v == 1) k_scan_grp<2, true, true><<<1, kScanThreads, kScanSmem>>>(p);
        else if (v == 2) k_scan_grp<4, true, false><<<1, kScanThreads, kScanSmem>>>(p);
        else k_scan_grp<2, true, false><<<1, kScanThreads, kScanSmem>>>(p);
    }
    const bool ok = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    if (!ok) return -1;
    const bool allow = !(e && e[0] == '0');
    g_grp_imm[dev] = allow && (h[0] & 0xFFFFu) == kGrpSbLo && (h[1] & 0xFFFFu) == kGrpSbLo;
    g_grp_imm_plain[dev] = allow && (h[2] & 0xFFFFu) == kGrpSbLoPlain && (h[3] & 0xFFFFu) == kGrpSbLoPlain;
    if (std::getenv("GCR_TRACE"))
        std::fprintf(stderr,
                     "{\"gcr_scan_probe\": {\"sb_hooks\": [%u, %u], \"sb_plain\": [%u, %u], \"expected_lo\": [%u, %u], "
                     "\"k1g_imm\": [%d, %d]}}\n",
                     h[0], h[1], h[2], h[3], kGrpSbLo, kGrpSbLoPlain, (int)g_grp_imm[dev], (int)g_grp_imm_plain[dev]);
    return 0;
}

bool scan_grp_imm() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 64 && (g_grp_imm[dev] || g_grp_imm_plain[dev]);
}

int launch_scan(const ScanParams &p, int /*n_sms: the grid comes from p.workers*/, cudaStream_t st) {
    // once per device: setting a function attribute can serialise with work in
    // flight, which would leave the GPU idle between pipelined launches
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        if (scan_attrs() != 0) return -1;
        attr_done[dev] = true;
    }
    if (p.n_chunks == 0) return 0;
    const uint64_t wpb = kScanThreads / 32;
    const uint64_t grid = (p.workers + wpb - 1) / wpb;
    // K1g instance: hook-free immediate base unless f1 is on (or GCR_K1_HOOKS=1),
    // else the hooked immediate base, else (a probe mismatched) the IADD one
    const bool hooks = p.isp.img != nullptr || k1_hooks_always();
    const int v = dev >= 64 ? 2 : (!hooks && g_grp_imm_plain[dev]) ? 0 : g_grp_imm[dev] ? 1 : 2;
    const size_t gsm = kScanSmem + (p.t4rep ? kT4RepBytes : 0u);
    if (p.chunk_groups != nullptr && p.page_size == kGroupBytes / 4) {
        if (v == 0) k_scan_grp<4, true, false><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
        else if (v == 1) k_scan_grp<4, true, true><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
        else k_scan_grp<4, false, true><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
    } else if (p.chunk_groups != nullptr && p.page_size == kGroupBytes / 2) {
        if (v == 0) k_scan_grp<2, true, false><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
        else if (v == 1) k_scan_grp<2, true, true><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
        else k_scan_grp<2, false, true><<<(unsigned)grid, kScanThreads, gsm, st>>>(p);
    } else if (p.isp.img != nullptr || p.mode == kScanVerify || p.page_size > kTileBytes || k1_hooks_always()) {
        // The hook-free instance wins only for scans at <= 64 KiB pages
        // (profiles/r2zr_*: incremental 5.35 -> 5.51, full +1 %).  The verify
        // (K8) measured ~1 % faster through the hooked instance (5.24-5.25 vs
        // 5.18-5.20 TB/s on C2) and so did scans of > 64 KiB pages, where
        // every warp range ends in a cut-page fold (C5 16 GiB at 2 MiB: 6.01-6.03
        // vs 5.49-5.50, profiles/r2zv_*) -- code placement, not work: the hooks
        // are inactive there (p.isp.img is null).
        k_scan<true><<<(unsigned)grid, kScanThreads, kScanSmem, st>>>(p);
    } else {
        k_scan<false><<<(unsigned)grid, kScanThreads, kScanSmem, st>>>(p);
    }
    return launched(1);
}

int launch_tile_scan(TileInfo *tile_info, uint64_t tb, uint64_t te, const uint32_t *chunk_done, uint32_t chunk,
                     uint32_t epoch, TileRec *host_rec, unsigned long long *rec_count, ChunkTotals *totals_host,
                     unsigned long long *isp_base, uint32_t *isp_ready, cudaStream_t st) {
    const size_t smem = (size_t)(te - tb) * 4;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {  // up to 2 GiB chunks: 32768 tiles = 128 KiB
        if (cudaFuncSetAttribute(k_tile_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4) != cudaSuccess)
            return -1;
        attr_done[dev] = true;
    }
    k_tile_scan<<<1, kTileScanThreads, smem, st>>>(tile_info, tb, te, chunk_done, chunk, epoch, host_rec, rec_count,
                                                   totals_host, isp_base, isp_ready);
    return launched(1);
}

int launch_pack(const AllocDev *allocs, const uint32_t *tile_alloc, const uint8_t *cls, uint64_t tb, uint32_t P,
                uint32_t lg, uint8_t *slot, const StageItem *items, uint32_t n_items, int n_sms, int scan_free,
                const uint32_t *scan_done, uint32_t epoch, uint32_t *decision, cudaStream_t st) {
    if (n_items == 0) return 0;
    // up to 2 CTAs of 1024 per SM; narrowed on the device while the scan runs
    uint64_t grid = ((uint64_t)n_items * kSlicesPerTile + kPackThreads / 32 - 1) / (kPackThreads / 32);
    const uint64_t cap = (uint64_t)n_sms * 2;
    if (grid > cap) grid = cap;
    // narrow while the scan runs only if it left room for K2 + >= 1 pack CTA
    if (scan_free < 3 || n_sms <= 4 * scan_free) scan_done = nullptr;
    if (tma_mode() >= 2) {  // one 192 KiB CTA per SM, 3 issuing warps
        if (!tma_attr(reinterpret_cast<const void *>(k_pack_tma))) return -1;
        uint64_t g = ((uint64_t)n_items + kTWarps - 1) / kTWarps;
        if (g > (uint64_t)n_sms) g = (uint64_t)n_sms;
        if (scan_done != nullptr && g < (uint64_t)(scan_free - 2)) g = (uint64_t)(scan_free - 2);
        k_pack_tma<<<(unsigned)g, kTWarps * 32, kTSmem, st>>>(allocs, tile_alloc, cls, tb, P, lg, slot, items, n_items,
                                                              scan_done, epoch, decision, (uint32_t)(scan_free - 2));
        return launched(1);
    }
    k_pack<<<(unsigned)grid, kPackThreads, 0, st>>>(allocs, tile_alloc, cls, tb, P, lg, slot, items, n_items,
                                                    scan_done, epoch, decision, (uint32_t)(scan_free - 2));
    return launched(1);
}

int launch_pagemap_count(const uint8_t *cls, uint64_t n, uint32_t *blk_cnt, uint32_t *blk_off,
                         unsigned long long *n_entries_dev, cudaStream_t st) {
    const uint64_t nblk = (n + 4095) / 4096;
    k_pm_count<<<(unsigned)nblk, 1024, 0, st>>>(cls, n, blk_cnt);
    k_pm_scan<<<1, 1024, 0, st>>>(blk_cnt, blk_off, nblk, n_entries_dev);
    return launched(2);
}

int launch_pagemap_write(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls, uint64_t n,
                         uint32_t lg, const uint32_t *blk_off, uint32_t *run_start, uint64_t ne,
                         void *entries_dev, cudaStream_t st) {
    const uint64_t nblk = (n + 4095) / 4096;
    k_pm_starts<<<(unsigned)nblk, 1024, 0, st>>>(cls, n, blk_off, run_start);
    uint64_t g = (ne + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g == 0) g = 1;
    k_pm_entries<<<(unsigned)g, 256, 0, st>>>(allocs, page_alloc, cls, n, lg, run_start, ne,
                                              static_cast<PmEntry *>(entries_dev));
    return launched(2);
}

int launch_scatter(const ScatterDesc *desc, uint64_t n, const uint8_t *slot, int n_sms, cudaStream_t st) {
    if (n == 0) return 0;
    if (tma_mode() >= 1) {
        if (!tma_attr(reinterpret_cast<const void *>(k_scatter_tma))) return -1;
        const uint64_t pieces = n * kTPiecesPerDesc;
        uint64_t g = (pieces + kTWarps - 1) / kTWarps;
        if (g > (uint64_t)n_sms) g = (uint64_t)n_sms;
        k_scatter_tma<<<(unsigned)g, kTWarps * 32, kTSmem, st>>>(desc, n, slot);
        return launched(1);
    }
    const uint64_t pieces = n * kPiecesPerDesc, cap = (uint64_t)n_sms * 8;
    k_scatter<<<(unsigned)(pieces < cap ? pieces : cap), 256, 0, st>>>(desc, n, slot);
    return launched(1);
}

int launch_zero_fill(const ZeroDesc *desc, uint64_t n, int n_sms, cudaStream_t st) {
    if (n == 0) return 0;
    const uint64_t g = n < (uint64_t)n_sms * 2 ? n : (uint64_t)n_sms * 2;
    k_zero_fill<<<(unsigned)g, 128, 0, st>>>(desc, n);
    return launched(1);
}

}  // namespace gcr
