// kernels.cu -- sm_100a kernels of the device-memory snapshot path
// (SURVEY.md §8(a) rows A1-A9).
//
//  K0 build_page_table   A1: page -> allocation, tile -> allocation maps
//  K1 scan               A2+A3+A4 (+A9 in verify mode): per-page CRC32C,
//                        all-zero test, dirty diff, class; tile summaries
//  K1b fold_slices       pages > 64 KiB: fold the 64 KiB slice registers
//  K2 chunk_scan         A5: chunk-local exclusive scan of PRESENT bytes (last CTA of K1)
//  K3 pagemap_*          A5: maximal runs -> CRIU-style pagemap entries
//  K4 pack               A6: stream-compaction of PRESENT pages into staging
//  K6 scatter            A8: staged image pieces -> allocation pages
//  K7 zero_fill          A8: ZERO runs
//
// CRC32C arithmetic.  raw(x) is the register after x from 0
// (GF(2)-linear); crc(x) = raw(x) ^ Z(|x|).  A group of 8 lanes streams its
// segment as 128-byte rows; lane q owns words 4q..4q+3 of every row ("braids",
// the zlib braided-CRC idea).  The braid register x_b evolves as
// x_b <- adv_128(x_b) ^ w_b per row; after the last row the 128-byte block
// Y = (x_0..x_31) satisfies raw(segment) = raw(Y).  Each lane folds its 16
// bytes of Y (raw16) and a 3-level shuffle tree combines the lanes
// (distances 16/32/64 B).  Segments combine with adv_16K / adv_32K and
// 64 KiB slices of large pages with adv_64K.  Short (tail) pages are
// processed as if front-padded with zeros to the full page, which leaves raw()
// unchanged, so every page uses the same geometry and constants.
//
// adv_128 is evaluated with four 256-entry tables held LANE-PRIVATE in shared
// memory (entry e of table k for lane l at byte (k>>1)*64K + e*256 +
// (k&1)*128 + l*4, so the bank always equals the lane: conflict-free).  The
// byte index is extracted and scaled in ONE prmt: prmt(x, l*4, 0x55k4) =
// (byte_k(x) << 8) | l*4.  Per 4 data bytes: 4 PRMT + 4 LDS + 2 LOP3.
#include <cstdio>

#include "gcr_internal.h"

namespace gcr {

namespace {

constexpr uint32_t kBraidSmem = 4u * 256u * 32u * 4u;  // 128 KiB
constexpr uint32_t kSmallTables = 6;                   // t4 a16 a32 a64 a16k a32k
constexpr uint32_t kScanSmem = kBraidSmem + kSmallTables * 4096u;
#ifndef GCR_SCAN_THREADS
#define GCR_SCAN_THREADS 640
#endif
constexpr int kScanThreads = GCR_SCAN_THREADS;
#ifndef GCR_SCAN_UNROLL
#define GCR_SCAN_UNROLL 5
#endif
constexpr int kScanUnroll = GCR_SCAN_UNROLL;

enum : uint32_t { kT4 = 0, kA16 = 1, kA32 = 2, kA64 = 3, kA16K = 4, kA32K = 5 };

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

__device__ __forceinline__ uint32_t lds_at(const char *base, uint32_t off) {
    return *reinterpret_cast<const uint32_t *>(base + off);
}

// x -> adv_128(x) through the lane-private braid tables.
__device__ __forceinline__ uint32_t braid(const char *smb, uint32_t x, uint32_t lane4) {
    const uint32_t i0 = prmt(x, lane4, 0x5504u);
    const uint32_t i1 = prmt(x, lane4, 0x5514u);
    const uint32_t i2 = prmt(x, lane4, 0x5524u);
    const uint32_t i3 = prmt(x, lane4, 0x5534u);
    return lds_at(smb, i0) ^ lds_at(smb, i1 + 128u) ^ lds_at(smb, i2 + 65536u) ^
           lds_at(smb, i3 + 65536u + 128u);
}

// v -> adv_d(v) through an unreplicated 4x256 table (used once per segment).
__device__ __forceinline__ uint32_t apply_tab(const uint32_t *tb, uint32_t v) {
    return tb[v & 255u] ^ tb[256u + ((v >> 8) & 255u)] ^ tb[512u + ((v >> 16) & 255u)] ^
           tb[768u + (v >> 24)];
}

__device__ __forceinline__ void row_step(const char *smb, uint32_t lane4, uint32_t (&x)[4],
                                         uint32_t &acc, const uint4 &w) {
    acc |= w.x | w.y | w.z | w.w;
    x[0] = braid(smb, x[0], lane4) ^ w.x;
    x[1] = braid(smb, x[1], lane4) ^ w.y;
    x[2] = braid(smb, x[2], lane4) ^ w.z;
    x[3] = braid(smb, x[3], lane4) ^ w.w;
}

// Stream rows [r0, R) of one segment.  gp is this lane's pointer for virtual
// row 0 (gp + r*128 is its 16 bytes of row r); first_ok masks lanes of row r0
// that lie in the virtual zero padding of a short page.
template <int U>
__device__ __forceinline__ void load_block(uint4 (&w)[U], const char *gp, int r, bool mask_first, bool first_ok) {
    const char *p = gp + (size_t)r * kRowBytes;
#pragma unroll
    for (int u = 0; u < U; u++)
        w[u] = (u > 0 || !mask_first || first_ok) ? ldg_stream(p + u * kRowBytes) : make_uint4(0, 0, 0, 0);
}

template <int U, bool kFirst>
__device__ __forceinline__ void proc_block(const char *smb, uint32_t lane4, uint32_t (&x)[4], uint32_t &acc,
                                           const uint4 (&w)[U]) {
#pragma unroll
    for (int u = 0; u < U; u++) {
        if (kFirst && u == 0) {  // x = 0 before the first row: adv_128(0) ^ w == w
            x[0] = w[0].x;
            x[1] = w[0].y;
            x[2] = w[0].z;
            x[3] = w[0].w;
            acc = w[0].x | w[0].y | w[0].z | w[0].w;
        } else {
            row_step(smb, lane4, x, acc, w[u]);
        }
    }
}

// Rows are consumed in blocks of U with the next block's loads in flight
// (register double buffering): the scan is bound by bytes in flight per SM.
template <int U>
__device__ __forceinline__ void seg_stream(const char *smb, uint32_t lane4, const char *gp, int r0,
                                           int R, bool first_ok, uint32_t (&x)[4], uint32_t &acc) {
    const int nblk = (R - r0) / U;
    int r = r0;
    bool started = false;
    if (nblk > 0) {
        uint4 wa[U], wb[U];
        load_block<U>(wa, gp, r, true, first_ok);
        if (nblk > 1) load_block<U>(wb, gp, r + U, false, true);
        proc_block<U, true>(smb, lane4, x, acc, wa);
        r += U;
        int b = 1;
        for (; b + 1 < nblk; b += 2) {
            load_block<U>(wa, gp, r + U, false, true);
            proc_block<U, false>(smb, lane4, x, acc, wb);
            r += U;
            if (b + 2 < nblk) load_block<U>(wb, gp, r + U, false, true);
            proc_block<U, false>(smb, lane4, x, acc, wa);
            r += U;
        }
        if (b < nblk) {
            proc_block<U, false>(smb, lane4, x, acc, wb);
            r += U;
        }
        started = true;
    }
    for (; r < R; r++) {  // rows left over by a short (padded) page
        const bool ok = started || r > r0 || first_ok;
        const uint4 v = ok ? ldg_stream(gp + (size_t)r * kRowBytes) : make_uint4(0, 0, 0, 0);
        if (!started && r == r0) {
            x[0] = v.x;
            x[1] = v.y;
            x[2] = v.z;
            x[3] = v.w;
            acc = v.x | v.y | v.z | v.w;
        } else {
            row_step(smb, lane4, x, acc, v);
        }
    }
}

// raw() of the group's 128-byte Y block; valid in the group's lane q == 0.
__device__ __forceinline__ uint32_t group_raw(const uint32_t *small, const uint32_t (&x)[4],
                                              unsigned gmask) {
    const uint32_t *t4 = small + kT4 * 1024u;
    uint32_t v = apply_tab(t4, x[0]);
    v = apply_tab(t4, v ^ x[1]);
    v = apply_tab(t4, v ^ x[2]);
    v = apply_tab(t4, v ^ x[3]);
    uint32_t o = __shfl_down_sync(gmask, v, 1, 8);
    v = apply_tab(small + kA16 * 1024u, v) ^ o;
    o = __shfl_down_sync(gmask, v, 2, 8);
    v = apply_tab(small + kA32 * 1024u, v) ^ o;
    o = __shfl_down_sync(gmask, v, 4, 8);
    v = apply_tab(small + kA64 * 1024u, v) ^ o;
    return v;
}

struct PageAcc {
    uint32_t present_bytes = 0, counts = 0;
};

// c.1 steps 3-5 for one page given its raw register and non-zero flag
// (or the A9 verify comparison).  Executed by one lane.
__device__ __forceinline__ void finalize_page(const ScanParams &p, uint64_t g, bool alloc_start,
                                              uint32_t len, uint32_t zlen, uint32_t raw, bool nz,
                                              PageAcc &acc) {
    const uint32_t d = raw ^ zlen;
    if (p.mode == kScanVerify) {
        if (d != __ldg(p.d_ref + g)) {
            atomicAdd(p.verify_count, 1ull);
            atomicMin(p.first_bad, (unsigned long long)g);
        }
        return;
    }
    uint8_t c;
    if (!nz) {
        c = kClsZero;
        acc.counts += 1u << 10;
    } else if (p.mode == kScanIncremental && __ldg(p.d_ref + g) == d) {
        c = kClsParent;
        acc.counts += 1u << 20;
    } else {
        c = kClsPresent;
        acc.counts += 1u;
        acc.present_bytes += len;
    }
    p.d_out[g] = d;
    p.cls[g] = c | (alloc_start ? kClsAllocStart : 0);
}

// Block-wide exclusive scan of one u64 per thread (blockDim.x <= 1024).
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long *total) {
    __shared__ unsigned long long warp_sums[32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x >> 5;
        unsigned long long s = lane < nw ? warp_sums[lane] : 0ull;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xFFFFFFFFu, s, d);
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

// K2 (run by the LAST CTA of the chunk's scan): chunk-local exclusive scan of
// PRESENT bytes over tiles -> tile_off, and the chunk totals, stored both to
// device memory and straight into mapped pinned host memory so the host learns
// the chunk's image size without a DMA queued behind the drain.
__device__ void chunk_scan(const TileInfo *ti, uint64_t tb, uint64_t te, uint32_t *tile_off,
                           ChunkTotals *tot_dev, ChunkTotals *tot_host) {
    const uint64_t n = te - tb;
    const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = tb + per * threadIdx.x;
    const uint64_t hi = min(te, lo + per);
    unsigned long long s = 0, np = 0, nzr = 0, npa = 0;
    for (uint64_t t = lo; t < hi; t++) {
        const uint2 v = __ldcg(reinterpret_cast<const uint2 *>(ti) + t);
        const TileInfo x{v.x, v.y};
        s += x.present_bytes;
        np += x.counts & 1023u;
        nzr += (x.counts >> 10) & 1023u;
        npa += (x.counts >> 20) & 1023u;
    }
    unsigned long long total;
    unsigned long long off = block_exclusive_scan(s, &total);
    for (uint64_t t = lo; t < hi; t++) {
        tile_off[t] = (uint32_t)off;
        off += __ldcg(reinterpret_cast<const unsigned *>(ti) + 2 * t);
    }
    unsigned long long tp, tz, tpa;
    block_exclusive_scan(np, &tp);
    block_exclusive_scan(nzr, &tz);
    block_exclusive_scan(npa, &tpa);
    if (threadIdx.x == 0) {
        const ChunkTotals T{total, tp, tz, tpa};
        *tot_dev = T;
        volatile unsigned long long *h = reinterpret_cast<volatile unsigned long long *>(tot_host);
        h[0] = T.image_bytes;
        h[1] = T.n_present;
        h[2] = T.n_zero;
        h[3] = T.n_parent;
        __threadfence_system();
    }
}

// Last-CTA-done: every CTA fences its tile_info writes, takes a ticket, and the
// CTA holding the last ticket runs chunk_scan (then re-arms the counter).
__device__ __forceinline__ void last_cta_chunk_scan(const ScanParams &p) {
    __shared__ bool am_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = atomicAdd(p.done + p.chunk_idx, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    chunk_scan(p.tile_info, p.tile_begin, p.tile_end, p.tile_off, p.totals_dev, p.totals_host);
    if (threadIdx.x == 0) p.done[p.chunk_idx] = 0u;
}

__global__ void __launch_bounds__(kScanThreads, 1) k_scan(const ScanParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    const char *smb = reinterpret_cast<const char *>(sm);
    const uint32_t *small = sm + kBraidSmem / 4;

    // Stage the tables.  Each thread loads a few table words once (all loads
    // issued before any store) and writes the braid words to all 32 lane-private
    // replicas: word (k>>1)*16384 + e*64 + (k&1)*32 + l.
    {
        const uint32_t *gb = &p.tables->braid[0][0];
        const uint32_t *gs = &p.tables->t4[0][0];  // t4..a32k are contiguous
        constexpr uint32_t kPer = (1024u + kScanThreads - 1) / kScanThreads;
        constexpr uint32_t kPerS = (kSmallTables * 1024u + kScanThreads - 1) / kScanThreads;
        uint32_t bv[kPer], sv[kPerS];
#pragma unroll
        for (uint32_t j = 0; j < kPer; j++) {
            const uint32_t ke = threadIdx.x + j * kScanThreads;
            bv[j] = ke < 1024u ? __ldg(gb + ke) : 0u;
        }
#pragma unroll
        for (uint32_t j = 0; j < kPerS; j++) {
            const uint32_t i = threadIdx.x + j * kScanThreads;
            sv[j] = i < kSmallTables * 1024u ? __ldg(gs + i) : 0u;
        }
#pragma unroll
        for (uint32_t j = 0; j < kPer; j++) {
            const uint32_t ke = threadIdx.x + j * kScanThreads;
            if (ke < 1024u) {
                const uint32_t k = ke >> 8, e = ke & 255u;
                uint4 *dst = reinterpret_cast<uint4 *>(sm + (k >> 1) * 16384u + e * 64u + (k & 1u) * 32u);
                const uint4 v4 = make_uint4(bv[j], bv[j], bv[j], bv[j]);
#pragma unroll
                for (int l = 0; l < 8; l++) dst[l] = v4;
            }
        }
        uint32_t *ss = sm + kBraidSmem / 4;
#pragma unroll
        for (uint32_t j = 0; j < kPerS; j++) {
            const uint32_t i = threadIdx.x + j * kScanThreads;
            if (i < kSmallTables * 1024u) ss[i] = sv[j];
        }
    }
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t grp = lane >> 3, q = lane & 7u;
    const uint32_t lane4 = lane * 4u;
    const unsigned gmask = 0xFFu << (8u * grp);
    const uint32_t P = p.page_size, lg = p.log2_page;
    const uint32_t seg = P < kGroupBytes ? P : kGroupBytes;
    const int R = (int)(seg / kRowBytes);
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);

    for (uint64_t t = p.tile_begin + (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < p.tile_end;
         t += nwarps) {
        const uint32_t a = __ldg(p.tile_alloc + t);
        const AllocDev *al = p.allocs + a;
        const uint64_t base = __ldg(&al->base), page0 = __ldg(&al->page0), tile0 = __ldg(&al->tile0);
        const uint32_t n_pages = __ldg(&al->n_pages), tail_len = __ldg(&al->tail_len),
                       z_tail = __ldg(&al->z_tail);
        const uint64_t lt = t - tile0;
        PageAcc pa;

        if (P <= kGroupBytes) {
            // ---- pages <= 16 KiB: each group owns 16K/P whole pages ------------
            const uint32_t ppg = kGroupBytes >> lg;          // pages per group
            const uint64_t pi0 = lt * (kTileBytes >> lg) + (uint64_t)grp * ppg;
            for (uint32_t i = 0; i < ppg; i++) {
                const uint64_t pi = pi0 + i;
                if (pi >= n_pages) break;                    // group-uniform
                const bool tail = pi == (uint64_t)n_pages - 1;
                const uint32_t len = tail ? tail_len : P;
                const uint32_t pad = P - len;
                const char *gp = reinterpret_cast<const char *>(base + (pi << lg)) - pad + q * 16u;
                const int r0 = (int)(pad >> 7);
                const bool first_ok = ((uint32_t)r0 * kRowBytes + q * 16u) >= pad;
                uint32_t x[4], acc;
                seg_stream<kScanUnroll>(smb, lane4, gp, r0, R, first_ok, x, acc);
                const uint32_t raw = group_raw(small, x, gmask);
                const bool nz = (__ballot_sync(gmask, acc != 0) & gmask) != 0;
                if (q == 0)
                    finalize_page(p, page0 + pi, pi == 0, len, tail ? z_tail : p.z_page, raw, nz, pa);
            }
            __syncwarp();
        } else {
            // ---- pages >= 32 KiB: each group streams one 16 KiB segment --------
            uint64_t pi;
            uint32_t po;
            if (P <= kTileBytes) {
                pi = lt * (kTileBytes >> lg) + ((grp * kGroupBytes) >> lg);
                po = (grp * kGroupBytes) & (P - 1u);
            } else {
                const uint32_t tpp = P >> kLog2Tile;
                pi = lt / tpp;
                po = (uint32_t)(lt % tpp) * kTileBytes + grp * kGroupBytes;
            }
            uint32_t x[4] = {0u, 0u, 0u, 0u}, acc = 0u;
            const bool exists = pi < n_pages;
            const bool tail = pi == (uint64_t)n_pages - 1;
            const uint32_t len = tail ? tail_len : P;
            if (exists) {
                const uint32_t pad = P - len;
                const uint32_t ds = pad > po ? pad - po : 0u;
                if (ds < kGroupBytes) {
                    const char *gp = reinterpret_cast<const char *>(base + (pi << lg)) + po - pad + q * 16u;
                    const int r0 = (int)(ds >> 7);
                    const bool first_ok = ((uint32_t)r0 * kRowBytes + q * 16u) >= ds;
                    seg_stream<kScanUnroll>(smb, lane4, gp, r0, R, first_ok, x, acc);
                }
            }
            __syncwarp();
            const uint32_t graw = group_raw(small, x, gmask);
            const unsigned nzb = __ballot_sync(0xFFFFFFFFu, acc != 0);
            // combine groups: (g0,g1) and (g2,g3) with adv_16K
            uint32_t o = __shfl_down_sync(0xFFFFFFFFu, graw, 8);
            const uint32_t c01 = apply_tab(small + kA16K * 1024u, graw) ^ o;
            if (P == 2u * kGroupBytes) {
                // two pages per tile: lanes 0 and 16 finalize
                if ((lane & 15u) == 0 && exists) {
                    const bool nz = ((nzb >> (lane & 16u)) & 0xFFFFu) != 0;
                    finalize_page(p, page0 + pi, pi == 0, len, tail ? z_tail : p.z_page, c01, nz, pa);
                }
            } else {
                o = __shfl_down_sync(0xFFFFFFFFu, c01, 16);
                const uint32_t c = apply_tab(small + kA32K * 1024u, c01) ^ o;
                if (lane == 0 && exists) {
                    if (P == kTileBytes) {
                        finalize_page(p, page0 + pi, pi == 0, len, tail ? z_tail : p.z_page, c, nzb != 0, pa);
                    } else {
                        p.slice_raw[t] = c;
                        p.slice_nz[t] = nzb != 0;
                    }
                }
            }
        }
        if (p.mode != kScanVerify && P <= kTileBytes) {
            const uint32_t pb = __reduce_add_sync(0xFFFFFFFFu, pa.present_bytes);
            const uint32_t cn = __reduce_add_sync(0xFFFFFFFFu, pa.counts);
            if (lane == 0) p.tile_info[t] = TileInfo{pb, cn};
        }
    }
    if (p.mode != kScanVerify && P <= kTileBytes) last_cta_chunk_scan(p);
}

// K1b: pages > 64 KiB.  One thread per tile; the thread owning slice 0 of a
// page folds the page's slices: raw = fold_s adv_64K(raw) ^ slice_s.
__global__ void __launch_bounds__(256) k_fold_slices(const ScanParams p) {
    __shared__ uint32_t a64k[1024];
    for (uint32_t i = threadIdx.x; i < 1024u; i += blockDim.x) a64k[i] = __ldg(&p.tables->a64k[0][0] + i);
    __syncthreads();
    const uint32_t tpp = p.page_size >> kLog2Tile;
    for (uint64_t t = p.tile_begin + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.tile_end;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = __ldg(p.tile_alloc + t);
        const AllocDev *al = p.allocs + a;
        const uint64_t lt = t - __ldg(&al->tile0);
        if (lt % tpp != 0) {
            if (p.mode != kScanVerify) p.tile_info[t] = TileInfo{0u, 0u};
            continue;
        }
        const uint64_t pi = lt / tpp;
        uint32_t raw = 0;
        bool nz = false;
        for (uint32_t s = 0; s < tpp; s++) {
            raw = apply_tab(a64k, raw) ^ p.slice_raw[t + s];
            nz |= p.slice_nz[t + s] != 0;
        }
        const uint32_t n_pages = __ldg(&al->n_pages);
        const bool tail = pi == (uint64_t)n_pages - 1;
        const uint32_t len = tail ? __ldg(&al->tail_len) : p.page_size;
        PageAcc pa;
        finalize_page(p, __ldg(&al->page0) + pi, pi == 0, len, tail ? __ldg(&al->z_tail) : p.z_page, raw,
                      nz, pa);
        if (p.mode != kScanVerify) p.tile_info[t] = TileInfo{pa.present_bytes, pa.counts};
    }
    if (p.mode != kScanVerify) last_cta_chunk_scan(p);
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
__device__ __forceinline__ void warp_copy(uint8_t *dst, const uint8_t *src, uint64_t bytes, uint32_t lane) {
    constexpr int U = 8;
    uint64_t off = (uint64_t)lane * 16u;
    for (; off + (U - 1) * 512u < bytes; off += U * 512u) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = ldg_stream(src + off + u * 512u);
#pragma unroll
        for (int u = 0; u < U; u++) *reinterpret_cast<uint4 *>(dst + off + u * 512u) = v[u];
    }
    for (; off < bytes; off += 512u)
        *reinterpret_cast<uint4 *>(dst + off) = ldg_stream(src + off);
}

// K4: gather PRESENT pages of the tiles [tb, te) into the staging slot.
__global__ void __launch_bounds__(256) k_pack(const AllocDev *allocs, const uint32_t *tile_alloc,
                                              const uint8_t *cls, const uint32_t *tile_off,
                                              uint64_t tb, uint64_t te, uint32_t P, uint32_t lg,
                                              uint8_t *slot) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t t = tb + (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < te;
         t += nwarps) {
        const uint32_t a = __ldg(tile_alloc + t);
        const AllocDev *al = allocs + a;
        const uint64_t base = __ldg(&al->base), page0 = __ldg(&al->page0), tile0 = __ldg(&al->tile0);
        const uint32_t n_pages = __ldg(&al->n_pages), tail_len = __ldg(&al->tail_len);
        const uint64_t lt = t - tile0;
        if (P <= kTileBytes) {
            const uint32_t ppt = kTileBytes >> lg;
            const uint64_t pi0 = lt * ppt;
            // lane j < ppt looks at page pi0 + j
            uint32_t my_len = 0;
            const uint64_t pi = pi0 + lane;
            if (lane < ppt && pi < n_pages && (cls[page0 + pi] & 3u) == kClsPresent)
                my_len = pi == (uint64_t)n_pages - 1 ? tail_len : P;
            uint32_t inc = my_len;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            const uint32_t my_off = inc - my_len;
            uint8_t *dst0 = slot + tile_off[t];
            unsigned present = __ballot_sync(0xFFFFFFFFu, my_len != 0);
            while (present) {
                // merge consecutive present pages into one contiguous copy
                const int j = __ffs(present) - 1;
                int k = j;
                while (k + 1 < 32 && ((present >> (k + 1)) & 1u)) k++;
                const uint32_t off_j = __shfl_sync(0xFFFFFFFFu, my_off, j);
                const uint32_t end_k = __shfl_sync(0xFFFFFFFFu, my_off + my_len, k);
                warp_copy(dst0 + off_j, reinterpret_cast<const uint8_t *>(base + ((pi0 + j) << lg)),
                          end_k - off_j, lane);
                present &= (k + 1 < 32) ? ~((2u << k) - 1u) : 0u;
            }
        } else {
            const uint32_t tpp = P >> kLog2Tile;
            const uint64_t pi = lt / tpp;
            const uint32_t s = (uint32_t)(lt % tpp);
            if ((cls[page0 + pi] & 3u) != kClsPresent) continue;
            const uint32_t len = pi == (uint64_t)n_pages - 1 ? tail_len : P;
            const uint32_t lo = s * kTileBytes;
            if (lo >= len) continue;
            const uint32_t hi = min(len, lo + kTileBytes);
            warp_copy(slot + tile_off[t - s] + lo, reinterpret_cast<const uint8_t *>(base + (pi << lg) + lo),
                      hi - lo, lane);
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

// K6: staged image pieces -> allocation pages.  One CTA per descriptor.
__global__ void __launch_bounds__(256) k_scatter(const ScatterDesc *desc, uint64_t n, const uint8_t *slot) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const uint64_t dst = desc[i].dst, so = desc[i].src_off, by = desc[i].bytes;
        const uint8_t *src = slot + so;
        uint8_t *d = reinterpret_cast<uint8_t *>(dst);
        constexpr int U = 4;
        uint64_t off = (uint64_t)threadIdx.x * 16u;
        const uint32_t stride = blockDim.x * 16u;
        for (; off + (U - 1) * stride < by; off += U * stride) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++) v[u] = ldg_stream(src + off + u * stride);
#pragma unroll
            for (int u = 0; u < U; u++) *reinterpret_cast<uint4 *>(d + off + u * stride) = v[u];
        }
        for (; off < by; off += stride) *reinterpret_cast<uint4 *>(d + off) = ldg_stream(src + off);
    }
}

// K7: zero fill of ZERO runs.
__global__ void __launch_bounds__(256) k_zero_fill(const ZeroDesc *desc, uint64_t n) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        uint8_t *d = reinterpret_cast<uint8_t *>(desc[i].dst);
        const uint64_t by = desc[i].bytes;
        for (uint64_t off = (uint64_t)threadIdx.x * 16u; off < by; off += blockDim.x * 16u)
            *reinterpret_cast<uint4 *>(d + off) = make_uint4(0, 0, 0, 0);
    }
}

}  // namespace

size_t scan_smem_bytes() { return kScanSmem; }

static int launched(int n) { return cudaPeekAtLastError() == cudaSuccess ? n : -1; }

int launch_build_page_table(const AllocDev *allocs, uint32_t n_allocs, uint32_t *page_alloc,
                            uint32_t *tile_alloc, uint32_t, uint32_t, cudaStream_t st) {
    k_build_page_table<<<n_allocs, 256, 0, st>>>(allocs, page_alloc, tile_alloc);
    return launched(1);
}

int launch_scan(const ScanParams &p, int n_sms, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem) !=
            cudaSuccess)
            return -1;
        attr = true;
    }
    const uint64_t tiles = p.tile_end - p.tile_begin;
    if (tiles == 0) return 0;
    const uint64_t wpb = kScanThreads / 32;
    uint64_t grid = (tiles + wpb - 1) / wpb;
    if (grid > (uint64_t)n_sms) grid = n_sms;
    k_scan<<<(unsigned)grid, kScanThreads, kScanSmem, st>>>(p);
    int n = 1;
    if (p.page_size > kTileBytes) {
        uint64_t g2 = (tiles + 255) / 256;
        if (g2 > (uint64_t)n_sms * 8) g2 = n_sms * 8;
        k_fold_slices<<<(unsigned)g2, 256, 0, st>>>(p);
        n++;
    }
    return launched(n);
}

int launch_pack(const AllocDev *allocs, const uint32_t *tile_alloc, const uint8_t *cls, const uint32_t *tile_off,
                uint64_t tb, uint64_t te, uint32_t P, uint32_t lg, uint8_t *slot, int n_sms, cudaStream_t st) {
    const uint64_t tiles = te - tb;
    if (tiles == 0) return 0;
    uint64_t grid = (tiles + 7) / 8;
    if (grid > (uint64_t)n_sms * 4) grid = n_sms * 4;
    k_pack<<<(unsigned)grid, 256, 0, st>>>(allocs, tile_alloc, cls, tile_off, tb, te, P, lg, slot);
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
    uint64_t g = n < (uint64_t)n_sms * 8 ? n : (uint64_t)n_sms * 8;
    k_scatter<<<(unsigned)g, 256, 0, st>>>(desc, n, slot);
    return launched(1);
}

int launch_zero_fill(const ZeroDesc *desc, uint64_t n, int n_sms, cudaStream_t st) {
    if (n == 0) return 0;
    uint64_t g = n < (uint64_t)n_sms * 8 ? n : (uint64_t)n_sms * 8;
    k_zero_fill<<<(unsigned)g, 256, 0, st>>>(desc, n);
    return launched(1);
}

}  // namespace gcr
