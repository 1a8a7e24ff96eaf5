// codec.cu -- sm_100a kernels of the f4 page codec ("data
// compression ... could further improve the efficiency of checkpoint/restore
// operations").  DESIGN.md reading R-19, the byte-plane
// dictionary code: a page of n = L/4 LE words is four byte planes; a plane
// with d <= 128 distinct values (and a shorter packed form) is stored as its
// ascending dictionary + ceil(log2 d)-bit ranks (LSB-first fields), else raw.
// Training state puts its exponent bits in the top byte of every fp32 / bf16
// value, so that plane has few distinct values while the mantissa planes stay
// raw.
//
//  KA  k_codec_plan     one warp per page of a chunk: byte-value presence of
//                       each plane (lane-private bitmaps in shared memory,
//                       warp-reduced), the page's stored length, its 4x256-bit
//                       presence masks (scratch for KC)
//  KB  k_codec_offsets  one CTA per sub-chunk: exclusive scan of the stored
//                       lengths (slot offsets from the sub-chunk's base), its
//                       entries of the compact stored-length table, its stored
//                       total and PRESENT count -> mapped host
//  KC  k_codec_encode   one warp per PRESENT page: header, dictionaries, packed
//                       ranks / raw planes into the staging slot
//  KD  k_codec_decode   restore: one warp per PRESENT page of a staged group,
//                       stored form in a slot -> page in its allocation
//
// Every kernel is bandwidth-light next to the host link it feeds (a page is
// read twice from HBM, written once to the slot), so the design favours
// simple, exact warp-per-page code over fusing into the scan.
#include "gcr_internal.h"

namespace gcr {

namespace {

constexpr int kCodecThreads = 256;  // 8 warps per CTA
// A page of more than kSliceValues words (128 KiB) is worked on by several
// warps, one per SLICE of kSliceValues values (32 blocks of 1024): a 2 MiB page
// has 16.  Blocks are independent once the page's dictionaries are known, so
// KC / KD slices need no coordination; KA slices OR their presence masks into
// the page's (zeroed) masks and the last one to finish computes the size.
constexpr uint32_t kSliceValues = 32u * 1024u;

__host__ __device__ __forceinline__ uint32_t slices_of(uint32_t P) {
    return P / 4u > kSliceValues ? P / 4u / kSliceValues : 1u;
}
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t pad16(uint32_t x) { return (x + 15u) & ~15u; }
__device__ __forceinline__ uint32_t ceil_log2(uint32_t d) { return d <= 1u ? 0u : 32u - __clz(d - 1u); }

// Page geometry of global page g.
struct PageGeo {
    const uint8_t *base;  // page address
    uint32_t len;         // true length
};

__device__ __forceinline__ PageGeo page_geo(const AllocDev *allocs, const uint32_t *page_alloc, uint64_t g,
                                            uint32_t P, uint32_t lg) {
    const AllocDev *al = allocs + __ldg(page_alloc + g);
    const uint64_t pi = g - __ldg(&al->page0);
    PageGeo q;
    q.base = reinterpret_cast<const uint8_t *>(__ldg(&al->base) + (pi << lg));
    q.len = pi == (uint64_t)__ldg(&al->n_pages) - 1 ? __ldg(&al->tail_len) : P;
    return q;
}

// Coded length of a page with plane dictionary sizes d[k] (R-19); modes out.
__device__ __forceinline__ uint32_t coded_len(uint32_t n, const uint32_t (&d)[4], uint32_t (&mode)[4]) {
    uint32_t C = 16;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t b = ceil_log2(d[k]);
        const uint32_t sp = pad16(d[k]) + pad16((n * b + 7u) / 8u), sr = pad16(n);
        if (d[k] <= 128u && sp < sr) {
            mode[k] = b;
            C += sp;
        } else {
            mode[k] = 8;
            C += sr;
        }
    }
    return C;
}

// Section offsets (from the page start) of the four planes.
__device__ __forceinline__ void section_offsets(uint32_t n, const uint32_t (&d)[4], const uint32_t (&mode)[4],
                                                uint32_t (&off)[4]) {
    uint32_t o = 16;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        off[k] = o;
        o += mode[k] == 8u ? pad16(n) : pad16(d[k]) + pad16((n * mode[k] + 7u) / 8u);
    }
}

// Warp: d[k] for every plane from the lane-held mask word (lane l holds word
// l&7 of plane l>>3); returns them in every lane.
__device__ __forceinline__ void plane_counts(uint32_t mword, uint32_t (&d)[4]) {
    uint32_t c = __popc(mword);
    c += __shfl_xor_sync(kFull, c, 1);
    c += __shfl_xor_sync(kFull, c, 2);
    c += __shfl_xor_sync(kFull, c, 4);
#pragma unroll
    for (int k = 0; k < 4; k++) d[k] = __shfl_sync(kFull, c, 8 * k);
}

// KA.  plan[p] = stored length of chunk-local page p (0 if not PRESENT);
// masks[32 p + w] = presence word w (plane w>>3, values 32(w&7) .. +31).
// `done` (sliced pages only) counts the finished slices of each page (zeroed
// by the host, re-zeroed by the page's last slice; KB reuses the array).
__global__ void __launch_bounds__(kCodecThreads) k_codec_plan(const AllocDev *allocs, const uint32_t *page_alloc,
                                                              const uint8_t *cls, uint64_t pb, uint32_t np,
                                                              uint32_t P, uint32_t lg, uint32_t *plan,
                                                              uint32_t *masks, uint32_t *done) {
    __shared__ uint32_t bm[kCodecThreads / 32][32 * 32];  // per warp: word (k*8+j) of lane l at [(k*8+j)*32 + l]
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    uint32_t *sm = bm[wib];
    const uint32_t S = slices_of(P);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5), items = (uint64_t)np * S;
    for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; u < items; u += nw) {
        const uint32_t p = (uint32_t)(u / S), sl = (uint32_t)(u % S);
        const uint64_t g = pb + p;
        if ((cls[g] & 3u) != kClsPresent) {
            if (lane == 0 && sl == 0) plan[p] = 0u;
            continue;
        }
        const PageGeo q = page_geo(allocs, page_alloc, g, P, lg);
        const uint32_t n = q.len >> 2;
        const uint32_t v0 = sl * kSliceValues;
        if (v0 >= n) continue;  // a short tail page has fewer slices
        const uint32_t v1 = min(n, v0 + kSliceValues);
#pragma unroll
        for (int w = 0; w < 32; w++) sm[w * 32 + lane] = 0u;
        const uint4 *src = reinterpret_cast<const uint4 *>(q.base);
        for (uint32_t i = (v0 >> 2) + lane; i < (v1 >> 2); i += 32u) {
            const uint4 v = __ldg(src + i);
            const uint32_t xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int t = 0; t < 4; t++) {
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t b = (xs[t] >> (8 * k)) & 255u;
                    uint32_t *a = sm + (k * 8 + (b >> 5)) * 32 + lane;
                    *a |= 1u << (b & 31u);
                }
            }
        }
        __syncwarp();
        // lane l ORs presence word l over all lanes (staggered: conflict-free)
        uint32_t acc = 0;
#pragma unroll 8
        for (uint32_t t = 0; t < 32; t++) acc |= sm[lane * 32 + ((t + lane) & 31u)];
        __syncwarp();
        if (S > 1) {  // sliced page: merge into the page's masks; the last slice sizes the page
            atomicOr(masks + (uint64_t)p * 32 + lane, acc);
            __threadfence();
            uint32_t last = 0;
            if (lane == 0) last = atomicAdd(done + p, 1u) == (n + kSliceValues - 1) / kSliceValues - 1;
            if (!__shfl_sync(kFull, last, 0)) continue;
            __threadfence();
            acc = __ldcg(masks + (uint64_t)p * 32 + lane);
            if (lane == 0) done[p] = 0u;
        } else {
            masks[(uint64_t)p * 32 + lane] = acc;
        }
        uint32_t d[4], mode[4];
        plane_counts(acc, d);
        const uint32_t C = coded_len(n, d, mode);
        if (lane == 0) plan[p] = C < q.len ? C : q.len;
    }
}

// Block-wide exclusive scan (one value per thread, blockDim.x <= 1024).
__device__ __forceinline__ unsigned long long block_scan(unsigned long long v, unsigned long long *total) {
    __shared__ unsigned long long ws[32];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const unsigned long long o = __shfl_up_sync(kFull, inc, s);
        if (lane >= (uint32_t)s) inc += o;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long x = lane < nwarp ? ws[lane] : 0ull;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, x, s);
            if (lane >= (uint32_t)s) x += o;
        }
        if (lane < nwarp) ws[lane] = x;
    }
    __syncthreads();
    const unsigned long long r = (warp ? ws[warp - 1] : 0ull) + inc - v;
    if (total) *total = ws[nwarp - 1];
    __syncthreads();
    return r;
}

// KB.  off[p] = chunk-local slot offset of page p's stored form; the compact
// stored-length table of the image (PRESENT pages in page order) gets this
// chunk's entries from index present_base on; the chunk's stored total is
// written to mapped host memory.
__global__ void __launch_bounds__(1024) k_codec_offsets(const uint32_t *plan, uint32_t np, uint32_t *off,
                                                        uint32_t *stored_compact, uint64_t present_base,
                                                        uint64_t slot_base, unsigned long long *total_host) {
    const uint32_t per = (np + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(np, per * threadIdx.x), hi = min(np, lo + per);
    unsigned long long s = 0, c = 0;
    for (uint32_t p = lo; p < hi; p++) {
        const uint32_t v = plan[p];
        s += v;
        c += v != 0u;
    }
    unsigned long long tot, totc;
    unsigned long long o = block_scan(s, &tot) + slot_base;
    unsigned long long k = block_scan(c, &totc);
    for (uint32_t p = lo; p < hi; p++) {
        const uint32_t v = plan[p];
        off[p] = (uint32_t)o;
        if (v) stored_compact[present_base + k++] = v;
        o += v;
    }
    if (threadIdx.x == 0) {
        reinterpret_cast<volatile unsigned long long *>(total_host)[0] = tot;
        reinterpret_cast<volatile unsigned long long *>(total_host)[1] = totc;
        __threadfence_system();
    }
}

// 32 b-bit codes -> b words, code m at bit m*b (LSB first).
template <int B>
__device__ __forceinline__ void pack_codes(const uint32_t (&c)[32], uint32_t (&w)[8]) {
#pragma unroll
    for (int j = 0; j < B; j++) w[j] = 0u;
#pragma unroll
    for (int m = 0; m < 32; m++) {
        const int bit = m * B, wi = bit >> 5, sh = bit & 31;
        w[wi] |= c[m] << sh;
        if (sh + B > 32) w[wi + 1] |= c[m] >> (32 - sh);
    }
}

template <int B>
__device__ __forceinline__ void unpack_codes(const uint32_t (&w)[8], uint32_t (&c)[32]) {
#pragma unroll
    for (int m = 0; m < 32; m++) {
        const int bit = m * B, wi = bit >> 5, sh = bit & 31;
        uint32_t v = w[wi] >> sh;
        if (sh + B > 32) v |= w[wi + 1] << (32 - sh);
        c[m] = v & ((1u << B) - 1u);
    }
}

__device__ __forceinline__ void pack_any(uint32_t b, const uint32_t (&c)[32], uint32_t (&w)[8]) {
    switch (b) {
        case 1: pack_codes<1>(c, w); break;
        case 2: pack_codes<2>(c, w); break;
        case 3: pack_codes<3>(c, w); break;
        case 4: pack_codes<4>(c, w); break;
        case 5: pack_codes<5>(c, w); break;
        case 6: pack_codes<6>(c, w); break;
        default: pack_codes<7>(c, w); break;
    }
}

__device__ __forceinline__ void unpack_any(uint32_t b, const uint32_t (&w)[8], uint32_t (&c)[32]) {
    switch (b) {
        case 1: unpack_codes<1>(w, c); break;
        case 2: unpack_codes<2>(w, c); break;
        case 3: unpack_codes<3>(w, c); break;
        case 4: unpack_codes<4>(w, c); break;
        case 5: unpack_codes<5>(w, c); break;
        case 6: unpack_codes<6>(w, c); break;
        default: unpack_codes<7>(w, c); break;
    }
}

// Warp copy of `bytes` (multiple of 16), 16-B vectors.
__device__ __forceinline__ void warp_copy16(uint8_t *dst, const uint8_t *src, uint32_t bytes, uint32_t lane) {
    for (uint32_t o = lane * 16u; o < bytes; o += 512u)
        *reinterpret_cast<uint4 *>(dst + o) = __ldg(reinterpret_cast<const uint4 *>(src + o));
}

// KC.
__global__ void __launch_bounds__(kCodecThreads) k_codec_encode(const AllocDev *allocs, const uint32_t *page_alloc,
                                                                const uint8_t *cls, uint64_t pb, uint32_t np,
                                                                uint32_t P, uint32_t lg, const uint32_t *plan,
                                                                const uint32_t *off, const uint32_t *masks,
                                                                uint8_t *slot) {
    __shared__ uint8_t lut[kCodecThreads / 32][4][256];   // rank of each byte value, per plane
    __shared__ uint8_t dict[kCodecThreads / 32][4][128];  // dictionary (ascending), per plane
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t S = slices_of(P);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5), items = (uint64_t)np * S;
    for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; u < items; u += nw) {
        const uint32_t p = (uint32_t)(u / S), sl = (uint32_t)(u % S);
        const uint64_t g = pb + p;
        if ((cls[g] & 3u) != kClsPresent) continue;
        const PageGeo q = page_geo(allocs, page_alloc, g, P, lg);
        const uint32_t stored = plan[p];
        uint8_t *dst = slot + off[p];
        const uint32_t n = q.len >> 2;
        if (sl * kSliceValues >= n) continue;
        if (stored == q.len) {  // raw page: this slice's bytes
            const uint32_t b0 = sl * kSliceValues * 4u, b1 = min(q.len, b0 + kSliceValues * 4u);
            warp_copy16(dst + b0, q.base + b0, b1 - b0, lane);
            continue;
        }
        const uint32_t mw = masks[(uint64_t)p * 32 + lane];
        uint32_t d[4], mode[4], so[4];
        plane_counts(mw, d);
        coded_len(n, d, mode);
        section_offsets(n, d, mode, so);
        // ranks: exclusive count of present values below word (l & 7) of plane l >> 3
        const uint32_t k0 = lane >> 3, j0 = lane & 7u;
        uint32_t pre = __popc(mw), x = pre;
#pragma unroll
        for (int s = 1; s < 8; s <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, x, s);
            if (j0 >= (uint32_t)s) x += o;
        }
        pre = x - pre;
        for (uint32_t t = 0; t < 32; t++)
            if (mw >> t & 1u) {
                const uint32_t r = pre + __popc(mw & ((1u << t) - 1u));
                lut[wib][k0][32 * j0 + t] = (uint8_t)r;
                if (r < 128u) dict[wib][k0][r] = (uint8_t)(32 * j0 + t);
            }
        __syncwarp();
        // header (16 B), the dictionaries of packed planes (zero-padded to 16)
        // and the code sections' tail padding: slice 0 of the page
        if (lane == 0 && sl == 0) {
            uint4 h;
            h.x = mode[0] | mode[1] << 8 | mode[2] << 16 | mode[3] << 24;
            const uint32_t dm[4] = {mode[0] < 8 ? d[0] - 1 : 0u, mode[1] < 8 ? d[1] - 1 : 0u,
                                    mode[2] < 8 ? d[2] - 1 : 0u, mode[3] < 8 ? d[3] - 1 : 0u};
            h.y = dm[0] | dm[1] << 8 | dm[2] << 16 | dm[3] << 24;
            h.z = h.w = 0u;
            *reinterpret_cast<uint4 *>(dst) = h;
        }
#pragma unroll
        for (int k = 0; k < 4 && sl == 0; k++) {
            if (mode[k] == 8u) continue;
            const uint32_t dp = pad16(d[k]);
            if (4 * lane < dp) {
                uint32_t v = 0;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const uint32_t i = 4 * lane + e;
                    v |= (i < d[k] ? (uint32_t)dict[wib][k][i] : 0u) << (8 * e);
                }
                *reinterpret_cast<uint32_t *>(dst + so[k] + 4 * lane) = v;
            }
            // zero the code section's tail padding (whole words past the codes)
            const uint32_t cw = (n * mode[k] + 31u) / 32u, cb = pad16((n * mode[k] + 7u) / 8u) / 4u;
            if (lane < cb - cw) *reinterpret_cast<uint32_t *>(dst + so[k] + dp + 4 * (cw + lane)) = 0u;
        }
        // this slice's blocks of 1024 values: lane l takes values [32 l, 32 l + 32) of a block
        const uint32_t nblk = (n + 1023u) / 1024u, bpsl = kSliceValues / 1024u;
        for (uint32_t blk = sl * bpsl; blk < min(nblk, (sl + 1) * bpsl); blk++) {
            const uint32_t i0 = blk * 1024u + 32u * lane;
            uint32_t wv[32];
            const uint4 *s4 = reinterpret_cast<const uint4 *>(q.base) + (i0 >> 2);
#pragma unroll
            for (int u = 0; u < 8; u++) {
                uint4 v = make_uint4(0, 0, 0, 0);
                if (i0 + 4 * u < n) v = __ldg(s4 + u);
                wv[4 * u] = v.x;
                wv[4 * u + 1] = v.y;
                wv[4 * u + 2] = v.z;
                wv[4 * u + 3] = v.w;
            }
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (mode[k] == 8u) {  // raw plane: byte k of the 32 words, at plane byte offset i0
                    uint32_t pk[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        // byte k of words 4u, 4u+1 (and 4u+2, 4u+3), then the four side by side
                        const uint32_t a = __byte_perm(wv[4 * u], wv[4 * u + 1], k | ((k + 4) << 4));
                        const uint32_t b2 = __byte_perm(wv[4 * u + 2], wv[4 * u + 3], k | ((k + 4) << 4));
                        pk[u] = __byte_perm(a, b2, 0x5410u);
                    }
                    const uint32_t pn = pad16(n);
                    uint8_t *o = dst + so[k] + i0;
                    if (i0 < pn) *reinterpret_cast<uint4 *>(o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    if (i0 + 16u < pn) *reinterpret_cast<uint4 *>(o + 16) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                } else if (mode[k] != 0u) {  // packed plane: lane's 32 codes -> b words
                    uint32_t cde[32], w8[8];
#pragma unroll
                    for (int m = 0; m < 32; m++)
                        cde[m] = i0 + m < n ? (uint32_t)lut[wib][k][(wv[m] >> (8 * k)) & 255u] : 0u;
                    const uint32_t b = mode[k];
                    pack_any(b, cde, w8);
                    const uint32_t cw = (n * b + 31u) / 32u;          // code words of the plane
                    uint32_t *o = reinterpret_cast<uint32_t *>(dst + so[k] + pad16(d[k])) + (blk * 32u + lane) * b;
                    const uint32_t w0 = (blk * 32u + lane) * b;
#pragma unroll
                    for (int j = 0; j < 7; j++)
                        if ((uint32_t)j < b && w0 + j < cw) o[j] = w8[j];
                }
            }
        }
        __syncwarp();
    }
}

// KD.  One warp per descriptor: stored form at slot + src_off -> the page at dst.
__global__ void __launch_bounds__(kCodecThreads) k_codec_decode(const DecodeDesc *desc, uint64_t n_desc,
                                                                const uint8_t *slot, uint32_t S) {
    __shared__ uint8_t dict[kCodecThreads / 32][4][128];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5), items = n_desc * S;
    for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; u < items; u += nw) {
        const uint64_t i = u / S;
        const uint32_t sl = (uint32_t)(u % S);
        const DecodeDesc dd = desc[i];
        uint8_t *dst = reinterpret_cast<uint8_t *>(dd.dst);
        const uint8_t *src = slot + dd.src_off;
        const uint32_t len = dd.len, stored = dd.stored, n = len >> 2;
        if (sl * kSliceValues >= n) continue;
        const uint32_t b0 = sl * kSliceValues * 4u, b1 = min(len, b0 + kSliceValues * 4u);  // this slice's bytes
        if (stored == len) {
            warp_copy16(dst + b0, src + b0, b1 - b0, lane);
            continue;
        }
        // header + validation (R-19 malformed rule: the page restores as zeros)
        const uint4 h = stored >= 16u ? __ldg(reinterpret_cast<const uint4 *>(src)) : make_uint4(0xFF, 0, 0, 0);
        uint32_t mode[4], d[4], so[4];
        bool bad = stored < 16u || h.z != 0u || h.w != 0u;
        uint32_t o = 16;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            mode[k] = (h.x >> (8 * k)) & 255u;
            const uint32_t dm1 = (h.y >> (8 * k)) & 255u;
            d[k] = dm1 + 1u;
            so[k] = o;
            if (mode[k] > 8u) bad = true;
            else if (mode[k] == 8u) {
                if (dm1) bad = true;
                o += pad16(n);
            } else {
                if (d[k] > 128u || ceil_log2(d[k]) != mode[k]) bad = true;
                o += pad16(d[k]) + pad16((n * mode[k] + 7u) / 8u);
            }
        }
        if (o != stored) bad = true;
        if (bad) {
            for (uint32_t x = b0 + lane * 16u; x < b1; x += 512u) *reinterpret_cast<uint4 *>(dst + x) = make_uint4(0, 0, 0, 0);
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (mode[k] == 8u) continue;
            for (uint32_t e = lane; e < 128u; e += 32u) dict[wib][k][e] = e < d[k] ? src[so[k] + e] : (uint8_t)0;
        }
        __syncwarp();
        const uint32_t nblk = (n + 1023u) / 1024u, bpsl = kSliceValues / 1024u;
        for (uint32_t blk = sl * bpsl; blk < min(nblk, (sl + 1) * bpsl); blk++) {
            const uint32_t i0 = blk * 1024u + 32u * lane;
            uint32_t wv[32];
#pragma unroll
            for (int m = 0; m < 32; m++) wv[m] = 0u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (mode[k] == 8u) {
                    const uint8_t *s = src + so[k] + i0;
                    const uint32_t pn = pad16(n);
                    uint4 a = make_uint4(0, 0, 0, 0), b2 = make_uint4(0, 0, 0, 0);
                    if (i0 < pn) a = __ldg(reinterpret_cast<const uint4 *>(s));
                    if (i0 + 16u < pn) b2 = __ldg(reinterpret_cast<const uint4 *>(s + 16));
                    const uint32_t pk[8] = {a.x, a.y, a.z, a.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
                    for (int m = 0; m < 32; m++) wv[m] |= ((pk[m >> 2] >> (8 * (m & 3))) & 255u) << (8 * k);
                } else {
                    uint32_t byte0 = dict[wib][k][0];
                    if (mode[k] == 0u) {
#pragma unroll
                        for (int m = 0; m < 32; m++) wv[m] |= byte0 << (8 * k);
                        continue;
                    }
                    const uint32_t b = mode[k], cw = (n * b + 31u) / 32u, w0 = (blk * 32u + lane) * b;
                    const uint32_t *cs = reinterpret_cast<const uint32_t *>(src + so[k] + pad16(d[k])) + w0;
                    uint32_t w8[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cde[32];
#pragma unroll
                    for (int j = 0; j < 7; j++)
                        if ((uint32_t)j < b && w0 + j < cw) w8[j] = __ldg(cs + j);
                    unpack_any(b, w8, cde);
#pragma unroll
                    for (int m = 0; m < 32; m++) wv[m] |= (uint32_t)dict[wib][k][cde[m] & 127u] << (8 * k);
                }
            }
            uint4 *d4 = reinterpret_cast<uint4 *>(dst) + (i0 >> 2);
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (i0 + 4 * u < n) d4[u] = make_uint4(wv[4 * u], wv[4 * u + 1], wv[4 * u + 2], wv[4 * u + 3]);
        }
        __syncwarp();
    }
}

}  // namespace

static int codec_launched(int n) { return cudaPeekAtLastError() == cudaSuccess ? n : -1; }

static unsigned codec_grid(uint64_t items, int n_sms) {
    const uint64_t per = kCodecThreads / 32;
    uint64_t g = (items + per - 1) / per;
    const uint64_t cap = (uint64_t)n_sms * 8;
    return (unsigned)(g < 1 ? 1 : g > cap ? cap : g);
}

int launch_codec_plan(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls, uint64_t page_begin,
                      uint32_t n_pages, uint32_t P, uint32_t lg, uint32_t *plan, uint32_t *masks, uint32_t *done,
                      int n_sms, cudaStream_t st) {
    if (n_pages == 0) return 0;
    const uint32_t S = slices_of(P);
    if (S > 1) {  // sliced pages merge presence masks with atomics: start from zero
        if (cudaMemsetAsync(masks, 0, 128ull * n_pages, st) != cudaSuccess ||
            cudaMemsetAsync(done, 0, 4ull * n_pages, st) != cudaSuccess)
            return -1;
    }
    k_codec_plan<<<codec_grid((uint64_t)n_pages * S, n_sms), kCodecThreads, 0, st>>>(allocs, page_alloc, cls,
                                                                                    page_begin, n_pages, P, lg, plan,
                                                                                    masks, done);
    return codec_launched(1);
}

int launch_codec_offsets(const uint32_t *plan, uint32_t n_pages, uint32_t *off, uint32_t *stored_compact,
                         uint64_t present_base, uint64_t slot_base, unsigned long long *total_host, cudaStream_t st) {
    k_codec_offsets<<<1, 1024, 0, st>>>(plan, n_pages, off, stored_compact, present_base, slot_base, total_host);
    return codec_launched(1);
}

int launch_codec_encode(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls, uint64_t page_begin,
                        uint32_t n_pages, uint32_t P, uint32_t lg, const uint32_t *plan, const uint32_t *off,
                        const uint32_t *masks, uint8_t *slot, int n_sms, cudaStream_t st) {
    if (n_pages == 0) return 0;
    k_codec_encode<<<codec_grid((uint64_t)n_pages * slices_of(P), n_sms), kCodecThreads, 0, st>>>(allocs, page_alloc, cls, page_begin,
                                                                          n_pages, P, lg, plan, off, masks, slot);
    return codec_launched(1);
}

int launch_codec_decode(const DecodeDesc *desc, uint64_t n_desc, const uint8_t *slot, uint32_t page_size, int n_sms,
                        cudaStream_t st) {
    if (n_desc == 0) return 0;
    const uint32_t S = slices_of(page_size);
    k_codec_decode<<<codec_grid(n_desc * S, n_sms), kCodecThreads, 0, st>>>(desc, n_desc, slot, S);
    return codec_launched(1);
}

}  // namespace gcr
