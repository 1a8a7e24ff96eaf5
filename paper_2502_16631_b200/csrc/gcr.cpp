// gcr.cpp -- libgcr host runtime and C-ABI (include/gcr.h).
//
// Registry + phase machine (§3.1.1 lock/checkpoint/restore/unlock,
// P:157-173), A1 page table, the chunked checkpoint pipeline
// (K1 scan -> K2 compaction -> K4 pack -> pinned D2H on copy streams,
// overlapped with K1 of the next chunk), the pagemap (K3), the
// restore pipeline (H2D -> K6 scatter, K7 zero fill, K8 verify; §3.4), the
// pinned-host pool and the image model.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: a no-op unless a tool (nsys) injects itself
#include <cuda.h>  // VMM types only: entry points come from cudaGetDriverEntryPoint (no -lcuda)

#include "../../include/gcr.h"
#include "gcr_internal.h"

using namespace gcr;

static_assert(sizeof(gcr_image_hdr) == 96, "header is 96 bytes");
static_assert(offsetof(gcr_image_hdr, page_size) == 12 && offsetof(gcr_image_hdr, generation) == 16 &&
                  offsetof(gcr_image_hdr, n_allocs) == 32 && offsetof(gcr_image_hdr, n_pages) == 40 &&
                  offsetof(gcr_image_hdr, image_bytes) == 80 && offsetof(gcr_image_hdr, meta_crc32c) == 88,
              "header offsets fixed by the format contract");
static_assert(sizeof(gcr_alloc_rec) == 24 && sizeof(gcr_pagemap_entry) == 16, "record sizes");

namespace {

using Clock = std::chrono::steady_clock;
// NVTX range over an API call or a pipeline stage (gcr.lock, gcr.checkpoint,
// gcr.checkpoint.pagemap, gcr.restore, gcr.restore.verify, ...): nsys shows
// the library's phases on the host timeline next to its kernels and copies.
struct NvtxScope {
    explicit NvtxScope(const char *name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope &) = delete;
    NvtxScope &operator=(const NvtxScope &) = delete;
};

uint64_t ns_since(Clock::time_point t0) {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
}

constexpr uint64_t kMaxChunk = 2ull << 30;
constexpr uint64_t kPieceBytes = 1ull << 20;  // restore descriptor granularity (K6 assumes <= 1 MiB)
constexpr uint64_t kGroupMax = 64ull << 20;   // restore: bytes per staged H2D group
constexpr uint64_t kCodecSub = 256ull << 20;  // f4 checkpoint: page bytes per encode + D2H sub-chunk
constexpr uint64_t kCodecSubFirst = 32ull << 20;  // f4 checkpoint: the first chunk's first sub-chunk (ramp start)
constexpr size_t kDigestChunks = 4;           // checkpoint: chunks per digest D2H
const char kMagic[8] = {'G', 'C', 'R', 'I', 'M', 'G', 0x00, 0x01};

// ---------------------------------------------------------------------------
// Pinned host pool: slabs from cudaHostAlloc, first-fit free lists with
// coalescing.  gcr_reserve_host pre-pins slabs so the locked window never
// pays for pinning.
struct Slab {
    uint8_t *base = nullptr;
    uint64_t size = 0;
    std::map<uint64_t, uint64_t> free_;  // offset -> length
};

struct PinnedPool {
    std::vector<Slab *> slabs;
    uint64_t pin_ns = 0;

    ~PinnedPool() {
        for (Slab *s : slabs) {
            cudaFreeHost(s->base);
            delete s;
        }
    }
    static uint64_t round(uint64_t b) { return (b + 4095) & ~4095ull; }

    bool add_slab(uint64_t bytes) {
        auto t0 = Clock::now();
        void *p = nullptr;
        // mapped: the f1 in-scan pack writes image data from the scan kernel
        if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        pin_ns += ns_since(t0);
        Slab *s = new Slab;
        s->base = static_cast<uint8_t *>(p);
        s->size = bytes;
        s->free_[0] = bytes;
        slabs.push_back(s);
        return true;
    }
    void *try_alloc(uint64_t bytes) {
        for (Slab *s : slabs)
            for (auto it = s->free_.begin(); it != s->free_.end(); ++it)
                if (it->second >= bytes) {
                    uint64_t off = it->first, len = it->second;
                    s->free_.erase(it);
                    if (len > bytes) s->free_[off + bytes] = len - bytes;
                    return s->base + off;
                }
        return nullptr;
    }
    void *alloc(uint64_t bytes) {
        bytes = round(std::max<uint64_t>(bytes, 1));
        void *p = try_alloc(bytes);
        if (p) return p;
        if (!add_slab(std::max<uint64_t>(bytes, 256ull << 20))) return nullptr;
        return try_alloc(bytes);
    }
    Slab *owner(void *p) {
        for (Slab *s : slabs)
            if ((uint8_t *)p >= s->base && (uint8_t *)p < s->base + s->size) return s;
        return nullptr;
    }
    void release(void *p, uint64_t bytes) {
        if (!p) return;
        bytes = round(std::max<uint64_t>(bytes, 1));
        Slab *s = owner(p);
        if (!s) return;
        uint64_t off = (uint8_t *)p - s->base;
        auto it = s->free_.emplace(off, bytes).first;
        auto nx = std::next(it);
        if (nx != s->free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            s->free_.erase(nx);
        }
        if (it != s->free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                s->free_.erase(it);
            }
        }
    }
    // keep the first new_bytes of an allocation of old_bytes
    void shrink(void *p, uint64_t old_bytes, uint64_t new_bytes) {
        uint64_t o = round(std::max<uint64_t>(old_bytes, 1)), n = round(std::max<uint64_t>(new_bytes, 1));
        if (n < o) release((uint8_t *)p + n, o - n);
    }
    uint64_t free_bytes() const {
        uint64_t f = 0;
        for (Slab *s : slabs)
            for (auto &kv : s->free_) f += kv.second;
        return f;
    }
};

struct RegEntry {
    uint32_t id;
    uint64_t dptr, bytes;
};

// A gcr_mem_alloc block (f2): reserved VA range + physical backing.
struct MemBlock {
    uint64_t va, user_bytes, size;  // size: user_bytes rounded up to the granularity
    CUmemGenericAllocationHandle h;
    bool mapped;
};

// Driver VMM entry points, resolved once through the runtime.
struct Vmm {
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    bool ok = false;
};

const Vmm &vmm() {
    static const Vmm v = [] {
        Vmm r;
        auto get = [](const char *name, void *fp) {
            cudaDriverEntryPointQueryResult q{};
            return cudaGetDriverEntryPoint(name, reinterpret_cast<void **>(fp), cudaEnableDefault, &q) ==
                       cudaSuccess &&
                   q == cudaDriverEntryPointSuccess;
        };
        r.ok = get("cuMemGetAllocationGranularity", &r.granularity) && get("cuMemAddressReserve", &r.reserve) &&
               get("cuMemAddressFree", &r.addr_free) && get("cuMemCreate", &r.create) &&
               get("cuMemRelease", &r.release) && get("cuMemMap", &r.map) && get("cuMemUnmap", &r.unmap) &&
               get("cuMemSetAccess", &r.set_access);
        cudaGetLastError();
        return r;
    }();
    return v;
}

CUmemAllocationProp mem_prop(int device) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    return prop;
}

// Back [b.va, b.va + b.size) with new physical memory (cuMemCreate + Map + SetAccess).
CUresult map_block(int device, MemBlock &b) {
    const Vmm &v = vmm();
    const CUmemAllocationProp prop = mem_prop(device);
    CUmemGenericAllocationHandle h{};
    CUresult r = v.create(&h, b.size, &prop, 0);
    if (r != CUDA_SUCCESS) return r;
    r = v.map(b.va, b.size, 0, h, 0);
    if (r != CUDA_SUCCESS) {
        v.release(h);
        return r;
    }
    CUmemAccessDesc ad{};
    ad.location = prop.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = v.set_access(b.va, b.size, &ad, 1);
    if (r != CUDA_SUCCESS) {
        v.unmap(b.va, b.size);
        v.release(h);
        return r;
    }
    b.h = h;
    b.mapped = true;
    return CUDA_SUCCESS;
}

// Return the physical memory (the VA range stays reserved).
CUresult unmap_block(MemBlock &b) {
    const Vmm &v = vmm();
    CUresult r = v.unmap(b.va, b.size);
    if (r != CUDA_SUCCESS) return r;
    r = v.release(b.h);
    b.mapped = false;
    return r;
}

struct Chunk {
    uint64_t tile_begin, tile_end, page_begin, page_end, row_begin, row_end;
};

}  // namespace

struct gcr_image {
    gcr_ctx *ctx = nullptr;
    gcr_image_hdr hdr{};
    std::vector<gcr_alloc_rec> allocs;
    gcr_pagemap_entry *pagemap = nullptr;
    uint64_t pagemap_cap = 0;
    uint32_t *digests = nullptr;
    uint64_t digests_cap = 0;
    uint8_t *data = nullptr;
    uint64_t data_cap = 0;
    uint32_t *stored = nullptr;  // f4: stored length per PRESENT page (flags bit 1), pinned
    uint64_t stored_cap = 0;
};

struct gcr_ctx {
    int device = 0;
    int n_sms = 148;
    gcr_config cfg{};
    gcr_phase phase = GCR_RUNNING;
    std::string err;
    gcr_stats stats{};

    std::vector<RegEntry> reg;
    uint32_t next_id = 1;
    std::vector<MemBlock> blocks;  // gcr_mem_alloc (f2)
    std::vector<cudaStream_t> watched;

    cudaStream_t compute = nullptr;
    cudaStream_t post = nullptr;  // K2 compaction + totals, off the scan's critical path
    cudaStream_t packs = nullptr; // K4 packs, one at a time, feeding the copy streams
    std::vector<cudaStream_t> copy;
    std::vector<uint8_t *> slots;
    CrcTables *tables_d = nullptr;
    uint32_t basis[8][32] = {};  // ScanParams::basis rows: braid(512), t4, a16 .. a256, then a128 / a256 for K1g
    PinnedPool pool;
    std::vector<gcr_image *> images;

    // layout (A1), rebuilt when the registry changes
    bool layout_valid = false;
    uint32_t P = 0, lg = 0;
    uint64_t n_pages = 0, n_tiles = 0, n_rows = 0;
    std::vector<AllocDev> allocs_h;
    std::vector<Chunk> chunks;
    AllocDev *allocs_d = nullptr;
    uint32_t *page_alloc = nullptr, *tile_alloc = nullptr;
    uint32_t *D[2] = {nullptr, nullptr};
    uint8_t *cls = nullptr;
    TileInfo *tile_info = nullptr;
    uint64_t *chunk_rows_d = nullptr;  // chunk row boundaries (nch + 1), then {0, n_rows} for verify
    uint64_t *chunk_groups_d = nullptr;  // K1g (4/8 KiB pages): the same in page groups, else null
    uint32_t *chunk_sync_d = nullptr;  // per chunk: K1 arrival counter [0, nch), chunk_done [nch, 2 nch),
                                       // K4 width decision [2 nch, 3 nch)
    uint32_t epoch = 0;                // K1 launch id published in chunk_done
    unsigned long long *fold_slots = nullptr;  // K1's cut-page fold: one u64 per K1 warp and chunk, zero between launches
    FoldSlots fold{};
    uint32_t *pm_blk_cnt = nullptr, *pm_blk_off = nullptr, *run_start = nullptr;
    void *entries_d = nullptr;
    // f4 codec (cfg.compress): per staging slot the KA/KB/KC scratch (plan,
    // offsets, presence masks of one chunk's pages), the image's compact
    // stored-length table, and each chunk's stored total (mapped pinned)
    std::vector<uint32_t *> cx_scratch;
    // f1 in-scan pack (cfg.in_scan_pack): per-CTA aggregates, chunk bases,
    // per-warp page lists, error word (InScanPack)
    unsigned long long *isp_cta = nullptr, *isp_base = nullptr, *isp_err = nullptr;
    uint32_t *isp_ready = nullptr, *isp_list = nullptr;
    uint32_t isp_cap = 0;
    uint64_t cx_pages = 0;  // pages per chunk at most (chunk_bytes / P)
    uint32_t *stored_d = nullptr;
    unsigned long long *ctot_h = nullptr, *ctot_map = nullptr;
    ChunkTotals *totals_h = nullptr, *totals_map = nullptr;  // mapped pinned, written by K2
    unsigned long long *misc_d = nullptr, *misc_h = nullptr;  // [0] n_entries, [1] verify count, [2] first bad
    unsigned long long *nent_h = nullptr, *nent_map = nullptr;  // mapped pinned n_entries
    TileRec *tile_rec_h = nullptr, *tile_rec_map = nullptr;     // mapped pinned non-empty tile records
    unsigned long long *rec_count_h = nullptr, *rec_count_map = nullptr;  // per chunk: records written
    uint8_t *pack_flags_h = nullptr;   // per-tile plan scratch: packed (1) or direct (0)
    StageItem *stage_h = nullptr, *stage_map = nullptr;  // mapped pinned K4 work lists, indexed by global tile
    uint32_t z_page = 0;

    // restore descriptor buffers (grow on demand)
    uint8_t *desc_d = nullptr, *desc_h = nullptr;
    uint64_t desc_cap = 0;

    // incremental parent state (R-8)
    bool have_parent = false;
    int parent_idx = 0;
    uint64_t parent_gen = 0;
    uint64_t next_gen = 1;
    // the parent state before the last successful checkpoint, and its image:
    // gcr_checkpoint_abort undoes that checkpoint (multi-rank all-or-nothing)
    gcr_image *last_ckpt = nullptr;
    bool prev_have_parent = false;
    int prev_parent_idx = 0;
    uint64_t prev_parent_gen = 0, prev_next_gen = 1;

    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t ev_spec = nullptr;  // restore: the speculative prefix H2D (outlives the pool's per-call reset)
    size_t ev_used = 0;
    cudaEvent_t ev() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
};

namespace {

gcr_status fail(gcr_ctx *c, gcr_status s, const std::string &msg) {
    if (c) c->err = msg;
    return s;
}

#define CUDA_TRY(ctx, call)                                                                            \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) {                                                                       \
            cudaGetLastError();                                                                        \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? GCR_E_NOMEM : GCR_E_CUDA,               \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                           \
        }                                                                                              \
    } while (0)

#define LAUNCH_TRY(ctx, call)                                                                          \
    do {                                                                                               \
        int n_ = (call);                                                                               \
        if (n_ < 0) {                                                                                  \
            cudaError_t e_ = cudaGetLastError();                                                       \
            return fail(ctx, GCR_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
        }                                                                                              \
        ctx->stats.kernel_launches += (uint64_t)n_;                                                   \
    } while (0)

uint32_t log2u(uint64_t v) {
    uint32_t r = 0;
    while ((1ull << r) < v) r++;
    return r;
}

bool valid_page_size(uint32_t P) { return P >= 4096u && P <= 2097152u && (P & (P - 1u)) == 0; }

void free_layout(gcr_ctx *c) {
    void *ptrs[] = {c->allocs_d, c->page_alloc, c->tile_alloc, c->D[0], c->D[1], c->cls, c->tile_info,
                    c->chunk_rows_d, c->chunk_groups_d, c->chunk_sync_d, c->fold_slots, c->pm_blk_cnt,
                    c->pm_blk_off, c->run_start, c->entries_d, c->misc_d};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    for (uint32_t *p : c->cx_scratch)
        if (p) cudaFree(p);
    c->cx_scratch.clear();
    for (void *p : {(void *)c->isp_cta, (void *)c->isp_base, (void *)c->isp_err, (void *)c->isp_ready,
                    (void *)c->isp_list})
        if (p) cudaFree(p);
    c->isp_cta = c->isp_base = c->isp_err = nullptr;
    c->isp_ready = c->isp_list = nullptr;
    if (c->stored_d) cudaFree(c->stored_d);
    c->stored_d = nullptr;
    if (c->ctot_h) cudaFreeHost(c->ctot_h);
    c->ctot_h = c->ctot_map = nullptr;
    if (c->totals_h) cudaFreeHost(c->totals_h);
    if (c->misc_h) cudaFreeHost(c->misc_h);
    if (c->nent_h) cudaFreeHost(c->nent_h);
    if (c->tile_rec_h) cudaFreeHost(c->tile_rec_h);
    if (c->rec_count_h) cudaFreeHost(c->rec_count_h);
    c->rec_count_h = c->rec_count_map = nullptr;
    if (c->pack_flags_h) cudaFreeHost(c->pack_flags_h);
    if (c->stage_h) cudaFreeHost(c->stage_h);
    c->stage_h = c->stage_map = nullptr;
    c->tile_rec_h = c->tile_rec_map = nullptr;
    c->pack_flags_h = nullptr;
    c->nent_h = c->nent_map = nullptr;
    c->totals_map = nullptr;
    c->allocs_d = nullptr;
    c->page_alloc = c->tile_alloc = c->D[0] = c->D[1] = nullptr;
    c->cls = nullptr;
    c->tile_info = nullptr;
    c->chunk_rows_d = nullptr;
    c->chunk_groups_d = nullptr;
    c->chunk_sync_d = nullptr;
    c->fold_slots = nullptr;
    c->pm_blk_cnt = c->pm_blk_off = c->run_start = nullptr;
    c->entries_d = nullptr;
    c->totals_h = nullptr;
    c->misc_d = c->misc_h = nullptr;
    c->layout_valid = false;
    c->have_parent = false;
}

// A1: per-allocation page/tile bases, chunk plan, device buffers, K0.
gcr_status build_layout(gcr_ctx *c) {
    if (c->layout_valid) return GCR_OK;
    free_layout(c);
    const uint32_t P = c->cfg.page_size, lg = log2u(P);
    c->P = P;
    c->lg = lg;
    c->allocs_h.clear();
    uint64_t g = 0, t = 0, rows = 0, groups = 0;
    const bool grp = scan_uses_groups(P);
    const uint64_t G = grp ? kGroupBytes / P : 1;
    for (const RegEntry &r : c->reg) {
        AllocDev a{};
        a.base = r.dptr;
        a.bytes = r.bytes;
        a.page0 = g;
        a.tile0 = t;
        a.n_pages = (uint32_t)((r.bytes + P - 1) / P);
        a.n_tiles = P <= kTileBytes ? (uint32_t)((a.n_pages + (kTileBytes / P) - 1) / (kTileBytes / P))
                                    : a.n_pages * (P / kTileBytes);
        a.tail_len = (uint32_t)(r.bytes - (uint64_t)(a.n_pages - 1) * P);
        a.z_tail = zero_digest(a.tail_len);
        a.row0 = rows;
        a.n_rows = (uint64_t)(a.n_pages - 1) * (P / kRowBytes) + (a.tail_len + kRowBytes - 1) / kRowBytes;
        rows += a.n_rows;
        a.grp0 = groups;
        groups += (a.n_pages + G - 1) / G;
        g += a.n_pages;
        t += a.n_tiles;
        c->allocs_h.push_back(a);
    }
    c->n_pages = g;
    c->n_tiles = t;
    c->z_page = zero_digest(P);
    // chunk plan: uniform tile ranges; page ranges from the allocation walk
    // chunk plan: uniform tile ranges of chunk_bytes.  GCR_CHUNK_RAMP=1 ramps
    // a long registry (>= 8 chunks) up and down (1/8, 1/4, 1/2 chunk at both
    // ends, whole pages): the first drain starts ~0.4 ms earlier, but measured
    // on C4 the step did not improve (1 %: 8.90 -> 9.00 ms, 5 %: 39.65 ->
    // 39.46 ms; profiles/r1s_chunk_ramp_ab.jsonl) -- the drain, not its start,
    // bounds it -- and every extra chunk costs each K1 warp a range restart.
    const uint64_t ct = c->cfg.chunk_bytes / kTileBytes;
    const uint64_t tpp = P > kTileBytes ? P / kTileBytes : 1;  // tiles per page
    c->chunks.clear();
    {
        std::vector<uint64_t> sizes;
        const char *ramp_env = std::getenv("GCR_CHUNK_RAMP");  // read per layout (tests flip it)
        const int ramp_mode = ramp_env ? std::atoi(ramp_env) : 0;  // 1: both ends, 2: the end only
        if (ramp_mode >= 1 && ramp_mode <= 2 && t >= 8 * ct && ct >= 8 * tpp) {
            const uint64_t r[3] = {ct / 8, ct / 4, ct / 2};
            uint64_t ramp = 0;
            for (uint64_t x : r) ramp += x / tpp * tpp;
            uint64_t mid = t - (ramp_mode == 1 ? 2 : 1) * ramp;
            if (ramp_mode == 1)
                for (uint64_t x : r) sizes.push_back(x / tpp * tpp);
            for (; mid > 0; mid -= std::min(mid, ct)) sizes.push_back(std::min(mid, ct));
            for (int k = 2; k >= 0; k--) sizes.push_back(r[k] / tpp * tpp);
        } else {
            for (uint64_t tb = 0; tb < t; tb += ct) sizes.push_back(std::min(ct, t - tb));
        }
        uint64_t tb = 0;
        for (uint64_t n : sizes) {
            if (n == 0) continue;
            c->chunks.push_back(Chunk{tb, tb + n, 0, 0, 0, 0});
            tb += n;
        }
    }
    auto page_of_tile = [&](uint64_t tile) -> uint64_t {
        if (tile >= t) return g;
        // allocation containing tile (linear walk is fine: done once per layout)
        size_t lo = 0, hi = c->allocs_h.size();
        while (hi - lo > 1) {
            size_t mid = (lo + hi) / 2;
            if (c->allocs_h[mid].tile0 <= tile) lo = mid; else hi = mid;
        }
        const AllocDev &a = c->allocs_h[lo];
        const uint64_t lt = tile - a.tile0;
        return a.page0 + (P <= kTileBytes ? lt * (kTileBytes / P) : lt / (P / kTileBytes));
    };
    auto row_of_page = [&](uint64_t page) -> uint64_t {
        if (page >= g) return rows;
        size_t lo = 0, hi = c->allocs_h.size();
        while (hi - lo > 1) {
            size_t mid = (lo + hi) / 2;
            if (c->allocs_h[mid].page0 <= page) lo = mid; else hi = mid;
        }
        return c->allocs_h[lo].row0 + (page - c->allocs_h[lo].page0) * (P / kRowBytes);
    };
    for (Chunk &ch : c->chunks) {
        ch.page_begin = page_of_tile(ch.tile_begin);
        ch.page_end = page_of_tile(ch.tile_end);
        ch.row_begin = row_of_page(ch.page_begin);
        ch.row_end = row_of_page(ch.page_end);
    }
    c->n_rows = rows;
    const uint64_t na = c->allocs_h.size(), nblk = (g + 4095) / 4096, nch = c->chunks.size();
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMalloc(&c->allocs_d, sizeof(AllocDev) * na));
    CUDA_TRY(c, cudaMalloc(&c->page_alloc, 4 * g));
    CUDA_TRY(c, cudaMalloc(&c->tile_alloc, 4 * t));
    CUDA_TRY(c, cudaMalloc(&c->D[0], 4 * g));
    CUDA_TRY(c, cudaMalloc(&c->D[1], 4 * g));
    CUDA_TRY(c, cudaMalloc(&c->cls, g));
    CUDA_TRY(c, cudaMalloc(&c->tile_info, sizeof(TileInfo) * t));
    CUDA_TRY(c, cudaMemset(c->tile_info, 0, sizeof(TileInfo) * t));
    {
        std::vector<uint64_t> cr;
        for (const Chunk &ch : c->chunks) cr.push_back(ch.row_begin);
        cr.push_back(rows);
        cr.push_back(0);
        cr.push_back(rows);
        CUDA_TRY(c, cudaMalloc(&c->chunk_rows_d, 8 * cr.size()));
        CUDA_TRY(c, cudaMemcpy(c->chunk_rows_d, cr.data(), 8 * cr.size(), cudaMemcpyHostToDevice));
        if (grp) {  // K1g: chunk boundaries in page groups (tile-aligned chunks are group-aligned)
            auto group_of_page = [&](uint64_t page) -> uint64_t {
                if (page >= g) return groups;
                size_t lo = 0, hi = c->allocs_h.size();
                while (hi - lo > 1) {
                    size_t mid = (lo + hi) / 2;
                    if (c->allocs_h[mid].page0 <= page) lo = mid; else hi = mid;
                }
                return c->allocs_h[lo].grp0 + (page - c->allocs_h[lo].page0) / G;
            };
            std::vector<uint64_t> cg;
            for (const Chunk &ch : c->chunks) cg.push_back(group_of_page(ch.page_begin));
            cg.push_back(groups);
            cg.push_back(0);
            cg.push_back(groups);
            CUDA_TRY(c, cudaMalloc(&c->chunk_groups_d, 8 * cg.size()));
            CUDA_TRY(c, cudaMemcpy(c->chunk_groups_d, cg.data(), 8 * cg.size(), cudaMemcpyHostToDevice));
        }
        const uint64_t ns = std::max<uint64_t>(nch, 1);
        CUDA_TRY(c, cudaMalloc(&c->chunk_sync_d, 3 * 4 * ns));
        CUDA_TRY(c, cudaMemset(c->chunk_sync_d, 0, 3 * 4 * ns));
        // fold slots: one pair per K1 warp per chunk (warps run ahead into later
        // chunks independently, so chunks never share slots)
        const uint64_t w = scan_workers(c->n_sms, 0) * ns;  // the verify K8 uses every SM
        CUDA_TRY(c, cudaMalloc(&c->fold_slots, 8 * w));
        CUDA_TRY(c, cudaMemset(c->fold_slots, 0, 8 * w));
        c->fold = FoldSlots{c->fold_slots};
    }
    CUDA_TRY(c, cudaMalloc(&c->pm_blk_cnt, 4 * nblk));
    CUDA_TRY(c, cudaMalloc(&c->pm_blk_off, 4 * nblk));
    CUDA_TRY(c, cudaMalloc(&c->run_start, 4 * g));
    CUDA_TRY(c, cudaMalloc(&c->entries_d, sizeof(gcr_pagemap_entry) * g));
    CUDA_TRY(c, cudaHostAlloc(&c->totals_h, sizeof(ChunkTotals) * nch, cudaHostAllocMapped));
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->totals_map), c->totals_h, 0));
    CUDA_TRY(c, cudaHostAlloc(&c->nent_h, 64, cudaHostAllocMapped));
    CUDA_TRY(c, cudaHostAlloc(&c->tile_rec_h, sizeof(TileRec) * t, cudaHostAllocMapped));
    CUDA_TRY(c, cudaHostAlloc(&c->rec_count_h, sizeof(unsigned long long) * nch, cudaHostAllocMapped));
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->rec_count_map), c->rec_count_h, 0));
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->tile_rec_map), c->tile_rec_h, 0));
    CUDA_TRY(c, cudaHostAlloc(&c->pack_flags_h, t, cudaHostAllocDefault));
    CUDA_TRY(c, cudaHostAlloc(&c->stage_h, sizeof(StageItem) * t, cudaHostAllocMapped));
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->stage_map), c->stage_h, 0));
    CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->nent_map), c->nent_h, 0));
    CUDA_TRY(c, cudaMalloc(&c->misc_d, 8 * 4));
    CUDA_TRY(c, cudaHostAlloc(&c->misc_h, 8 * 4, cudaHostAllocDefault));
    if (c->cfg.in_scan_pack) {  // f1 buffers, sized for the narrowest K1 grid (incremental: most rows per warp)
        const uint64_t w_min = scan_workers(c->n_sms, scan_free_sms(true));
        const uint64_t w_max = scan_workers(c->n_sms, 0);
        uint64_t max_rows = 0;
        for (const Chunk &ch : c->chunks) max_rows = std::max(max_rows, ch.row_end - ch.row_begin);
        // pages one warp can finalize in a chunk: its rows' worth + the pages cut at both ends
        uint64_t cap = (max_rows + w_min - 1) / w_min * kRowBytes / P + 3;
        if (grp) cap = std::max<uint64_t>(cap, ((max_rows * kRowBytes / kGroupBytes) + w_min - 1) / w_min * G + 2 * G);
        c->isp_cap = (uint32_t)cap;
        const uint64_t ctas = (w_max + 19) / 20 + 1;
        CUDA_TRY(c, cudaMalloc(&c->isp_cta, 8 * (nch + 1) * ctas));
        CUDA_TRY(c, cudaMemset(c->isp_cta, 0, 8 * (nch + 1) * ctas));
        CUDA_TRY(c, cudaMalloc(&c->isp_base, 8 * (nch + 2)));
        CUDA_TRY(c, cudaMemset(c->isp_base, 0, 8 * (nch + 2)));
        CUDA_TRY(c, cudaMalloc(&c->isp_ready, 4 * (nch + 2)));
        CUDA_TRY(c, cudaMemset(c->isp_ready, 0, 4 * (nch + 2)));
        CUDA_TRY(c, cudaMalloc(&c->isp_err, 8));
        CUDA_TRY(c, cudaMalloc(&c->isp_list, 4 * 2 * w_max * cap));
    }
    if (c->cfg.compress) {  // f4 scratch: {plan, offsets, 32 mask words} per page of a chunk, per slot
        c->cx_pages = c->cfg.chunk_bytes / P;
        for (size_t k = 0; k < c->slots.size(); k++) {
            uint32_t *x = nullptr;
            CUDA_TRY(c, cudaMalloc(&x, 4 * 34 * c->cx_pages));
            c->cx_scratch.push_back(x);
        }
        CUDA_TRY(c, cudaMalloc(&c->stored_d, 4 * std::max<uint64_t>(g, 1)));
        CUDA_TRY(c, cudaHostAlloc(&c->ctot_h, 16, cudaHostAllocMapped));  // {sub-chunk stored bytes, PRESENT pages}
        CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->ctot_map), c->ctot_h, 0));
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->allocs_d, c->allocs_h.data(), sizeof(AllocDev) * na, cudaMemcpyHostToDevice,
                                c->compute));
    LAUNCH_TRY(c, launch_build_page_table(c->allocs_d, (uint32_t)na, c->page_alloc, c->tile_alloc,
                                          P > kTileBytes ? P / kTileBytes : 1, P <= kTileBytes ? kTileBytes / P : 1,
                                          c->compute));
    CUDA_TRY(c, cudaStreamSynchronize(c->compute));
    c->layout_valid = true;
    c->have_parent = false;
    return GCR_OK;
}

void sync_all(gcr_ctx *c) {
    cudaStreamSynchronize(c->compute);
    if (c->post) cudaStreamSynchronize(c->post);
    if (c->packs) cudaStreamSynchronize(c->packs);
    for (cudaStream_t s : c->copy) cudaStreamSynchronize(s);
    cudaGetLastError();
}

void image_free_buffers(gcr_image *img) {
    if (!img || !img->ctx) return;
    PinnedPool &p = img->ctx->pool;
    p.release(img->pagemap, img->pagemap_cap);
    p.release(img->digests, img->digests_cap);
    p.release(img->data, img->data_cap);
    p.release(img->stored, img->stored_cap);
    img->pagemap = nullptr;
    img->digests = nullptr;
    img->data = nullptr;
    img->stored = nullptr;
}

void destroy_image(gcr_ctx *c, gcr_image *img) {
    if (c->last_ckpt == img) c->last_ckpt = nullptr;
    image_free_buffers(img);
    auto it = std::find(c->images.begin(), c->images.end(), img);
    if (it != c->images.end()) c->images.erase(it);
    delete img;
}

// meta_crc32c = CRC32C(header with the field 0 | alloc table | pagemap |
// digests).  digests_reg, if given, is reg(0, digests) computed earlier (the
// checkpoint CRCs digest batches while the drain runs); it is joined by
// linearity: reg(s, X|D) = adv_|D|(reg(s, X)) ^ reg(0, D).
uint32_t meta_crc(const gcr_image *img, const uint32_t *digests_reg = nullptr) {
    gcr_image_hdr h = img->hdr;
    h.meta_crc32c = 0;
    uint32_t s = host_crc32c_update(0xFFFFFFFFu, &h, sizeof h);
    s = host_crc32c_update(s, img->allocs.data(), sizeof(gcr_alloc_rec) * img->allocs.size());
    s = host_crc32c_update(s, img->pagemap, sizeof(gcr_pagemap_entry) * img->hdr.n_entries);
    if (digests_reg) s = crc_shift(s, 4ull * img->hdr.n_pages) ^ *digests_reg;
    else s = host_crc32c_update(s, img->digests, 4ull * img->hdr.n_pages);
    if (img->hdr.flags & 2u) s = host_crc32c_update(s, img->stored, 4ull * img->hdr.n_present);
    return s ^ 0xFFFFFFFFu;
}

uint64_t pages_of(uint64_t bytes, uint32_t P) { return (bytes + P - 1) / P; }
uint64_t page_len(uint64_t bytes, uint32_t P, uint64_t p) {
    uint64_t rest = bytes - p * (uint64_t)P;
    return rest < P ? rest : P;
}

// Structural check of an image against its own alloc table (CORRUPT on failure).
gcr_status check_pagemap(gcr_ctx *c, const gcr_image *img) {
    const gcr_image_hdr &h = img->hdr;
    const uint32_t P = h.page_size;
    if (!valid_page_size(P)) return fail(c, GCR_E_CORRUPT, "image page size invalid");
    uint64_t e = 0, np = 0, nz = 0, npa = 0, pb = 0, tot = 0, sb = 0;
    const bool coded = h.flags & 2u;
    for (uint32_t a = 0; a < h.n_allocs; a++) {
        const gcr_alloc_rec &r = img->allocs[a];
        if (r.bytes == 0) return fail(c, GCR_E_CORRUPT, "image alloc of 0 bytes");
        const uint64_t m = pages_of(r.bytes, P);
        tot += m;
        uint64_t p = 0;
        while (p < m) {
            if (e >= h.n_entries) return fail(c, GCR_E_CORRUPT, "pagemap too short");
            const gcr_pagemap_entry &pe = img->pagemap[e];
            if (pe.vaddr != r.vaddr + p * P || pe.nr_pages == 0 || p + pe.nr_pages > m)
                return fail(c, GCR_E_CORRUPT, "pagemap entry inconsistent with alloc table");
            if (pe.flags == GCR_PE_PRESENT) {
                if (coded) {  // f4: raw (== length) or a coded form, a multiple of 16 shorter
                    for (uint64_t q = p; q < p + pe.nr_pages; q++) {
                        if (np + (q - p) >= h.n_present) return fail(c, GCR_E_CORRUPT, "stored-length table too short");
                        const uint64_t L = page_len(r.bytes, P, q), st = img->stored[np + (q - p)];
                        if (st > L || (st != L && (st % 16 != 0 || st < 16)))
                            return fail(c, GCR_E_CORRUPT, "stored length inconsistent with its page");
                        sb += st;
                    }
                }
                np += pe.nr_pages;
                uint64_t last = p + pe.nr_pages;
                pb += (last == m) ? (uint64_t)(pe.nr_pages - 1) * P + page_len(r.bytes, P, m - 1)
                                  : (uint64_t)pe.nr_pages * P;
            } else if (pe.flags == GCR_PE_ZERO) {
                nz += pe.nr_pages;
            } else if (pe.flags == GCR_PE_PARENT) {
                npa += pe.nr_pages;
            } else {
                return fail(c, GCR_E_CORRUPT, "pagemap flags invalid");
            }
            p += pe.nr_pages;
            e++;
        }
    }
    if (e != h.n_entries || tot != h.n_pages || np != h.n_present || nz != h.n_zero || npa != h.n_parent ||
        (coded ? sb : pb) != h.image_bytes)
        return fail(c, GCR_E_CORRUPT, "pagemap counts inconsistent with header");
    return GCR_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

gcr_status gcr_config_default(gcr_config *out) {
    if (!out) return GCR_E_INVAL;
    out->page_size = 65536;
    out->n_copy_streams = 2;
    out->chunk_bytes = 1ull << 30;
    out->n_staging_slots = 0;
    out->verify = 1;
    out->lock_timeout_ms = 10000;
    out->direct_min_bytes = 16ull << 20;
    out->compress = 0;
    out->in_scan_pack = 0;
    return GCR_OK;
}

gcr_status gcr_create(int cuda_device, const gcr_config *cfg_in, gcr_ctx **out) {
    if (!out) return GCR_E_INVAL;
    *out = nullptr;
    gcr_config cfg;
    gcr_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (!valid_page_size(cfg.page_size) || cfg.n_copy_streams < 1 || cfg.n_copy_streams > 8 ||
        cfg.chunk_bytes == 0 || cfg.chunk_bytes % cfg.page_size != 0 || cfg.chunk_bytes % kTileBytes != 0 ||
        cfg.chunk_bytes > kMaxChunk || cfg.compress > 1 || cfg.in_scan_pack > 2 ||
        (cfg.n_staging_slots != 0 && (cfg.n_staging_slots < cfg.n_copy_streams || cfg.n_staging_slots > 16)))
        return GCR_E_INVAL;
    if (!crc_self_test()) return GCR_E_INVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
        cudaGetLastError();
        return GCR_E_CUDA;
    }
    gcr_ctx *c = new (std::nothrow) gcr_ctx;
    if (!c) return GCR_E_NOMEM;
    c->device = cuda_device;
    c->cfg = cfg;
    c->stats.first_bad_page = UINT64_MAX;
    auto bail = [&](gcr_status s) {
        gcr_destroy(c);
        return s;
    };
    if (cudaSetDevice(cuda_device) != cudaSuccess) return bail(GCR_E_CUDA);
    cudaDeviceGetAttribute(&c->n_sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking) != cudaSuccess) return bail(GCR_E_CUDA);
    if (cudaStreamCreateWithFlags(&c->post, cudaStreamNonBlocking) != cudaSuccess) return bail(GCR_E_CUDA);
    if (cudaStreamCreateWithFlags(&c->packs, cudaStreamNonBlocking) != cudaSuccess) return bail(GCR_E_CUDA);
    if (cudaEventCreate(&c->ev_spec) != cudaSuccess) return bail(GCR_E_CUDA);
    scan_probe();  // K1g's immediate-base variant when this build's smem layout is confirmed (else the IADD one)
    cudaGetLastError();
    for (uint32_t i = 0; i < cfg.n_copy_streams; i++) {
        cudaStream_t s;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return bail(GCR_E_CUDA);
        c->copy.push_back(s);
    }
    for (uint32_t i = 0; i < (cfg.n_staging_slots ? cfg.n_staging_slots : cfg.n_copy_streams); i++) {
        void *slot = nullptr;
        if (cudaMalloc(&slot, cfg.chunk_bytes) != cudaSuccess) {
            cudaGetLastError();
            return bail(GCR_E_NOMEM);
        }
        c->slots.push_back(static_cast<uint8_t *>(slot));
    }
    CrcTables *th = new CrcTables;
    build_tables(th);
    table_basis(th->braid, c->basis[0]);
    table_basis(th->t4, c->basis[1]);
    table_basis(th->a16, c->basis[2]);
    table_basis(th->a32, c->basis[3]);
    table_basis(th->a64, c->basis[4]);
    table_basis(th->a128, c->basis[5]);
    table_basis(th->a256, c->basis[6]);
    if (cudaMalloc(&c->tables_d, sizeof(CrcTables)) != cudaSuccess ||
        cudaMemcpy(c->tables_d, th, sizeof(CrcTables), cudaMemcpyHostToDevice) != cudaSuccess) {
        delete th;
        cudaGetLastError();
        return bail(GCR_E_NOMEM);
    }
    delete th;
    *out = c;
    return GCR_OK;
}

gcr_status gcr_destroy(gcr_ctx *c) {
    if (!c) return GCR_E_INVAL;
    cudaSetDevice(c->device);
    sync_all(c);
    while (!c->images.empty()) destroy_image(c, c->images.back());
    free_layout(c);
    for (MemBlock &b : c->blocks) {
        if (b.mapped) unmap_block(b);
        vmm().addr_free(b.va, b.size);
    }
    for (uint8_t *s : c->slots) cudaFree(s);
    for (cudaStream_t s : c->copy) cudaStreamDestroy(s);
    if (c->compute) cudaStreamDestroy(c->compute);
    if (c->post) cudaStreamDestroy(c->post);
    if (c->packs) cudaStreamDestroy(c->packs);
    if (c->ev_spec) cudaEventDestroy(c->ev_spec);
    if (c->tables_d) cudaFree(c->tables_d);
    if (c->desc_d) cudaFree(c->desc_d);
    if (c->desc_h) cudaFreeHost(c->desc_h);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    cudaGetLastError();
    delete c;
    return GCR_OK;
}

gcr_status gcr_register(gcr_ctx *c, uint64_t dptr, uint64_t bytes, uint32_t *id_out) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "register: not RUNNING");
    if (!id_out || dptr == 0 || bytes == 0 || dptr % 16 || bytes % 16)
        return fail(c, GCR_E_INVAL, "register: null, empty or not 16-byte aligned (R-2)");
    if (dptr + bytes < dptr) return fail(c, GCR_E_INVAL, "register: range overflows");
    for (const RegEntry &r : c->reg)
        if (dptr < r.dptr + r.bytes && r.dptr < dptr + bytes)
            return fail(c, GCR_E_INVAL, "register: overlaps a registered allocation");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, reinterpret_cast<void *>(dptr)) != cudaSuccess ||
        at.type != cudaMemoryTypeDevice || at.device != c->device) {
        cudaGetLastError();
        return fail(c, GCR_E_INVAL, "register: not device memory of this ctx's device");
    }
    cudaPointerAttributes at2{};
    if (cudaPointerGetAttributes(&at2, reinterpret_cast<void *>(dptr + bytes - 1)) != cudaSuccess ||
        at2.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return fail(c, GCR_E_INVAL, "register: range end is not device memory");
    }
    c->reg.push_back(RegEntry{c->next_id, dptr, bytes});
    *id_out = c->next_id++;
    c->layout_valid = false;
    c->have_parent = false;
    return GCR_OK;
}

gcr_status gcr_unregister(gcr_ctx *c, uint32_t id) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "unregister: not RUNNING");
    for (size_t i = 0; i < c->reg.size(); i++)
        if (c->reg[i].id == id) {
            c->reg.erase(c->reg.begin() + i);
            c->layout_valid = false;
            c->have_parent = false;
            return GCR_OK;
        }
    return fail(c, GCR_E_INVAL, "unregister: unknown alloc_id");
}

gcr_status gcr_watch_stream(gcr_ctx *c, void *stream) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "watch_stream: not RUNNING");
    c->watched.push_back(static_cast<cudaStream_t>(stream));
    return GCR_OK;
}

gcr_status gcr_reserve_host(gcr_ctx *c, uint64_t bytes) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "reserve_host: not RUNNING");
    if (bytes == 0) return GCR_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (!c->pool.add_slab(PinnedPool::round(bytes))) return fail(c, GCR_E_NOMEM, "reserve_host: cudaHostAlloc failed");
    c->stats.pinned_alloc_ns = c->pool.pin_ns;
    return GCR_OK;
}

gcr_status gcr_lock(gcr_ctx *c) {
    NvtxScope nvtx_("gcr.lock");
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "lock: not RUNNING");
    auto t0 = Clock::now();
    CUDA_TRY(c, cudaSetDevice(c->device));
    // "waiting for active operations ... to complete" with a timeout
    const std::vector<cudaStream_t> &ws = c->watched;
    const uint64_t limit = c->cfg.lock_timeout_ms * 1000000ull;
    if (ws.empty()) {
        // Nothing watched: the whole device must be idle (every stream of the
        // process, blocking or not).  cudaDeviceSynchronize has no timeout, so
        // it runs on a helper thread that the lock waits for, bounded; on
        // expiry the helper is left to finish on its own (it touches only its
        // shared state) and the lock rolls back.
        struct Waiter {
            std::mutex m;
            std::condition_variable cv;
            bool done = false;
            cudaError_t err = cudaSuccess;
        };
        auto w = std::make_shared<Waiter>();
        const int dev = c->device;
        std::thread([w, dev] {
            cudaError_t e = cudaSetDevice(dev);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            std::lock_guard<std::mutex> g(w->m);
            w->done = true;
            w->err = e;
            w->cv.notify_all();
        }).detach();
        std::unique_lock<std::mutex> g(w->m);
        if (!w->cv.wait_for(g, std::chrono::nanoseconds(limit), [&] { return w->done; })) {
            c->stats.lock_ns = ns_since(t0);
            return fail(c, GCR_E_TIMEOUT, "lock: device not idle within lock_timeout_ms (rolled back)");
        }
        if (w->err != cudaSuccess)
            return fail(c, GCR_E_CUDA, std::string("lock: cudaDeviceSynchronize: ") + cudaGetErrorString(w->err));
    }
    while (!ws.empty()) {
        bool idle = true;
        for (cudaStream_t s : ws) {
            cudaError_t e = cudaStreamQuery(s);
            if (e == cudaErrorNotReady) {
                idle = false;
                break;
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail(c, GCR_E_CUDA, std::string("lock: cudaStreamQuery: ") + cudaGetErrorString(e));
            }
        }
        if (idle) break;
        if (ns_since(t0) >= limit) {
            c->stats.lock_ns = ns_since(t0);
            return fail(c, GCR_E_TIMEOUT, "lock: watched streams not idle within lock_timeout_ms (rolled back)");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    gcr_status s = build_layout(c);
    if (s != GCR_OK) {
        free_layout(c);
        return s;
    }
    c->phase = GCR_LOCKED;
    c->stats.lock_ns = ns_since(t0);
    return GCR_OK;
}

gcr_status gcr_unlock(gcr_ctx *c) {
    NvtxScope nvtx_("gcr.unlock");
    if (!c) return GCR_E_INVAL;
    if (c->phase == GCR_RELEASED) return fail(c, GCR_E_STATE, "unlock: device memory is released; restore first");
    if (c->phase != GCR_LOCKED && c->phase != GCR_CHECKPOINTED) return fail(c, GCR_E_STATE, "unlock: not locked");
    auto t0 = Clock::now();
    c->phase = GCR_RUNNING;
    c->stats.unlock_ns = ns_since(t0);
    return GCR_OK;
}

// Order a checkpoint / restore after every piece of caller work already
// enqueued: the watched streams, or the whole device when none is watched.
// Under the cooperative lock nothing should be pending, so this is a no-op
// wait; it makes "write the registered memory, then checkpoint / restore"
// on another stream (e.g. a test poisoning memory on torch's stream while
// LOCKED) safe instead of a race with the library's non-blocking streams.
static gcr_status fence_caller_work(gcr_ctx *c) {
    if (c->watched.empty()) {
        CUDA_TRY(c, cudaDeviceSynchronize());
        return GCR_OK;
    }
    for (cudaStream_t s : c->watched) CUDA_TRY(c, cudaStreamSynchronize(s));
    return GCR_OK;
}

// The launch's table bases (ScanParams::basis): the braid step is adv_512
// for K1, adv_{512/G} for K1g (a128 at 4 KiB pages, a256 at 8 KiB).
static void set_basis(const gcr_ctx *c, ScanParams &sp) {
    sp.t4rep = sp.chunk_groups != nullptr && grp_t4rep();
    int braid = 0;
    if (sp.chunk_groups != nullptr) braid = sp.page_size == kGroupBytes / 4 ? 5 : 6;
    std::memcpy(sp.basis[0], c->basis[braid], sizeof sp.basis[0]);
    for (int t = 1; t < 7; t++) std::memcpy(sp.basis[t], c->basis[t], sizeof sp.basis[t]);
}

static gcr_status checkpoint_impl(gcr_ctx *c, gcr_mode mode, gcr_image *img) {
    const uint32_t P = c->P;
    const int cur = c->have_parent ? 1 - c->parent_idx : 0;
    uint32_t *Dnew = c->D[cur];
    const uint32_t *Dref = mode == GCR_INCREMENTAL ? c->D[c->parent_idx] : nullptr;
    gcr_stats &st = c->stats;
    c->ev_used = 0;

    uint64_t R = 0;
    for (const RegEntry &r : c->reg) R += r.bytes;
    // Small metadata first, then the worst-case (R) data buffer, which is
    // shrunk to the image size right after the drain: nothing is ever placed
    // behind the data buffer, so the pool does not fragment across checkpoints.
    const bool coded = c->cfg.compress != 0;  // f4 page codec (R-19)
    img->digests_cap = 4 * c->n_pages;
    img->digests = static_cast<uint32_t *>(c->pool.alloc(img->digests_cap));
    if (coded) {  // worst case: every page PRESENT; shrunk after the drain
        img->stored_cap = 4 * c->n_pages;
        img->stored = static_cast<uint32_t *>(c->pool.alloc(img->stored_cap));
    }
    img->data_cap = R;
    img->data = static_cast<uint8_t *>(c->pool.alloc(R));
    st.pinned_alloc_ns = c->pool.pin_ns;
    if (!img->data || !img->digests || (coded && !img->stored))
        return fail(c, GCR_E_NOMEM, "checkpoint: pinned host allocation failed");

    ScanParams sp{};
    sp.allocs = c->allocs_d;
    sp.n_allocs = (uint32_t)c->allocs_h.size();
    sp.fold = c->fold;
    sp.page_size = P;
    sp.log2_page = c->lg;
    sp.z_page = c->z_page;
    sp.mode = mode == GCR_INCREMENTAL ? kScanIncremental : kScanFull;
    sp.d_ref = Dref;
    sp.d_out = Dnew;
    sp.cls = c->cls;
    sp.tile_info = c->tile_info;
    sp.tables = c->tables_d;
    sp.prefetch = scan_prefetch_bytes();

    const size_t nch = c->chunks.size();
    // One persistent K1 for the whole registry, walking the chunks in order;
    // K2(i) is enqueued ahead on the post stream and waits on K1's per-chunk
    // publication, so chunk i reaches the drain ~one chunk's scan after it
    // was scanned (no per-launch ramp and tail, no launch gaps: under a
    // saturated D2H every launch or event the GPU front-end fetches from host
    // memory costs tens of us).
    sp.chunk_rows = c->chunk_rows_d;
    sp.chunk_groups = c->chunk_groups_d;  // K1g for 4/8 KiB pages (null: K1)
    sp.grp_pf_block = grp_prefetch_block();
    sp.n_chunks = (uint32_t)nch;
    sp.epoch = ++c->epoch ? c->epoch : ++c->epoch;  // never 0 (the flags' initial value)
    sp.chunk_arrive = c->chunk_sync_d;
    sp.chunk_done = c->chunk_sync_d + std::max<size_t>(nch, 1);
    const int scan_free = scan_free_sms(mode == GCR_INCREMENTAL);
    sp.workers = scan_workers(c->n_sms, scan_free);
    set_basis(c, sp);
    // f1: the scan writes PRESENT pages straight into the mapped image
    const bool isp = !coded && (c->cfg.in_scan_pack == 2 || (c->cfg.in_scan_pack == 1 && mode == GCR_INCREMENTAL));
    // A full checkpoint needs chunk 0 early (the drain starts on it) and the
    // rest only before the link frees up (~a chunk's drain later, 10-100x the
    // scan of the rest): K1 splits chunks 1.. as ONE range over its warps and
    // publishes them together -- one range start per warp instead of one per
    // chunk.  Incremental checkpoints keep per-chunk publication (their drain
    // follows the scan chunk by chunk).  GCR_SCAN_MERGE=0: off (A/B).
    {
        const char *e = std::getenv("GCR_SCAN_MERGE");
        const bool merge = !(e && e[0] == '0');
        sp.merge_from = merge && mode == GCR_FULL && !isp && nch > 2 ? 1u : 0u;
    }
    if (isp) {
        void *dimg = nullptr;
        CUDA_TRY(c, cudaHostGetDevicePointer(&dimg, img->data, 0));
        sp.isp.img = static_cast<uint8_t *>(dimg);
        sp.isp.cta_agg = c->isp_cta;
        sp.isp.base = c->isp_base;
        sp.isp.base_ready = c->isp_ready;
        sp.isp.list = c->isp_list;
        sp.isp.cap = c->isp_cap;
        sp.isp.err = c->isp_err;
        {
            const char *e = std::getenv("GCR_ISP_WAIT_MS");  // diagnostics: shorter bound on the in-kernel waits
            sp.isp.wait_ns = (e ? std::strtoull(e, nullptr, 0) : 30000ull) * 1000000ull;
        }
        sp.isp_page_alloc = c->page_alloc;
        CUDA_TRY(c, cudaMemsetAsync(c->isp_err, 0, 8, c->compute));
    }
    std::vector<cudaEvent_t> k2s(nch), tot(nch), pks(nch), pke(nch), dde(nch);
    static const bool trace = std::getenv("GCR_TRACE") != nullptr;
    cudaEvent_t t0 = c->ev(), k1s = c->ev(), k1m = c->ev();
    CUDA_TRY(c, cudaEventRecord(t0, c->compute));
    const Clock::time_point host0 = Clock::now();  // trace: host enqueue times relative to t0
    std::vector<double> host_seen(trace ? nch : 0), host_enq(trace ? nch : 0);
    CUDA_TRY(c, cudaEventRecord(k1s, c->compute));
    LAUNCH_TRY(c, launch_scan(sp, c->n_sms, c->compute));
    CUDA_TRY(c, cudaEventRecord(k1m, c->compute));
    // K2 (per chunk: image offsets, non-empty tile records and chunk totals
    // straight into mapped pinned memory) on the post stream, beside the scan:
    // planning the drain never waits on a DMA queued behind the previous
    // drain.  Kept 3 chunks ahead of the drain (enqueueing everything up front
    // delays the first drain by the API calls).
    size_t enqueued = 0;  // K2s enqueued
    auto enqueue_k2 = [&](size_t i) -> gcr_status {
        const Chunk &ch = c->chunks[i];
        k2s[i] = c->ev();
        tot[i] = c->ev();
        CUDA_TRY(c, cudaEventRecord(k2s[i], c->post));
        LAUNCH_TRY(c, launch_tile_scan(c->tile_info, ch.tile_begin, ch.tile_end, sp.chunk_done, (uint32_t)i, sp.epoch,
                                       c->tile_rec_map + ch.tile_begin, c->rec_count_map + i, c->totals_map + i,
                                       isp ? c->isp_base : nullptr, isp ? c->isp_ready : nullptr, c->post));
        CUDA_TRY(c, cudaEventRecord(tot[i], c->post));
        return GCR_OK;
    };
    for (; enqueued < std::min<size_t>(nch, 3); enqueued++) {
        gcr_status es = enqueue_k2(enqueued);
        if (es != GCR_OK) return es;
    }
    // Drain: as each chunk's records land, plan it -- runs of fully PRESENT
    // tiles of at least direct_min_bytes go straight from the allocation to the
    // pinned image; the other PRESENT tiles are packed (K4) into the chunk's
    // staging slot and copied out in contiguous ranges.
    uint64_t base = 0, n_present = 0, n_zero = 0, n_parent = 0, raw_present = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> codec_ev;  // f4: KA+KB+KC span per sub-chunk
    struct SubTrace {  // GCR_TRACE: per f4 sub-chunk
        size_t chunk;
        cudaEvent_t ka, kb, kc, d2h;
        double host_enq;
    };
    std::vector<SubTrace> subs;
    Clock::time_point drain0;
    const size_t S = c->copy.size(), NS = c->slots.size();
    const uint64_t direct_min = c->cfg.direct_min_bytes;
    uint64_t direct_bytes = 0, staged_bytes = 0;
    struct Run {
        uint64_t src, off, bytes, t_first, t_last;
    };
    std::vector<Run> direct;
    std::vector<std::pair<uint64_t, uint64_t>> staged;  // chunk-local image ranges [lo, hi)
    size_t dg0 = 0;                                     // first chunk of the pending digest D2H
    // digest batches in page order: CRC'd on the host as their D2H completes
    struct DigestBatch {
        uint64_t pb, pe;
        cudaEvent_t done;
    };
    std::vector<DigestBatch> dbatch;
    size_t dnext = 0;
    uint32_t dreg = 0;  // reg(0, digests of the batches CRC'd so far)
    auto crc_batches = [&](bool wait) -> gcr_status {
        for (; dnext < dbatch.size(); dnext++) {
            const DigestBatch &b = dbatch[dnext];
            if (wait) CUDA_TRY(c, cudaEventSynchronize(b.done));
            else if (cudaEventQuery(b.done) != cudaSuccess) break;
            dreg = host_crc32c_update(dreg, img->digests + b.pb, 4 * (b.pe - b.pb));
        }
        cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
        return GCR_OK;
    };
    for (size_t i = 0; i < nch; i++) {
        const Chunk &ch = c->chunks[i];
        CUDA_TRY(c, cudaEventSynchronize(tot[i]));
        if (trace) host_seen[i] = ns_since(host0) * 1e-6;
        for (; enqueued < std::min(nch, i + 4); enqueued++) {
            gcr_status es = enqueue_k2(enqueued);
            if (es != GCR_OK) return es;
        }
        ChunkTotals T;
        {
            const volatile unsigned long long *h = reinterpret_cast<volatile unsigned long long *>(c->totals_h + i);
            T = ChunkTotals{h[0], h[1], h[2], h[3]};
        }
        const uint64_t present_base = n_present;  // f4: this chunk's first entry of the stored-length table
        n_present += T.n_present;
        n_zero += T.n_zero;
        n_parent += T.n_parent;
        raw_present += T.image_bytes;
        if (T.image_bytes == ~0ull) return fail(c, GCR_E_CUDA, "checkpoint: scan did not publish a chunk in time");
        if (base + T.image_bytes > R) return fail(c, GCR_E_CUDA, "checkpoint: image larger than registry");
        // ---- plan (host walk of the chunk's tiles) ----
        direct.clear();
        staged.clear();
        uint8_t *flags = c->pack_flags_h + ch.tile_begin;
        StageItem *items = c->stage_h + ch.tile_begin;
        uint32_t n_items = 0;
        bool any_staged = false;
        if (T.image_bytes && !coded && !isp) {
            std::memset(flags, 0, ch.tile_end - ch.tile_begin);
            Run run{0, 0, 0, 0, 0};
            bool open = false;
            auto stage_tiles = [&](uint64_t t_first, uint64_t t_last) {
                for (uint64_t t = t_first; t <= t_last; t++) flags[t - ch.tile_begin] = 1;
                any_staged = true;
            };
            auto close = [&]() {
                if (!open) return;
                if (run.bytes >= direct_min) direct.push_back(run);
                else stage_tiles(run.t_first, run.t_last);
                open = false;
            };
            size_t a = 0;
            {
                size_t lo = 0, hi = c->allocs_h.size();
                while (hi - lo > 1) {
                    size_t mid = (lo + hi) / 2;
                    if (c->allocs_h[mid].tile0 <= ch.tile_begin) lo = mid; else hi = mid;
                }
                a = lo;
            }
            const volatile uint32_t *rec = reinterpret_cast<const volatile uint32_t *>(c->tile_rec_h + ch.tile_begin);
            const uint64_t nrec = *reinterpret_cast<const volatile unsigned long long *>(c->rec_count_h + i);
            for (uint64_t k = 0; k < nrec; k++) {
                const uint64_t t = ch.tile_begin + rec[4 * k];
                const uint2 r = make_uint2(rec[4 * k + 1], rec[4 * k + 2]);
                while (t >= c->allocs_h[a].tile0 + c->allocs_h[a].n_tiles) a++;
                const AllocDev &al = c->allocs_h[a];
                const uint64_t lt = t - al.tile0;
                uint64_t src, span;
                if (P <= kTileBytes) {
                    src = al.base + lt * kTileBytes;
                    span = std::min<uint64_t>(kTileBytes, al.bytes - lt * kTileBytes);
                } else {  // anchor tile of a page: the whole page
                    const uint64_t pi = lt / (P / kTileBytes);
                    src = al.base + pi * P;
                    span = pi == al.n_pages - 1 ? al.tail_len : P;
                }
                // last tile the page(s) cover: the anchor itself, or all 64 KiB slices of a big page
                const uint64_t t_end = P <= kTileBytes ? t : t + P / kTileBytes - 1;
                if (r.x == span) {  // every page of the tile PRESENT: contiguous in memory and in the image
                    if (open && run.src + run.bytes == src && run.off + run.bytes == r.y) {
                        run.bytes += span;
                        run.t_last = t_end;
                    } else {
                        close();
                        run = Run{src, r.y, span, t, t_end};
                        open = true;
                    }
                } else {
                    close();
                    stage_tiles(t, t);
                }
            }
            close();
            if (any_staged) {  // K4's items, and contiguous image ranges of consecutive staged tiles
                for (uint64_t k = 0; k < nrec; k++) {
                    const uint32_t rt = rec[4 * k];
                    if (!flags[rt]) continue;
                    const uint32_t lo = rec[4 * k + 2], len = rec[4 * k + 1];
                    if (P <= kTileBytes) {
                        items[n_items++] = StageItem{rt, lo};
                    } else {  // the anchor's record covers the whole page: one item per 64 KiB slice
                        for (uint32_t j = 0; (uint64_t)j * kTileBytes < len; j++)
                            items[n_items++] = StageItem{rt + j, lo + j * kTileBytes};
                    }
                    if (!staged.empty() && staged.back().second == lo) staged.back().second += len;
                    else staged.emplace_back(lo, lo + len);
                }
            }
        }
        // ---- execute on copy stream i mod S ----
        cudaStream_t cs = c->copy[i % S];
        if (i == 0) drain0 = Clock::now();
        if (trace) host_enq[i] = ns_since(host0) * 1e-6;
        // Packs run one at a time on their own stream (two concurrent packs,
        // 16 CTAs, overflowed the SMs K1 leaves free and pushed the running
        // scan into a second wave: 0.1 -> 0.2 ms on C2's last group), after
        // K2(i) and once slot i mod S is drained; the copy streams then carry
        // only D2Hs.  The drains share one host link, so serialising the packs
        // costs nothing.
        pks[i] = c->ev();
        pke[i] = c->ev();
        CUDA_TRY(c, cudaStreamWaitEvent(c->packs, tot[i], 0));
        uint64_t chunk_stored = T.image_bytes;
        if (coded && T.n_present) {
            // f4, per SUB-chunk of <= kCodecSub bytes of pages (so the link starts
            // after the first 256 MiB is coded, not the whole chunk): KA (stored
            // length + presence masks per page), KB (slot offsets from the
            // sub-chunk's slot base, stored-length table entries, sub total and
            // PRESENT count -> mapped host), then KC encodes the sub-chunk into
            // slot i mod NS (the first one after that slot's previous drain) and
            // its D2H follows on the chunk's copy stream.  All kernels on the
            // packs stream, in order (KC(i - NS) is done with the scratch before
            // KA(i) overwrites it); the host waits for each KB to size the D2H.
            uint32_t *x = c->cx_scratch[i % NS];
            uint32_t *plan = x, *off = x + c->cx_pages, *masks = x + 2 * c->cx_pages;
            const uint64_t npg = ch.page_end - ch.page_begin;
            static const uint64_t sub_bytes_cfg = [] {  // GCR_CODEC_SUB_MB: tests exercise many sub-chunks
                const char *e = std::getenv("GCR_CODEC_SUB_MB");
                return e ? std::strtoull(e, nullptr, 0) << 20 : kCodecSub;
            }();
            const uint64_t sub_pages = std::max<uint64_t>(1, sub_bytes_cfg / P);
            // the first chunk ramps its sub-chunks up (32, 64, 128 MiB, then the
            // configured size): the link starts after 32 MiB is coded, not 256
            uint64_t ramp_pages = i == 0 ? std::max<uint64_t>(1, std::min<uint64_t>(kCodecSubFirst, sub_bytes_cfg) / P)
                                         : sub_pages;
            uint64_t slot_base = 0, pres_base = present_base;
            for (uint64_t p0 = 0, step = ramp_pages; p0 < npg; p0 += step, step = std::min(2 * step, sub_pages)) {
                const uint32_t n = (uint32_t)std::min(step, npg - p0);
                cudaEvent_t ca = c->ev(), kb = c->ev(), kc = c->ev();
                CUDA_TRY(c, cudaEventRecord(ca, c->packs));
                LAUNCH_TRY(c, launch_codec_plan(c->allocs_d, c->page_alloc, c->cls, ch.page_begin + p0, n, P, c->lg,
                                                plan + p0, masks + 32 * p0, off + p0, c->n_sms, c->packs));
                LAUNCH_TRY(c, launch_codec_offsets(plan + p0, n, off + p0, c->stored_d, pres_base, slot_base,
                                                   c->ctot_map, c->packs));
                CUDA_TRY(c, cudaEventRecord(kb, c->packs));
                if (p0 == 0) {
                    if (i >= NS) CUDA_TRY(c, cudaStreamWaitEvent(c->packs, dde[i - NS], 0));
                    CUDA_TRY(c, cudaEventRecord(pks[i], c->packs));
                }
                LAUNCH_TRY(c, launch_codec_encode(c->allocs_d, c->page_alloc, c->cls, ch.page_begin + p0, n, P, c->lg,
                                                  plan + p0, off + p0, masks + 32 * p0, c->slots[i % NS], c->n_sms,
                                                  c->packs));
                CUDA_TRY(c, cudaEventRecord(kc, c->packs));
                codec_ev.emplace_back(ca, kc);  // KA + KB + KC of the sub-chunk
                CUDA_TRY(c, cudaEventSynchronize(kb));
                const unsigned long long sub_bytes = reinterpret_cast<volatile unsigned long long *>(c->ctot_h)[0];
                const unsigned long long sub_present = reinterpret_cast<volatile unsigned long long *>(c->ctot_h)[1];
                if (sub_bytes) {
                    CUDA_TRY(c, cudaStreamWaitEvent(cs, kc, 0));
                    CUDA_TRY(c, cudaMemcpyAsync(img->data + base + slot_base, c->slots[i % NS] + slot_base, sub_bytes,
                                                cudaMemcpyDeviceToHost, cs));
                }
                if (trace) {
                    cudaEvent_t e = c->ev();
                    CUDA_TRY(c, cudaEventRecord(e, cs));
                    subs.push_back(SubTrace{i, ca, kb, kc, e, ns_since(host0) * 1e-6});
                }
                slot_base += sub_bytes;
                pres_base += sub_present;
            }
            chunk_stored = slot_base;
            staged_bytes += slot_base;
            if (chunk_stored > T.image_bytes || pres_base != n_present)
                return fail(c, GCR_E_CUDA, "checkpoint: coded chunk inconsistent with its pages");
        } else if (coded || isp) {  // f1: K1 itself writes the chunk's pages into the image
            CUDA_TRY(c, cudaEventRecord(pks[i], c->packs));
            if (isp) staged_bytes += T.image_bytes;
        } else if (any_staged) {  // slot i mod NS was last drained by chunk i - NS
            if (i >= NS) CUDA_TRY(c, cudaStreamWaitEvent(c->packs, dde[i - NS], 0));
            CUDA_TRY(c, cudaEventRecord(pks[i], c->packs));
            // narrowed to the SMs K1 leaves free while the scan's last chunk is unpublished
            LAUNCH_TRY(c, launch_pack(c->allocs_d, c->tile_alloc, c->cls, ch.tile_begin, P, c->lg, c->slots[i % NS],
                                      c->stage_map + ch.tile_begin, n_items, c->n_sms, scan_free,
                                      sp.chunk_done + (nch - 1),
                                      sp.epoch, c->chunk_sync_d + 2 * std::max<size_t>(nch, 1) + i, c->packs));
        } else {
            CUDA_TRY(c, cudaEventRecord(pks[i], c->packs));
        }
        CUDA_TRY(c, cudaEventRecord(pke[i], c->packs));
        CUDA_TRY(c, cudaStreamWaitEvent(cs, pke[i], 0));
        for (const auto &rg : staged) {
            CUDA_TRY(c, cudaMemcpyAsync(img->data + base + rg.first, c->slots[i % NS] + rg.first, rg.second - rg.first,
                                        cudaMemcpyDeviceToHost, cs));
            staged_bytes += rg.second - rg.first;
        }
        for (const Run &rn : direct) {
            CUDA_TRY(c, cudaMemcpyAsync(img->data + base + rn.off, reinterpret_cast<const void *>(rn.src), rn.bytes,
                                        cudaMemcpyDeviceToHost, cs));
            direct_bytes += rn.bytes;
        }
        // the digests of every kDigestChunks chunks in one DMA (one small DMA per
        // chunk cost ~10% of the drain at 1% dirty)
        if (i + 1 - dg0 == kDigestChunks || i + 1 == nch) {
            const uint64_t pb = c->chunks[dg0].page_begin, pe = ch.page_end;
            if (pe > pb)
                CUDA_TRY(c, cudaMemcpyAsync(img->digests + pb, Dnew + pb, 4 * (pe - pb), cudaMemcpyDeviceToHost, cs));
            dg0 = i + 1;
            dde[i] = c->ev();
            CUDA_TRY(c, cudaEventRecord(dde[i], cs));
            if (pe > pb) dbatch.push_back(DigestBatch{pb, pe, dde[i]});
        } else {
            dde[i] = c->ev();
            CUDA_TRY(c, cudaEventRecord(dde[i], cs));
        }
        {
            gcr_status cs_ = crc_batches(false);  // digests that already landed (the host is idle here)
            if (cs_ != GCR_OK) return cs_;
        }
        base += chunk_stored;
    }
    if (direct_bytes + staged_bytes != base) return fail(c, GCR_E_CUDA, "checkpoint: drain plan does not cover the image");
    st.direct_bytes = direct_bytes;
    c->pool.shrink(img->data, img->data_cap, base);  // the tail is free before the pagemap is allocated
    img->data_cap = base;
    if (coded) {  // the stored-length table (KB wrote it chunk by chunk on the packs stream)
        c->pool.shrink(img->stored, img->stored_cap, 4 * n_present);
        img->stored_cap = 4 * n_present;
        cudaEvent_t e = c->ev();
        CUDA_TRY(c, cudaEventRecord(e, c->packs));
        CUDA_TRY(c, cudaStreamWaitEvent(c->compute, e, 0));
        if (n_present)
            CUDA_TRY(c, cudaMemcpyAsync(img->stored, c->stored_d, 4 * n_present, cudaMemcpyDeviceToHost, c->compute));
    }
    // K3 pagemap over all pages (maximal runs, independent of chunking): every
    // class is final once the last K1 (same stream) has ended.
    NvtxScope nvtx_finish("gcr.checkpoint.pagemap_meta");
    auto pm0 = c->ev(), pm1 = c->ev();
    CUDA_TRY(c, cudaEventRecord(pm0, c->compute));
    LAUNCH_TRY(c, launch_pagemap_count(c->cls, c->n_pages, c->pm_blk_cnt, c->pm_blk_off, c->nent_map, c->compute));
    cudaEvent_t pmc = c->ev();
    CUDA_TRY(c, cudaEventRecord(pmc, c->compute));
    CUDA_TRY(c, cudaEventSynchronize(pmc));
    const uint64_t ne = *reinterpret_cast<volatile unsigned long long *>(c->nent_h);
    img->pagemap_cap = sizeof(gcr_pagemap_entry) * ne;
    img->pagemap = static_cast<gcr_pagemap_entry *>(c->pool.alloc(img->pagemap_cap));
    if (!img->pagemap) return fail(c, GCR_E_NOMEM, "checkpoint: pinned pagemap allocation failed");
    LAUNCH_TRY(c, launch_pagemap_write(c->allocs_d, c->page_alloc, c->cls, c->n_pages, c->lg, c->pm_blk_off,
                                       c->run_start, ne, c->entries_d, c->compute));
    CUDA_TRY(c, cudaEventRecord(pm1, c->compute));
    if (ne) CUDA_TRY(c, cudaMemcpyAsync(img->pagemap, c->entries_d, img->pagemap_cap, cudaMemcpyDeviceToHost, c->compute));
    for (size_t s = 0; s < S; s++) {
        cudaEvent_t e = c->ev();
        CUDA_TRY(c, cudaEventRecord(e, c->copy[s]));
        CUDA_TRY(c, cudaStreamWaitEvent(c->compute, e, 0));
    }
    if (isp) {  // f1: the kernel's own consistency: no wait timed out, no list overflowed, bases add up
        CUDA_TRY(c, cudaMemcpyAsync(c->misc_h, c->isp_err, 8, cudaMemcpyDeviceToHost, c->compute));
        CUDA_TRY(c, cudaMemcpyAsync(c->misc_h + 3, c->isp_base + nch, 8, cudaMemcpyDeviceToHost, c->compute));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->compute));
    st.drain_ns = ns_since(drain0);
    if (isp && (c->misc_h[0] != 0 || (nch && c->misc_h[3] != base)))
        return fail(c, GCR_E_CUDA, "checkpoint: in-scan pack failed (error word " + std::to_string(c->misc_h[0]) +
                                       ": 1 CTA prefix / 2 CTA aggregates / 3 chunk base wait timed out, 4 list "
                                       "overflow; base " + std::to_string(c->misc_h[3]) + " vs " + std::to_string(base) + ")");
    const double host_synced = ns_since(host0) * 1e-6;

    // stats from the events
    float ms;
    st.scan_dev_ns = 0;
    st.pack_dev_ns = 0;
    CUDA_TRY(c, cudaEventElapsedTime(&ms, k1s, k1m));
    st.scan_dev_ns = (uint64_t)(ms * 1e6);
    for (size_t i = 0; i < nch; i++) {
        CUDA_TRY(c, cudaEventElapsedTime(&ms, pks[i], pke[i]));
        st.pack_dev_ns += (uint64_t)(ms * 1e6);
    }
    CUDA_TRY(c, cudaEventElapsedTime(&ms, pm0, pm1));
    st.compact_dev_ns = (uint64_t)(ms * 1e6);
    st.codec_dev_ns = 0;
    for (const auto &ce : codec_ev) {
        CUDA_TRY(c, cudaEventElapsedTime(&ms, ce.first, ce.second));
        st.codec_dev_ns += (uint64_t)(ms * 1e6);
    }
    if (coded) st.pack_dev_ns = 0;  // no K4 pack: the codec kernels (codec_dev_ns) staged the data
    st.present_raw_bytes = raw_present;
    const double host_stats = ns_since(host0) * 1e-6;
    if (trace) {  // GCR_TRACE=1: per-chunk timeline (ms from the checkpoint's first event) on stderr
        auto rel = [&](cudaEvent_t e) {
            float m = 0;
            cudaEventElapsedTime(&m, t0, e);
            return m;
        };
        std::fprintf(stderr, "{\"gcr_trace\": \"checkpoint\", \"scans\": [[0, %zu, %.3f, %.3f]", nch, rel(k1s),
                     rel(k1m));
        std::fprintf(stderr, "], \"chunks\": [");
        for (size_t i = 0; i < nch; i++)
            std::fprintf(stderr, "%s[%.3f, %.3f, %.3f, %.3f, %.3f, %.3f, %.3f]", i ? ", " : "", rel(k2s[i]),
                         rel(tot[i]), rel(pks[i]), rel(pke[i]), rel(dde[i]), host_seen[i], host_enq[i]);
        std::fprintf(stderr, "], \"subs\": [");
        for (size_t k = 0; k < subs.size(); k++)
            std::fprintf(stderr, "%s[%zu, %.3f, %.3f, %.3f, %.3f, %.3f]", k ? ", " : "", subs[k].chunk, rel(subs[k].ka),
                         rel(subs[k].kb), rel(subs[k].kc), rel(subs[k].d2h), subs[k].host_enq);
        std::fprintf(stderr, "], \"pagemap\": [%.3f, %.3f], \"fields\": {\"scans\": \"chunk_lo chunk_hi k1_start "
                             "k1_end\", \"chunks\": \"k2_start k2_end pack_start pack_end d2h_end host_saw_k2 host_enqueued\", "
                             "\"subs\": \"chunk codec_start kb_done kc_done d2h_done host_enqueued\"}}\n",
                     rel(pm0), rel(pm1));
    }
    st.scan_launches = 1;
    st.scan_bytes = R;
    st.pages_scanned = c->n_pages;
    st.pages_zero = n_zero;
    st.pages_parent = n_parent;
    st.pages_written = n_present;
    st.image_bytes = base;
    st.n_entries = ne;

    // image model
    gcr_image_hdr &h = img->hdr;
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.page_size = P;
    h.generation = c->next_gen;
    h.parent_generation = mode == GCR_INCREMENTAL ? c->parent_gen : 0;
    h.n_allocs = (uint32_t)c->reg.size();
    h.flags = (mode == GCR_INCREMENTAL ? 1u : 0u) | (coded ? 2u : 0u);
    h.n_pages = c->n_pages;
    h.n_present = n_present;
    h.n_zero = n_zero;
    h.n_parent = n_parent;
    h.n_entries = ne;
    h.image_bytes = base;
    h.reserved = 0;
    img->allocs.clear();
    for (const RegEntry &r : c->reg) img->allocs.push_back(gcr_alloc_rec{r.dptr, r.bytes, r.id, 0});
    const double host_model = ns_since(host0) * 1e-6;
    {
        gcr_status cs_ = crc_batches(true);
        if (cs_ != GCR_OK) return cs_;
    }
    h.meta_crc32c = meta_crc(img, &dreg);
    if (trace)
        std::fprintf(stderr,
                     "{\"gcr_trace\": \"checkpoint_host\", \"synced_ms\": %.3f, \"stats_ms\": %.3f, \"model_ms\": %.3f, "
                     "\"meta_crc_done_ms\": %.3f}\n",
                     host_synced, host_stats, host_model, ns_since(host0) * 1e-6);
    if (n_present + n_zero + n_parent != c->n_pages)
        return fail(c, GCR_E_CUDA, "checkpoint: class counts do not cover every page");
    c->next_gen++;
    c->parent_idx = cur;
    c->parent_gen = h.generation;
    c->have_parent = true;
    return GCR_OK;
}

gcr_status gcr_checkpoint(gcr_ctx *c, gcr_mode mode, gcr_image **out) {
    NvtxScope nvtx_("gcr.checkpoint");
    if (!c) return GCR_E_INVAL;
    if (!out) return fail(c, GCR_E_INVAL, "checkpoint: out is NULL");
    *out = nullptr;
    if (c->phase != GCR_LOCKED) return fail(c, GCR_E_STATE, "checkpoint: not LOCKED");
    if (mode != GCR_FULL && mode != GCR_INCREMENTAL) return fail(c, GCR_E_INVAL, "checkpoint: bad mode");
    if (c->reg.empty()) return fail(c, GCR_E_INVAL, "checkpoint: no registered allocation");
    if (mode == GCR_INCREMENTAL && !c->have_parent)
        return fail(c, GCR_E_CHAIN, "checkpoint: INCREMENTAL without a parent digest state (R-8)");
    auto t0 = Clock::now();
    CUDA_TRY(c, cudaSetDevice(c->device));
    gcr_status s = build_layout(c);
    if (s != GCR_OK) return s;
    s = fence_caller_work(c);
    if (s != GCR_OK) return s;
    gcr_image *img = new (std::nothrow) gcr_image;
    if (!img) return fail(c, GCR_E_NOMEM, "checkpoint: out of host memory");
    img->ctx = c;
    const bool had_parent = c->have_parent;
    const int pidx = c->parent_idx;
    const uint64_t pgen = c->parent_gen;
    s = checkpoint_impl(c, mode, img);
    if (s != GCR_OK) {
        sync_all(c);
        // re-arm the per-launch device state the kernels leave zeroed on success
        cudaMemset(c->tile_info, 0, sizeof(TileInfo) * c->n_tiles);
        {
            const uint64_t ns = std::max<size_t>(c->chunks.size(), 1);
            cudaMemset(c->chunk_sync_d, 0, 3 * 4 * ns);
            cudaMemset(c->fold_slots, 0, 8 * scan_workers(c->n_sms, 0) * ns);
        }
        cudaGetLastError();
        image_free_buffers(img);
        delete img;
        c->have_parent = had_parent;  // failure atomicity
        c->parent_idx = pidx;
        c->parent_gen = pgen;
        return s;
    }
    c->images.push_back(img);
    c->phase = GCR_CHECKPOINTED;
    c->stats.checkpoint_ns = ns_since(t0);
    c->last_ckpt = img;
    c->prev_have_parent = had_parent;
    c->prev_parent_idx = pidx;
    c->prev_parent_gen = pgen;
    c->prev_next_gen = c->next_gen - 1;
    *out = img;
    return GCR_OK;
}

gcr_status gcr_checkpoint_abort(gcr_ctx *c, gcr_image *img) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_CHECKPOINTED) return fail(c, GCR_E_STATE, "checkpoint_abort: not CHECKPOINTED");
    if (!img || img != c->last_ckpt)
        return fail(c, GCR_E_INVAL, "checkpoint_abort: not the image of the ctx's last checkpoint");
    cudaSetDevice(c->device);
    sync_all(c);
    destroy_image(c, img);
    c->last_ckpt = nullptr;
    // the digest table the checkpoint wrote was the non-parent one: the old
    // parent table is intact, so the previous state is restored exactly
    c->have_parent = c->prev_have_parent;
    c->parent_idx = c->prev_parent_idx;
    c->parent_gen = c->prev_parent_gen;
    c->next_gen = c->prev_next_gen;
    c->phase = GCR_LOCKED;
    return GCR_OK;
}

static gcr_status ensure_desc(gcr_ctx *c, uint64_t bytes) {
    if (bytes <= c->desc_cap) return GCR_OK;
    uint64_t cap = std::max<uint64_t>(bytes, 1ull << 20);
    if (c->desc_d) cudaFree(c->desc_d);
    if (c->desc_h) cudaFreeHost(c->desc_h);
    c->desc_d = nullptr;
    c->desc_h = nullptr;
    c->desc_cap = 0;
    CUDA_TRY(c, cudaMalloc(&c->desc_d, cap));
    CUDA_TRY(c, cudaHostAlloc(&c->desc_h, cap, cudaHostAllocDefault));
    c->desc_cap = cap;
    return GCR_OK;
}

static gcr_status restore_impl(gcr_ctx *c, gcr_image *const *chain, uint32_t n, bool &writes_began) {
    if (c->phase != GCR_LOCKED && c->phase != GCR_CHECKPOINTED && c->phase != GCR_RELEASED)
        return fail(c, GCR_E_STATE, "restore: not locked");
    if (!chain || n == 0) return fail(c, GCR_E_INVAL, "restore: empty chain");
    for (uint32_t k = 0; k < n; k++)
        if (!chain[k] || chain[k]->ctx != c) return fail(c, GCR_E_INVAL, "restore: image of another ctx or NULL");
    auto t0 = Clock::now();
    gcr_stats &st = c->stats;
    // Speculative first H2D (f4 chains): the first staged group of a coded
    // image is its data prefix [0, <= group_max) and lands in region 0 of the
    // staging slots -- not in registered memory -- so it is issued before the
    // host validates and plans (~0.5 ms on C2) and used if the plan agrees.
    // Every failure path below syncs the streams before returning (gcr_restore).
    const uint64_t group_max = c->slots.empty() ? 0 : std::min<uint64_t>(c->cfg.chunk_bytes, kGroupMax);
    uint64_t spec_bytes = 0;
    cudaEvent_t spec_landed = nullptr;
    CUDA_TRY(c, cudaSetDevice(c->device));
    {  // before the speculative H2D: a whole-device fence would wait for it
        const gcr_status fs = fence_caller_work(c);
        if (fs != GCR_OK) return fs;
    }
    if (group_max && (chain[0]->hdr.flags & 2u) && chain[0]->data && chain[0]->hdr.image_bytes &&
        chain[0]->data_cap >= std::min<uint64_t>(chain[0]->hdr.image_bytes, group_max)) {
        spec_bytes = std::min<uint64_t>(chain[0]->hdr.image_bytes, group_max);
        CUDA_TRY(c, cudaMemcpyAsync(c->slots[0], chain[0]->data, spec_bytes, cudaMemcpyHostToDevice, c->copy[0]));
        spec_landed = c->ev_spec;
        CUDA_TRY(c, cudaEventRecord(spec_landed, c->copy[0]));
    }
    // ---- validation, in order: meta CRC, version, layout, chain (c.2 step 1)
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image *im = chain[k];
        if (std::memcmp(im->hdr.magic, kMagic, 8) != 0 || meta_crc(im) != im->hdr.meta_crc32c)
            return fail(c, GCR_E_CORRUPT, "restore: meta_crc32c mismatch");
        if (im->hdr.version != 1 || (im->hdr.flags & ~3u))
            return fail(c, GCR_E_VERSION, "restore: unknown image version or flag bits");
        gcr_status s = check_pagemap(c, im);
        if (s != GCR_OK) return s;
    }
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image *im = chain[k];
        if (im->hdr.page_size != c->cfg.page_size || im->hdr.n_allocs != c->reg.size())
            return fail(c, GCR_E_LAYOUT, "restore: page size or allocation count differs from the registry");
        for (uint32_t a = 0; a < im->hdr.n_allocs; a++)
            if (im->allocs[a].bytes != c->reg[a].bytes)
                return fail(c, GCR_E_LAYOUT, "restore: allocation sizes differ from the registry");
    }
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image_hdr &h = chain[k]->hdr;
        if (k == 0 && ((h.flags & 1u) || h.parent_generation != 0 || h.n_parent != 0))
            return fail(c, GCR_E_CHAIN, "restore: chain must start with a full image");
        if (k > 0 && (!(h.flags & 1u) || h.parent_generation != chain[k - 1]->hdr.generation))
            return fail(c, GCR_E_CHAIN, "restore: parent_generation link broken");
    }
    st.remap_ns = 0;
    writes_began = true;  // from here on a failure leaves the memory content undefined
    if (c->phase == GCR_RELEASED) {  // back the same VAs again, then apply the chain
        const auto r0 = Clock::now();
        for (MemBlock &b : c->blocks) {
            if (b.mapped) continue;
            const CUresult r = map_block(c->device, b);
            if (r != CUDA_SUCCESS)
                return fail(c, r == CUDA_ERROR_OUT_OF_MEMORY ? GCR_E_NOMEM : GCR_E_CUDA,
                            "restore: re-mapping released memory failed (driver error " + std::to_string((int)r) + ")");
        }
        st.remap_ns = ns_since(r0);
        // the phase stays RELEASED (content not valid: unlock refused) until
        // the chain has been applied and verified
    }
    gcr_status s = build_layout(c);
    if (s != GCR_OK) return s;
    c->ev_used = 0;
    const uint32_t P = c->P;
    const uint64_t slot = c->cfg.chunk_bytes;
    const size_t S = c->copy.size();

    // ---- plan every image (host walk of the pagemaps) ----------------------
    // In image-data order, a PRESENT run of at least direct_min_bytes is one
    // DIRECT item (H2D from the pinned image straight into the allocation); a
    // maximal sequence of consecutive shorter runs (contiguous in the image) up
    // to one slot is a STAGED item (one H2D into a staging slot + K6 scatter).
    struct Item {
        bool direct;
        uint64_t img_off, bytes, dst;  // direct: dst device address
        uint64_t d_begin, d_end;       // staged: scatter (or, f4 image, decode) descriptors
        bool decode;                   // f4: the group's pages are stored forms (K-D decodes them)
    };
    struct ImgPlan {
        std::vector<Item> items;
        uint64_t z_begin, z_end;
    };
    const uint64_t direct_min = c->cfg.direct_min_bytes;
    // staged groups (one H2D into a slot + scatter / decode) of at most
    // kGroupMax: the first kernel starts after 64 MiB instead of a whole slot,
    // and the last group's kernel -- the restore's tail -- is short
    std::vector<ImgPlan> plans(n);
    std::vector<ScatterDesc> sdesc;
    std::vector<ZeroDesc> zdesc;
    // f4 decode descriptors (one per PRESENT page of a coded image) are written
    // straight into the pinned descriptor buffer, ahead of the scatter / zero
    // descriptors (a 4 KiB-page C2 image has 364 k of them: building a vector
    // and copying it cost ~10 ms of host time per restore)
    uint64_t n_dec = 0, desc_bound = 0;
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image_hdr &h = chain[k]->hdr;
        if (h.flags & 2u) n_dec += h.n_present;
        else desc_bound += h.n_entries + h.image_bytes / kPieceBytes + h.image_bytes / kGroupMax + 2;
        desc_bound += h.n_entries + h.n_zero * (P / kPieceBytes + 1) + 1;
    }
    s = ensure_desc(c, sizeof(DecodeDesc) * n_dec + sizeof(ScatterDesc) * desc_bound + 64);
    if (s != GCR_OK) return s;
    DecodeDesc *ddh = reinterpret_cast<DecodeDesc *>(c->desc_h);
    uint64_t nd = 0;
    uint64_t h2d_bytes = 0, direct_bytes = 0;
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image *im = chain[k];
        ImgPlan &pl = plans[k];
        pl.z_begin = zdesc.size();
        uint64_t cursor = 0, e = 0, ip = 0;  // ip: ordinal of the next PRESENT page (f4 stored lengths)
        const bool coded = im->hdr.flags & 2u;
        bool group_open = false;
        auto close_group = [&]() {
            if (group_open) pl.items.back().d_end = coded ? nd : sdesc.size();
            group_open = false;
        };
        for (uint32_t a = 0; a < im->hdr.n_allocs; a++) {
            const uint64_t m = pages_of(c->reg[a].bytes, P);
            uint64_t p = 0;
            while (p < m) {
                const gcr_pagemap_entry &pe = im->pagemap[e++];
                const uint64_t last = p + pe.nr_pages;
                uint64_t bytes = (last == m) ? (uint64_t)(pe.nr_pages - 1) * P + page_len(c->reg[a].bytes, P, m - 1)
                                             : (uint64_t)pe.nr_pages * P;
                uint64_t dst = c->reg[a].dptr + p * P;  // remapped by allocation index (R-14)
                if (pe.flags == GCR_PE_PRESENT && coded) {
                    // f4: every page's stored form goes through a slot; groups of
                    // consecutive stored forms up to one slot, one decode
                    // descriptor per page
                    const uint64_t base_a = c->reg[a].dptr;
                    const uint32_t tail = (uint32_t)page_len(c->reg[a].bytes, P, m - 1);
                    for (uint64_t q = p; q < last; q++) {
                        const uint32_t L = q == m - 1 ? tail : P, sl = im->stored[ip++];
                        if (group_open && pl.items.back().bytes + sl > group_max) close_group();
                        if (!group_open) {
                            pl.items.push_back(Item{false, cursor, 0, 0, nd, 0, true});
                            group_open = true;
                        }
                        Item &g = pl.items.back();
                        ddh[nd++] = DecodeDesc{base_a + q * P, cursor - g.img_off, L, sl};
                        g.bytes += sl;
                        cursor += sl;
                    }
                } else if (pe.flags == GCR_PE_PRESENT) {
                    if (bytes >= direct_min) {
                        close_group();
                        while (bytes) {  // pieces of at most one slot keep the copy streams busy
                            const uint64_t piece = std::min(bytes, slot);
                            pl.items.push_back(Item{true, cursor, piece, dst, 0, 0, false});
                            direct_bytes += piece;
                            dst += piece;
                            cursor += piece;
                            bytes -= piece;
                        }
                    } else {
                        while (bytes) {
                            // a group closes when full: runs are cut across groups as needed (a
                            // test against the whole remaining run closed a group per 1 MiB piece
                            // of any run longer than a group)
                            if (group_open && pl.items.back().bytes >= group_max) close_group();
                            if (!group_open) {
                                pl.items.push_back(Item{false, cursor, 0, 0, sdesc.size(), 0, false});
                                group_open = true;
                            }
                            Item &g = pl.items.back();
                            const uint64_t piece = std::min(std::min(bytes, kPieceBytes), group_max - g.bytes);
                            sdesc.push_back(ScatterDesc{dst, cursor - g.img_off, piece});
                            g.bytes += piece;
                            dst += piece;
                            cursor += piece;
                            bytes -= piece;
                        }
                    }
                } else if (pe.flags == GCR_PE_ZERO) {
                    while (bytes) {
                        const uint64_t piece = std::min(bytes, kPieceBytes);
                        zdesc.push_back(ZeroDesc{dst, piece});
                        dst += piece;
                        bytes -= piece;
                    }
                }
                p = last;
            }
        }
        close_group();
        pl.z_end = zdesc.size();
        h2d_bytes += im->hdr.image_bytes;
    }
    const uint64_t sbytes = sizeof(ScatterDesc) * sdesc.size(), zbytes = sizeof(ZeroDesc) * zdesc.size();
    const uint64_t dbytes = sizeof(DecodeDesc) * nd;  // already in place at the buffer's start
    if (nd != n_dec || dbytes + sbytes + zbytes + 64 > c->desc_cap)
        return fail(c, GCR_E_CUDA, "restore: descriptor plan exceeds its bound");
    std::memcpy(c->desc_h + dbytes, sdesc.data(), sbytes);
    std::memcpy(c->desc_h + dbytes + sbytes, zdesc.data(), zbytes);
    const DecodeDesc *dd = reinterpret_cast<const DecodeDesc *>(c->desc_d);
    const ScatterDesc *sd = reinterpret_cast<const ScatterDesc *>(c->desc_d + dbytes);
    const ZeroDesc *zd = reinterpret_cast<const ZeroDesc *>(c->desc_d + dbytes + sbytes);
    CUDA_TRY(c, cudaMemcpyAsync(c->desc_d, c->desc_h, dbytes + sbytes + zbytes, cudaMemcpyHostToDevice, c->compute));

    // ---- apply the chain ----------------------------------------------------
    // Staged groups land in a ring of group_max-sized REGIONS carved out of the
    // staging slots (2 x 1 GiB = 32 regions of 64 MiB by default).  The H2Ds
    // alternate over the copy streams; every scatter / decode runs on the packs
    // stream once its group's H2D is done, and the H2D into a region waits only
    // for the kernel that last read that region.  (Group j's H2D used to follow
    // group j - S's kernel on the same copy stream: the link idled for one
    // decode every S groups, ~0.9 ms of a C2 f4 restore.)  A ZERO fill goes to
    // the packs stream at the image's start, beside the first H2D.
    std::vector<cudaEvent_t> sc0, sc1, dc0, dc1;  // scatter+zero / f4 decode spans
    const uint64_t regions_per_slot = std::max<uint64_t>(1, slot / group_max);
    const uint64_t NR = regions_per_slot * c->slots.size();
    std::vector<cudaEvent_t> region_free(NR, nullptr);  // kernel that last read the region
    uint64_t q = 0;                                      // staged groups issued (all images)
    bool spec_used = false;
    static const bool trace = std::getenv("GCR_TRACE") != nullptr;
    const bool ring = [] {  // read per call (tests flip it)
        const char *e = std::getenv("GCR_RESTORE_RING");
        return !(e && e[0] == '0');
    }();
    struct TraceGroup {  // GCR_TRACE: per staged group
        cudaEvent_t issued, landed, k0, k1;
        uint64_t bytes;
    };
    std::vector<TraceGroup> tg;
    cudaEvent_t rt0 = c->ev();
    CUDA_TRY(c, cudaEventRecord(rt0, c->compute));
    auto h2d0 = Clock::now();
    for (uint32_t k = 0; k < n; k++) {
        const gcr_image *im = chain[k];
        const ImgPlan &pl = plans[k];
        cudaEvent_t start = c->ev();
        CUDA_TRY(c, cudaEventRecord(start, c->compute));
        for (size_t i = 0; i < S; i++) CUDA_TRY(c, cudaStreamWaitEvent(c->copy[i], start, 0));
        CUDA_TRY(c, cudaStreamWaitEvent(c->packs, start, 0));
        if (pl.z_end > pl.z_begin) {  // disjoint from this image's PRESENT pages: beside its H2Ds
            cudaEvent_t a = c->ev(), b = c->ev();
            CUDA_TRY(c, cudaEventRecord(a, c->packs));
            LAUNCH_TRY(c, launch_zero_fill(zd + pl.z_begin, pl.z_end - pl.z_begin, c->n_sms, c->packs));
            CUDA_TRY(c, cudaEventRecord(b, c->packs));
            sc0.push_back(a);
            sc1.push_back(b);
        }
        for (size_t j = 0; j < pl.items.size(); j++) {
            const Item &it = pl.items[j];
            cudaStream_t cs = c->copy[j % S];
            if (it.direct) {
                CUDA_TRY(c, cudaMemcpyAsync(reinterpret_cast<void *>(it.dst), im->data + it.img_off, it.bytes,
                                            cudaMemcpyHostToDevice, cs));
                continue;
            }
            // GCR_RESTORE_RING=0 (A/B knob): round 2's first layout -- group j in
            // slot j mod S, its kernel on its own copy stream
            const uint64_t r = ring ? q++ % NR : j % S;
            uint8_t *reg = ring ? c->slots[r / regions_per_slot] + (r % regions_per_slot) * group_max : c->slots[j % S];
            cudaStream_t ks = ring ? c->packs : cs;
            if (ring && region_free[r]) CUDA_TRY(c, cudaStreamWaitEvent(cs, region_free[r], 0));
            cudaEvent_t issued = nullptr;
            if (trace) {
                issued = c->ev();
                CUDA_TRY(c, cudaEventRecord(issued, cs));
            }
            cudaEvent_t landed, a = c->ev(), b = c->ev();
            if (k == 0 && it.img_off == 0 && it.bytes <= spec_bytes && reg == c->slots[0]) {
                landed = spec_landed;  // the speculative prefix H2D already brought this group
                spec_used = true;
                if (!ring) CUDA_TRY(c, cudaStreamWaitEvent(ks, landed, 0));
            } else {
                CUDA_TRY(c, cudaMemcpyAsync(reg, im->data + it.img_off, it.bytes, cudaMemcpyHostToDevice, cs));
                landed = c->ev();
                CUDA_TRY(c, cudaEventRecord(landed, cs));
            }
            if (trace) tg.push_back(TraceGroup{issued, landed, a, b, it.bytes});
            if (ring) CUDA_TRY(c, cudaStreamWaitEvent(ks, landed, 0));
            CUDA_TRY(c, cudaEventRecord(a, ks));
            if (it.decode)
                LAUNCH_TRY(c, launch_codec_decode(dd + it.d_begin, it.d_end - it.d_begin, reg, P, c->n_sms, ks));
            else
                LAUNCH_TRY(c, launch_scatter(sd + it.d_begin, it.d_end - it.d_begin, reg, c->n_sms, ks));
            CUDA_TRY(c, cudaEventRecord(b, ks));
            region_free[r] = b;
            (it.decode ? dc0 : sc0).push_back(a);
            (it.decode ? dc1 : sc1).push_back(b);
        }
        for (size_t i = 0; i < S; i++) {
            cudaEvent_t e = c->ev();
            CUDA_TRY(c, cudaEventRecord(e, c->copy[i]));
            CUDA_TRY(c, cudaStreamWaitEvent(c->compute, e, 0));
        }
        {
            cudaEvent_t e = c->ev();
            CUDA_TRY(c, cudaEventRecord(e, c->packs));
            CUDA_TRY(c, cudaStreamWaitEvent(c->compute, e, 0));
        }
    }
    st.restore_direct_bytes = direct_bytes;
    // ---- verify: recompute every digest and compare with D_k (R-11) ---------
    NvtxScope nvtx_verify("gcr.restore.verify");
    const gcr_image *last = chain[n - 1];
    const int scratch = c->have_parent ? 1 - c->parent_idx : 0;
    CUDA_TRY(c, cudaMemcpyAsync(c->D[scratch], last->digests, 4 * c->n_pages, cudaMemcpyHostToDevice, c->compute));
    cudaEvent_t v0 = c->ev(), v1 = c->ev();
    uint64_t verify_launches = 0;
    if (c->cfg.verify) {
        CUDA_TRY(c, cudaMemsetAsync(c->misc_d + 1, 0, 8, c->compute));
        CUDA_TRY(c, cudaMemsetAsync(c->misc_d + 2, 0xFF, 8, c->compute));
        ScanParams sp{};
        sp.allocs = c->allocs_d;
        sp.n_allocs = (uint32_t)c->allocs_h.size();
        sp.fold = c->fold;
        const size_t nch = c->chunks.size();
        sp.chunk_rows = c->chunk_rows_d + nch + 1;  // one chunk: every real row
        sp.chunk_groups = c->chunk_groups_d ? c->chunk_groups_d + nch + 1 : nullptr;
        sp.grp_pf_block = grp_prefetch_block();
        sp.n_chunks = 1;
        sp.epoch = ++c->epoch ? c->epoch : ++c->epoch;
        sp.chunk_arrive = c->chunk_sync_d;
        sp.chunk_done = c->chunk_sync_d + std::max<size_t>(nch, 1);
        sp.workers = scan_workers(c->n_sms, 0);  // nothing runs beside the verify: every SM
        sp.prefetch = scan_prefetch_bytes();
        sp.page_size = P;
        sp.log2_page = c->lg;
        sp.z_page = c->z_page;
        sp.mode = kScanVerify;
        sp.d_ref = c->D[scratch];
        sp.verify_count = c->misc_d + 1;
        sp.first_bad = c->misc_d + 2;
        sp.tables = c->tables_d;
        set_basis(c, sp);
        // GCR_SCAN_TIMES=1: per-warp globaltimer stamps of this verify launch
        // (entry, tables staged, first rows loaded, chunk done, exit),
        // summarised on stderr relative to the earliest entry (diagnostics)
        static const bool stamps = std::getenv("GCR_SCAN_TIMES") != nullptr;
        unsigned long long *wt = nullptr;
        const uint64_t SW = kScanStamps;
        if (stamps && cudaMalloc(&wt, 8 * SW * sp.workers) == cudaSuccess) {
            cudaMemsetAsync(wt, 0, 8 * SW * sp.workers, c->compute);
            sp.warp_times = wt;
        }
        CUDA_TRY(c, cudaEventRecord(v0, c->compute));
        LAUNCH_TRY(c, launch_scan(sp, c->n_sms, c->compute));
        CUDA_TRY(c, cudaEventRecord(v1, c->compute));
        if (wt) {
            std::vector<unsigned long long> h(SW * sp.workers);
            cudaMemcpy(h.data(), wt, 8 * SW * sp.workers, cudaMemcpyDeviceToHost);
            cudaFree(wt);
            unsigned long long tw0 = ~0ull;
            for (uint64_t w = 0; w < sp.workers; w++) tw0 = std::min(tw0, h[SW * w]);
            auto pct = [](std::vector<double> v, double qq) {
                std::sort(v.begin(), v.end());
                return v[(size_t)(qq * (v.size() - 1))];
            };
            float kms = 0;
            cudaEventSynchronize(v1);
            cudaEventElapsedTime(&kms, v0, v1);
            std::fprintf(stderr, "{\"gcr_scan_times\": \"verify\", \"warps\": %llu, \"event_us\": %.1f",
                         (unsigned long long)sp.workers, kms * 1e3);
            const char *names[5] = {"entry_us", "staged_us", "first_rows_us", "chunk0_us", "exit_us"};
            for (uint64_t k = 0; k < 5; k++) {
                std::vector<double> v;
                for (uint64_t w = 0; w < sp.workers; w++)
                    if (h[SW * w + k]) v.push_back((h[SW * w + k] - tw0) * 1e-3);
                if (v.empty()) continue;
                std::fprintf(stderr, ", \"%s\": [%.2f, %.2f, %.2f, %.2f, %.2f]", names[k], pct(v, 0), pct(v, 0.1),
                             pct(v, 0.5), pct(v, 0.9), pct(v, 1));
            }
            // per-SM mean exit time: is the tail a few slow SMs or spread evenly?
            {
                std::vector<double> sum(256, 0.0), cnt(256, 0.0);
                for (uint64_t w = 0; w < sp.workers; w++) {
                    const uint64_t sid = h[SW * w + 5] & 255u;
                    sum[sid] += (h[SW * w + 4] - tw0) * 1e-3;
                    cnt[sid] += 1;
                }
                std::vector<std::pair<double, int>> sms;
                for (int i = 0; i < 256; i++)
                    if (cnt[i] > 0) sms.emplace_back(sum[i] / cnt[i], i);
                std::sort(sms.begin(), sms.end());
                std::fprintf(stderr, ", \"sm_exit_mean_us\": {\"fastest\": [%d, %.2f], \"median\": %.2f, \"slowest\": [",
                             sms.front().second, sms.front().first, sms[sms.size() / 2].first);
                for (size_t i = sms.size() >= 8 ? sms.size() - 8 : 0; i < sms.size(); i++)
                    std::fprintf(stderr, "%s[%d, %.2f]", i + 8 == sms.size() || (sms.size() < 8 && i == 0) ? "" : ", ",
                                 sms[i].second, sms[i].first);
                std::fprintf(stderr, "]}");
            }
            {  // mean exit time by warp index within the CTA: is the tail a fixed scheduling order?
                const uint64_t wpc = scan_warps_per_cta();
                std::vector<double> sum(wpc, 0.0), cnt(wpc, 0.0);
                for (uint64_t w = 0; w < sp.workers; w++) {
                    sum[w % wpc] += (h[SW * w + 4] - tw0) * 1e-3;
                    cnt[w % wpc] += 1;
                }
                std::fprintf(stderr, ", \"exit_mean_us_by_warp_in_cta\": [");
                for (uint64_t i = 0; i < wpc; i++)
                    std::fprintf(stderr, "%s%.2f", i ? ", " : "", cnt[i] ? sum[i] / cnt[i] : 0.0);
                std::fprintf(stderr, "]");
            }
            std::fprintf(stderr, "}\n");
        }
        CUDA_TRY(c, cudaMemcpyAsync(c->misc_h + 1, c->misc_d + 1, 16, cudaMemcpyDeviceToHost, c->compute));
        verify_launches = 1;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->compute));
    st.restore_h2d_ns = ns_since(h2d0);
    float ms;
    if (trace) {  // GCR_TRACE=1: per-group restore timeline (ms from the first H2D's enqueue point) on stderr
        auto rel = [&](cudaEvent_t e) {
            float m = 0;
            cudaEventElapsedTime(&m, rt0, e);
            return m;
        };
        std::fprintf(stderr, "{\"gcr_trace\": \"restore\", \"groups\": [");
        for (size_t g = 0; g < tg.size(); g++)
            std::fprintf(stderr, "%s[%.3f, %.3f, %.3f, %.3f, %llu]", g ? ", " : "", rel(tg[g].issued), rel(tg[g].landed),
                         rel(tg[g].k0), rel(tg[g].k1), (unsigned long long)tg[g].bytes);
        std::fprintf(stderr, "], \"verify\": [%.3f, %.3f], \"host_ms\": %.3f, \"speculative_prefix\": %d, \"fields\": {\"groups\": \"h2d_enqueued "
                             "h2d_landed kernel_start kernel_end bytes\"}}\n",
                     c->cfg.verify ? rel(v0) : 0.f, c->cfg.verify ? rel(v1) : 0.f, ns_since(h2d0) * 1e-6, (int)spec_used);
    }
    st.scatter_dev_ns = 0;
    for (size_t i = 0; i < sc0.size(); i++) {
        CUDA_TRY(c, cudaEventElapsedTime(&ms, sc0[i], sc1[i]));
        st.scatter_dev_ns += (uint64_t)(ms * 1e6);
    }
    st.decode_dev_ns = 0;
    for (size_t i = 0; i < dc0.size(); i++) {
        CUDA_TRY(c, cudaEventElapsedTime(&ms, dc0[i], dc1[i]));
        st.decode_dev_ns += (uint64_t)(ms * 1e6);
    }
    st.verify_dev_ns = 0;
    st.verify_failures = 0;
    st.first_bad_page = UINT64_MAX;
    if (c->cfg.verify) {
        CUDA_TRY(c, cudaEventElapsedTime(&ms, v0, v1));
        st.verify_dev_ns = (uint64_t)(ms * 1e6);
        st.verify_failures = c->misc_h[1];
        st.first_bad_page = c->misc_h[2];
    }
    st.verify_launches = verify_launches;
    st.restore_h2d_bytes = h2d_bytes;
    st.restore_ns = ns_since(t0);
    if (st.verify_failures)
        return fail(c, GCR_E_VERIFY, "restore: " + std::to_string(st.verify_failures) + " page digest(s) differ");
    c->phase = GCR_LOCKED;
    // the next incremental diffs against the restored state (c.2 step 4)
    c->parent_idx = scratch;
    c->parent_gen = last->hdr.generation;
    c->have_parent = true;
    c->next_gen = std::max(c->next_gen, last->hdr.generation + 1);
    return GCR_OK;
}

gcr_status gcr_restore(gcr_ctx *c, gcr_image *const *chain, uint32_t n) {
    NvtxScope nvtx_("gcr.restore");
    if (!c) return GCR_E_INVAL;
    const gcr_phase ph0 = c->phase;
    bool writes_began = false;
    const gcr_status s = restore_impl(c, chain, n, writes_began);
    if (s != GCR_OK) sync_all(c);  // nothing of this call (e.g. the speculative H2D) outlives it
    if (s != GCR_OK && writes_began) {
        // memory content undefined: no incremental may diff against it, and
        // memory re-backed after a release stays RELEASED (unlock refused)
        // until a restore succeeds
        sync_all(c);
        c->have_parent = false;
        c->phase = ph0 == GCR_RELEASED ? GCR_RELEASED : GCR_LOCKED;
    }
    return s;
}

gcr_status gcr_mem_alloc(gcr_ctx *c, uint64_t bytes, uint64_t *dptr_out) {
    if (!c) return GCR_E_INVAL;
    if (!dptr_out || bytes == 0) return fail(c, GCR_E_INVAL, "mem_alloc: null or empty");
    *dptr_out = 0;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "mem_alloc: not RUNNING");
    const Vmm &v = vmm();
    if (!v.ok) return fail(c, GCR_E_CUDA, "mem_alloc: driver VMM entry points unavailable");
    CUDA_TRY(c, cudaSetDevice(c->device));
    const CUmemAllocationProp prop = mem_prop(c->device);
    size_t gran = 0;
    if (v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0)
        return fail(c, GCR_E_CUDA, "mem_alloc: cuMemGetAllocationGranularity failed");
    MemBlock b{};
    b.user_bytes = bytes;
    b.size = (bytes + gran - 1) / gran * gran;
    CUdeviceptr va = 0;
    if (v.reserve(&va, b.size, gran, 0, 0) != CUDA_SUCCESS)
        return fail(c, GCR_E_NOMEM, "mem_alloc: cuMemAddressReserve failed");
    b.va = va;
    const CUresult r = map_block(c->device, b);
    if (r != CUDA_SUCCESS) {
        v.addr_free(b.va, b.size);
        return fail(c, r == CUDA_ERROR_OUT_OF_MEMORY ? GCR_E_NOMEM : GCR_E_CUDA,
                    "mem_alloc: cuMemCreate/Map failed (driver error " + std::to_string((int)r) + ")");
    }
    c->blocks.push_back(b);
    *dptr_out = b.va;
    return GCR_OK;
}

gcr_status gcr_mem_free(gcr_ctx *c, uint64_t dptr) {
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_RUNNING) return fail(c, GCR_E_STATE, "mem_free: not RUNNING");
    for (size_t i = 0; i < c->blocks.size(); i++) {
        MemBlock &b = c->blocks[i];
        if (b.va != dptr) continue;
        for (const RegEntry &r : c->reg)
            if (r.dptr < b.va + b.size && b.va < r.dptr + r.bytes)
                return fail(c, GCR_E_INVAL, "mem_free: a registered allocation lies in the block");
        CUDA_TRY(c, cudaSetDevice(c->device));
        CUDA_TRY(c, cudaDeviceSynchronize());  // no kernel may still touch it
        if (b.mapped && unmap_block(b) != CUDA_SUCCESS) return fail(c, GCR_E_CUDA, "mem_free: cuMemUnmap failed");
        vmm().addr_free(b.va, b.size);
        c->blocks.erase(c->blocks.begin() + i);
        return GCR_OK;
    }
    return fail(c, GCR_E_INVAL, "mem_free: not a gcr_mem_alloc block");
}

gcr_status gcr_release(gcr_ctx *c) {
    NvtxScope nvtx_("gcr.release");
    if (!c) return GCR_E_INVAL;
    if (c->phase != GCR_CHECKPOINTED) return fail(c, GCR_E_STATE, "release: not CHECKPOINTED");
    // every registered allocation inside a block; every touched block fully registered
    std::vector<uint64_t> covered(c->blocks.size(), 0);
    for (const RegEntry &r : c->reg) {
        size_t k = 0;
        for (; k < c->blocks.size(); k++) {
            const MemBlock &b = c->blocks[k];
            if (r.dptr >= b.va && r.dptr + r.bytes <= b.va + b.user_bytes) break;
        }
        if (k == c->blocks.size())
            return fail(c, GCR_E_INVAL, "release: a registered allocation is not gcr_mem_alloc memory");
        covered[k] += r.bytes;
    }
    for (size_t k = 0; k < c->blocks.size(); k++)
        if (covered[k] != 0 && covered[k] != c->blocks[k].user_bytes)
            return fail(c, GCR_E_INVAL, "release: a block is only partly registered (its other bytes would be lost)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    sync_all(c);
    CUDA_TRY(c, cudaDeviceSynchronize());
    const auto t0 = Clock::now();
    uint64_t freed = 0;
    gcr_status s = GCR_OK;
    for (size_t k = 0; k < c->blocks.size(); k++) {
        MemBlock &b = c->blocks[k];
        if (covered[k] == 0 || !b.mapped) continue;
        if (unmap_block(b) != CUDA_SUCCESS) {
            s = fail(c, GCR_E_CUDA, "release: cuMemUnmap/cuMemRelease failed");
            if (b.mapped) break;  // still mapped: stop here
        }
        freed += b.size;
    }
    c->stats.release_ns = ns_since(t0);
    c->stats.released_bytes = freed;
    if (freed) c->phase = GCR_RELEASED;
    return s;
}

gcr_status gcr_probe_link(gcr_ctx *c, uint64_t bytes, double *d2h_gbs, double *h2d_gbs) {
    NvtxScope nvtx_("gcr.probe_link");
    if (!c) return GCR_E_INVAL;
    if (!d2h_gbs || !h2d_gbs || bytes == 0 || bytes > c->cfg.chunk_bytes || c->slots.empty())
        return fail(c, GCR_E_INVAL, "probe_link: null output, or bytes not in (0, chunk_bytes]");
    *d2h_gbs = *h2d_gbs = 0.0;
    CUDA_TRY(c, cudaSetDevice(c->device));
    sync_all(c);
    // the pool's first free range of `bytes`: where the next image's data lands
    void *h = c->pool.alloc(bytes);
    if (!h) return fail(c, GCR_E_NOMEM, "probe_link: pinned pool allocation failed");
    gcr_status st = GCR_OK;
    cudaStream_t cs = c->copy[0];
    for (int dir = 0; dir < 2 && st == GCR_OK; dir++) {
        cudaEvent_t e0 = c->ev(), e1 = c->ev();
        auto copy = [&]() {
            return dir == 0 ? cudaMemcpyAsync(h, c->slots[0], bytes, cudaMemcpyDeviceToHost, cs)
                            : cudaMemcpyAsync(c->slots[0], h, bytes, cudaMemcpyHostToDevice, cs);
        };
        cudaError_t e = copy();  // warm-up
        if (e == cudaSuccess) e = cudaEventRecord(e0, cs);
        for (int r = 0; r < 3 && e == cudaSuccess; r++) e = copy();
        if (e == cudaSuccess) e = cudaEventRecord(e1, cs);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e != cudaSuccess) {
            cudaGetLastError();
            st = fail(c, GCR_E_CUDA, std::string("probe_link: ") + cudaGetErrorString(e));
            break;
        }
        (dir == 0 ? *d2h_gbs : *h2d_gbs) = 3.0 * (double)bytes / (ms * 1e-3) / 1e9;
    }
    c->ev_used = 0;
    c->pool.release(h, bytes);
    return st;
}

gcr_status gcr_get_phase(const gcr_ctx *c, gcr_phase *out) {
    if (!c || !out) return GCR_E_INVAL;
    *out = c->phase;
    return GCR_OK;
}

gcr_status gcr_get_stats(const gcr_ctx *c, gcr_stats *out) {
    if (!c || !out) return GCR_E_INVAL;
    *out = c->stats;
    return GCR_OK;
}

gcr_status gcr_ctx_stream(const gcr_ctx *c, void **out) {
    if (!c || !out) return GCR_E_INVAL;
    *out = c->compute;
    return GCR_OK;
}

const char *gcr_last_error(const gcr_ctx *c) { return c ? c->err.c_str() : "null ctx"; }

gcr_status gcr_image_header(const gcr_image *img, gcr_image_hdr *out) {
    if (!img || !out) return GCR_E_INVAL;
    *out = img->hdr;
    return GCR_OK;
}

gcr_status gcr_image_allocs(const gcr_image *img, const gcr_alloc_rec **p, uint32_t *n) {
    if (!img || !p || !n) return GCR_E_INVAL;
    *p = img->allocs.data();
    *n = (uint32_t)img->allocs.size();
    return GCR_OK;
}

gcr_status gcr_image_pagemap(const gcr_image *img, const gcr_pagemap_entry **p, uint64_t *n) {
    if (!img || !p || !n) return GCR_E_INVAL;
    *p = img->pagemap;
    *n = img->hdr.n_entries;
    return GCR_OK;
}

gcr_status gcr_image_digests(const gcr_image *img, const uint32_t **p, uint64_t *n) {
    if (!img || !p || !n) return GCR_E_INVAL;
    *p = img->digests;
    *n = img->hdr.n_pages;
    return GCR_OK;
}

gcr_status gcr_image_data(const gcr_image *img, const uint8_t **p, uint64_t *bytes) {
    if (!img || !p || !bytes) return GCR_E_INVAL;
    *p = img->data;
    *bytes = img->hdr.image_bytes;
    return GCR_OK;
}

gcr_status gcr_image_free(gcr_image *img) {
    if (!img || !img->ctx) return GCR_E_INVAL;
    gcr_ctx *c = img->ctx;
    cudaSetDevice(c->device);
    sync_all(c);
    destroy_image(c, img);
    return GCR_OK;
}

gcr_status gcr_image_stored(const gcr_image *img, const uint32_t **p, uint64_t *n) {
    if (!img || !p || !n) return GCR_E_INVAL;
    const bool coded = img->hdr.flags & 2u;
    *p = coded ? img->stored : nullptr;
    *n = coded ? img->hdr.n_present : 0;
    return GCR_OK;
}

gcr_status gcr_image_stream_size(const gcr_image *img, uint64_t *bytes) {
    if (!img || !bytes) return GCR_E_INVAL;
    const gcr_image_hdr &h = img->hdr;
    *bytes = 96 + 24ull * h.n_allocs + 16ull * h.n_entries + 4ull * h.n_pages +
             ((h.flags & 2u) ? 4ull * h.n_present : 0ull) + h.image_bytes;
    return GCR_OK;
}

gcr_status gcr_image_serialize(const gcr_image *img, void *dst, uint64_t cap) {
    uint64_t need;
    if (!dst || gcr_image_stream_size(img, &need) != GCR_OK || cap < need) return GCR_E_INVAL;
    const gcr_image_hdr &h = img->hdr;
    uint8_t *o = static_cast<uint8_t *>(dst);
    std::memcpy(o, &h, 96);
    o += 96;
    std::memcpy(o, img->allocs.data(), 24ull * h.n_allocs);
    o += 24ull * h.n_allocs;
    if (h.n_entries) std::memcpy(o, img->pagemap, 16ull * h.n_entries);
    o += 16ull * h.n_entries;
    std::memcpy(o, img->digests, 4ull * h.n_pages);
    o += 4ull * h.n_pages;
    if ((h.flags & 2u) && h.n_present) {
        std::memcpy(o, img->stored, 4ull * h.n_present);
        o += 4ull * h.n_present;
    }
    if (h.image_bytes) std::memcpy(o, img->data, h.image_bytes);
    return GCR_OK;
}

gcr_status gcr_image_import(gcr_ctx *c, const void *stream, uint64_t bytes, gcr_image **out) {
    NvtxScope nvtx_("gcr.import");
    if (!c) return GCR_E_INVAL;
    if (!stream || !out) return fail(c, GCR_E_INVAL, "import: null argument");
    *out = nullptr;
    const uint8_t *s = static_cast<const uint8_t *>(stream);
    if (bytes < 96) return fail(c, GCR_E_CORRUPT, "import: shorter than a header");
    gcr_image_hdr h;
    std::memcpy(&h, s, 96);
    if (std::memcmp(h.magic, kMagic, 8) != 0) return fail(c, GCR_E_CORRUPT, "import: bad magic");
    if (h.n_pages > bytes / 4 || h.n_entries > bytes / 16 || h.n_allocs > bytes / 24 || h.n_present > bytes / 4)
        return fail(c, GCR_E_CORRUPT, "import: section sizes exceed the stream");
    const uint64_t nst = (h.flags & 2u) ? h.n_present : 0;  // f4 stored-length table
    const uint64_t meta = 96 + 24ull * h.n_allocs + 16ull * h.n_entries + 4ull * h.n_pages + 4ull * nst;
    if (meta > bytes || bytes - meta != h.image_bytes) return fail(c, GCR_E_CORRUPT, "import: framing mismatch");
    gcr_image_hdr h0 = h;
    h0.meta_crc32c = 0;
    uint32_t st = host_crc32c_update(0xFFFFFFFFu, &h0, 96);
    st = host_crc32c_update(st, s + 96, meta - 96) ^ 0xFFFFFFFFu;
    if (st != h.meta_crc32c) return fail(c, GCR_E_CORRUPT, "import: meta_crc32c mismatch");
    if (h.version != 1 || (h.flags & ~3u)) return fail(c, GCR_E_VERSION, "import: unknown version or flag bits");
    CUDA_TRY(c, cudaSetDevice(c->device));
    gcr_image *img = new (std::nothrow) gcr_image;
    if (!img) return fail(c, GCR_E_NOMEM, "import: out of host memory");
    img->ctx = c;
    img->hdr = h;
    img->allocs.resize(h.n_allocs);
    std::memcpy(img->allocs.data(), s + 96, 24ull * h.n_allocs);
    img->pagemap_cap = 16ull * h.n_entries;
    img->digests_cap = 4ull * h.n_pages;
    img->data_cap = h.image_bytes;
    img->pagemap = static_cast<gcr_pagemap_entry *>(c->pool.alloc(img->pagemap_cap));
    img->digests = static_cast<uint32_t *>(c->pool.alloc(img->digests_cap));
    img->data = static_cast<uint8_t *>(c->pool.alloc(img->data_cap));
    img->stored_cap = 4ull * nst;
    img->stored = nst ? static_cast<uint32_t *>(c->pool.alloc(img->stored_cap)) : nullptr;
    c->stats.pinned_alloc_ns = c->pool.pin_ns;
    if (!img->pagemap || !img->digests || !img->data || (nst && !img->stored)) {
        image_free_buffers(img);
        delete img;
        return fail(c, GCR_E_NOMEM, "import: pinned allocation failed");
    }
    const uint8_t *o = s + 96 + 24ull * h.n_allocs;
    std::memcpy(img->pagemap, o, 16ull * h.n_entries);
    o += 16ull * h.n_entries;
    std::memcpy(img->digests, o, 4ull * h.n_pages);
    o += 4ull * h.n_pages;
    if (nst) std::memcpy(img->stored, o, 4ull * nst);
    o += 4ull * nst;
    std::memcpy(img->data, o, h.image_bytes);
    c->images.push_back(img);
    *out = img;
    return GCR_OK;
}

// ---- storage tier (f3) ------------------------------------------------------
}  // extern "C"

namespace {

constexpr uint64_t kIoPiece = 64ull << 20;  // bytes per positional read/write unit

struct IoSeg {
    uint64_t file_off;
    uint8_t *buf;
    uint64_t len;
};

// Positional I/O of every segment, split into kIoPiece units handed out to
// n threads; returns 0 or the first errno.
int parallel_io(int fd, const std::vector<IoSeg> &segs, uint32_t n_threads, bool write) {
    struct Unit {
        uint64_t off;
        uint8_t *buf;
        uint64_t len;
    };
    std::vector<Unit> units;
    for (const IoSeg &sg : segs)
        for (uint64_t o = 0; o < sg.len; o += kIoPiece)
            units.push_back(Unit{sg.file_off + o, sg.buf + o, std::min(kIoPiece, sg.len - o)});
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    auto work = [&]() {
        for (size_t i; (i = next.fetch_add(1)) < units.size() && err.load() == 0;) {
            const Unit &u = units[i];
            uint64_t done = 0;
            while (done < u.len) {
                const ssize_t r = write ? pwrite(fd, u.buf + done, u.len - done, (off_t)(u.off + done))
                                        : pread(fd, u.buf + done, u.len - done, (off_t)(u.off + done));
                if (r < 0 && errno == EINTR) continue;
                if (r <= 0) {
                    int e0 = 0;
                    err.compare_exchange_strong(e0, r < 0 ? errno : EIO);
                    return;
                }
                done += (uint64_t)r;
            }
        }
    };
    const uint32_t T = std::max<uint32_t>(1, std::min<uint32_t>(n_threads ? n_threads : 8, 64));
    std::vector<std::thread> th;
    for (uint32_t t = 1; t < T && t < units.size(); t++) th.emplace_back(work);
    work();
    for (auto &x : th) x.join();
    return err.load();
}

}  // namespace

extern "C" {

gcr_status gcr_image_write_file(const gcr_image *img, const char *path, uint32_t n_threads, uint32_t flags) {
    NvtxScope nvtx_("gcr.write_file");
    if (!img || !path) return GCR_E_INVAL;
    gcr_ctx *c = img->ctx;
    const gcr_image_hdr &h = img->hdr;
    uint64_t total = 0;
    gcr_image_stream_size(img, &total);
    const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (fd < 0) return fail(c, GCR_E_IO, std::string("write_file: open: ") + std::strerror(errno));
    auto io_fail = [&](const char *what, int e) {
        close(fd);
        return fail(c, GCR_E_IO, std::string("write_file: ") + what + ": " + std::strerror(e));
    };
    if (ftruncate(fd, (off_t)total) != 0) return io_fail("ftruncate", errno);
    // header + alloc table are small host vectors: one contiguous prefix
    std::vector<uint8_t> prefix(96 + 24ull * h.n_allocs);
    std::memcpy(prefix.data(), &h, 96);
    if (h.n_allocs) std::memcpy(prefix.data() + 96, img->allocs.data(), 24ull * h.n_allocs);
    uint64_t o = 0;
    std::vector<IoSeg> segs;
    segs.push_back(IoSeg{o, prefix.data(), prefix.size()});
    o += prefix.size();
    segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->pagemap), 16ull * h.n_entries});
    o += 16ull * h.n_entries;
    segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->digests), 4ull * h.n_pages});
    o += 4ull * h.n_pages;
    if (h.flags & 2u) {
        segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->stored), 4ull * h.n_present});
        o += 4ull * h.n_present;
    }
    segs.push_back(IoSeg{o, img->data, h.image_bytes});
    const int e = parallel_io(fd, segs, n_threads, true);
    if (e) return io_fail("pwrite", e);
    if (flags & GCR_IO_SYNC) {
        if (fdatasync(fd) != 0) return io_fail("fdatasync", errno);
        posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);  // the next read comes from the device
    }
    if (close(fd) != 0) return fail(c, GCR_E_IO, std::string("write_file: close: ") + std::strerror(errno));
    return GCR_OK;
}

gcr_status gcr_image_read_file(gcr_ctx *c, const char *path, uint32_t n_threads, gcr_image **out) {
    NvtxScope nvtx_("gcr.read_file");
    if (!c) return GCR_E_INVAL;
    if (!path || !out) return fail(c, GCR_E_INVAL, "read_file: null argument");
    *out = nullptr;
    const int fd = open(path, O_RDONLY | O_CLOEXEC);
    if (fd < 0) return fail(c, GCR_E_IO, std::string("read_file: open: ") + std::strerror(errno));
    struct stat sb {};
    if (fstat(fd, &sb) != 0) {
        const int e = errno;
        close(fd);
        return fail(c, GCR_E_IO, std::string("read_file: fstat: ") + std::strerror(e));
    }
    const uint64_t bytes = (uint64_t)sb.st_size;
    gcr_image_hdr h{};
    if (bytes < 96 || pread(fd, &h, 96, 0) != 96) {
        close(fd);
        return fail(c, GCR_E_CORRUPT, "read_file: shorter than a header");
    }
    // framing checks as in gcr_image_import, before allocating anything
    if (std::memcmp(h.magic, kMagic, 8) != 0 || h.n_pages > bytes / 4 || h.n_entries > bytes / 16 ||
        h.n_allocs > bytes / 24 || h.n_present > bytes / 4) {
        close(fd);
        return fail(c, GCR_E_CORRUPT, "read_file: bad magic or section sizes exceed the file");
    }
    const uint64_t nst = (h.flags & 2u) ? h.n_present : 0;  // f4 stored-length table
    const uint64_t meta = 96 + 24ull * h.n_allocs + 16ull * h.n_entries + 4ull * h.n_pages + 4ull * nst;
    if (meta > bytes || bytes - meta != h.image_bytes) {
        close(fd);
        return fail(c, GCR_E_CORRUPT, "read_file: framing mismatch (file size != stream size)");
    }
    gcr_image *img = new (std::nothrow) gcr_image;
    if (!img) {
        close(fd);
        return fail(c, GCR_E_NOMEM, "read_file: out of host memory");
    }
    auto bail = [&](gcr_status s, const std::string &m) {
        close(fd);
        image_free_buffers(img);
        delete img;
        return fail(c, s, m);
    };
    if (cudaSetDevice(c->device) != cudaSuccess) {
        cudaGetLastError();
        return bail(GCR_E_CUDA, "read_file: cudaSetDevice failed");
    }
    img->ctx = c;
    img->hdr = h;
    img->allocs.resize(h.n_allocs);
    img->pagemap_cap = 16ull * h.n_entries;
    img->digests_cap = 4ull * h.n_pages;
    img->data_cap = h.image_bytes;
    img->pagemap = static_cast<gcr_pagemap_entry *>(c->pool.alloc(img->pagemap_cap));
    img->digests = static_cast<uint32_t *>(c->pool.alloc(img->digests_cap));
    img->data = static_cast<uint8_t *>(c->pool.alloc(img->data_cap));
    img->stored_cap = 4ull * nst;
    img->stored = nst ? static_cast<uint32_t *>(c->pool.alloc(img->stored_cap)) : nullptr;
    c->stats.pinned_alloc_ns = c->pool.pin_ns;
    if ((img->pagemap_cap && !img->pagemap) || (img->digests_cap && !img->digests) || (img->data_cap && !img->data) ||
        (nst && !img->stored))
        return bail(GCR_E_NOMEM, "read_file: pinned allocation failed");
    std::vector<IoSeg> segs;
    uint64_t o = 96;
    segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->allocs.data()), 24ull * h.n_allocs});
    o += 24ull * h.n_allocs;
    segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->pagemap), 16ull * h.n_entries});
    o += 16ull * h.n_entries;
    segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->digests), 4ull * h.n_pages});
    o += 4ull * h.n_pages;
    if (nst) {
        segs.push_back(IoSeg{o, reinterpret_cast<uint8_t *>(img->stored), 4ull * nst});
        o += 4ull * nst;
    }
    segs.push_back(IoSeg{o, img->data, h.image_bytes});
    const int e = parallel_io(fd, segs, n_threads, false);
    if (e) return bail(GCR_E_IO, std::string("read_file: pread: ") + std::strerror(e));
    close(fd);
    if (meta_crc(img) != h.meta_crc32c) {
        image_free_buffers(img);
        delete img;
        return fail(c, GCR_E_CORRUPT, "read_file: meta_crc32c mismatch");
    }
    if (h.version != 1 || (h.flags & ~3u)) {
        image_free_buffers(img);
        delete img;
        return fail(c, GCR_E_VERSION, "read_file: unknown version or flag bits");
    }
    c->images.push_back(img);
    *out = img;
    return GCR_OK;
}

}  // extern "C"
