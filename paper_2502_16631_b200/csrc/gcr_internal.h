// gcr_internal.h -- internal types shared by the libgcr host runtime
// (gcr.cpp, crc_host.cpp, pinned_pool.cpp) and the sm_100a kernels
// (kernels.cu).  Not part of the C-ABI (include/gcr.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gcr {

// ---------------------------------------------------------------------------
// Work geometry.  K1 streams 512-byte ROWS (one per warp
// instruction); a TILE is 64 KiB of page space, the unit of compaction/pack.
constexpr uint32_t kTileBytes = 65536;
constexpr uint32_t kRowBytes = 512;  // one warp row: 32 lanes x 16 B
constexpr uint32_t kLog2Tile = 16;

// Page classes (c.1 step 5).  cls[] bytes also carry kClsAllocStart on the
// first page of each allocation (runs never cross allocations, c.1 step 7).
constexpr uint8_t kClsPresent = 0, kClsZero = 1, kClsParent = 2;
constexpr uint8_t kClsAllocStart = 0x80;

enum ScanMode : int { kScanFull = 0, kScanIncremental = 1, kScanVerify = 2 };

// Per-allocation descriptor in device memory (A1 page table).
struct AllocDev {
    uint64_t base;      // device address of the allocation
    uint64_t bytes;     // registered length (multiple of 16)
    uint64_t page0;     // global index of its first page
    uint64_t tile0;     // global index of its first tile
    uint32_t n_pages;
    uint32_t n_tiles;
    uint32_t tail_len;  // length of its last page (== page_size if none is short)
    uint32_t z_tail;    // Z(tail_len) = CRC32C of tail_len zero bytes
    uint64_t row0;      // global index of its first REAL 512-byte row
    uint64_t n_rows;    // (n_pages-1)*P/512 + ceil(tail_len/512)
    uint64_t grp0;      // small pages (K1g): global index of its first page group
};

// GCR_SCAN_TIMES diagnostics: per K1 warp {entry, tables staged, first rows
// loaded, chunk 0 done, exit} globaltimer stamps (+1 spare).
constexpr uint32_t kScanStamps = 6;

// Small pages (P = 4 KiB / 8 KiB): K1g scans G = 16 KiB / P consecutive pages
// of one allocation (a page GROUP, 16 KiB) at once, one page per 32/G lanes,
// so the per-page lane tree is shared by G pages.
constexpr uint32_t kGroupBytes = 16384;

// A page cut by K1 warp-range boundaries is folded inside K1: every warp
// holding a piece of it folds the piece's contribution into the page's owner
// slot (owner = the warp whose range holds the page's first real row) with ONE
// 64-bit compare-and-swap that XORs the contribution into the low word and
// adds its row count (bits 32-47) and non-zero flag (bits 48-63) to the high
// word; the CAS that completes the page's rows holds the full XOR in its own
// result and finalizes the page (no fences, no second read), then re-zeroes the
// slot for the next launch.  One slot per K1 warp and chunk.
struct FoldSlots {
    unsigned long long *s;
};

// Per-tile result of the scan used by compaction (K2) and pack (K4).
struct TileInfo {
    uint32_t present_bytes;  // PRESENT bytes whose image offset is anchored at this tile
    uint32_t counts;         // n_present | n_zero << 10 | n_parent << 20 (pages anchored here)
};

// Record of one NON-EMPTY tile the host reads (mapped pinned) to plan the drain.
struct TileRec {
    uint32_t tile;           // chunk-local tile index
    uint32_t present_bytes;  // PRESENT bytes anchored at the tile
    uint32_t image_off;      // chunk-local image offset of the tile's first PRESENT byte
    uint32_t pad;
};

// One staged tile for K4 (host-written, mapped pinned): the chunk-local tile
// and the slot offset of its first PRESENT byte (for a page > 64 KiB: of the
// slice itself).
struct StageItem {
    uint32_t tile;
    uint32_t dst;
};

struct ChunkTotals {
    unsigned long long image_bytes;
    unsigned long long n_present, n_zero, n_parent;
};

// CRC32C tables in device global memory; kernels stage them in shared memory.
// Every table maps a 32-bit register v to adv_d(v) = v * x^(8d) mod P as the
// XOR of 4 byte-indexed entries: tab[k][e] = adv_d(e << 8k).
struct CrcTables {
    uint32_t braid[4][256];  // d = 512 (one row of 32 lanes x 16 B)
    uint32_t t4[4][256];     // d = 4   (word step for the lane raw16)
    uint32_t a16[4][256];    // d = 16  (lane tree, level 0)
    uint32_t a32[4][256];    // d = 32  (level 1)
    uint32_t a64[4][256];    // d = 64  (level 2)
    uint32_t a128[4][256];   // d = 128 (level 3)
    uint32_t a256[4][256];   // d = 256 (level 4)
    // fold_m[d] = x^(8 * 512 d) mod P in the reflected representation (x^0 =
    // 0x80000000), d < 4096 rows: a piece ending d rows before its page's end
    // contributes fold_m[d] (*) raw, a GF(2) product K1 forms lane-parallel.
    uint32_t fold_m[4096];
};

// f1 in-scan pack (incremental checkpoints, gcr_config.pack_mode = 1;
// SURVEY §8(f) f1): K1 itself writes every PRESENT page straight into the
// pinned host image through mapped memory -- no K4 pack, no staging slot, no
// D2H of page data.  A page's image offset = base[c] (the chunk's first
// PRESENT byte: K2(c - 1) computes base[c] = base[c - 1] + its chunk total)
// + the PRESENT bytes finalized in chunk c by earlier CTAs (per-CTA aggregates
// published by each CTA's last warp to finish the chunk) + those of earlier
// warps of the same CTA (shared memory) + the warp's own earlier pages.  A
// warp finalizes pages in page order and the pages it finalizes form a
// contiguous run in page order, so these groups tile the image in order.  The
// write-out of chunk c is deferred until the warp has scanned chunk c + 1 (by
// then every aggregate of chunk c is published); the last chunk's right after
// it.
struct InScanPack {
    uint8_t *img;                // device-visible address of the image data (null: off)
    unsigned long long *cta_agg; // [n_chunks][n_ctas]: tag(epoch, chunk) | PRESENT bytes finalized by the CTA
                                 // in the chunk (one slot per chunk: CTAs may be chunks apart)
    unsigned long long *base;    // [n_chunks + 1] image offset of each chunk (base[0] = 0), written by K2
    uint32_t *base_ready;        // [n_chunks + 1] epoch once base[c] is written
    uint32_t *list;              // [2][workers][cap] PRESENT pages the warp finalized, in page order
    uint32_t cap;
    unsigned long long *err;     // non-zero on a wait timeout (which | chunk << 8 | CTA << 32) or a list overflow (4)
    uint64_t wait_ns;            // bound of every wait (GCR_ISP_WAIT_MS, default 30 s)
};

// K1 is ONE persistent launch per checkpoint (or verify): every warp walks
// the chunks in order, taking its equal share of each chunk's real rows.  The
// last warp to finish chunk c publishes chunk_done[c] = epoch, on which K2(c),
// enqueued ahead on the post stream, waits -- no launch boundary, host
// round-trip or launch latency between a chunk's scan and its compaction.
struct ScanParams {
    const AllocDev *allocs;
    uint32_t n_allocs;
    const uint64_t *chunk_rows;    // n_chunks + 1 global real-row boundaries (page aligned), device
    uint32_t n_chunks;
    uint32_t epoch;                // this launch's id, published in chunk_done (never 0)
    uint32_t *chunk_arrive;        // per chunk: warps done (the last one re-zeroes it)
    uint32_t *chunk_done;          // per chunk: epoch of the launch that last completed it
    uint64_t workers;              // warps; every chunk is split among all of them
    FoldSlots fold;                // workers slot pairs per chunk
    uint32_t page_size, log2_page;
    uint32_t z_page;
    int mode;
    const uint32_t *d_ref;     // D_prev (incremental) or D_k (verify)
    uint32_t *d_out;           // D_new (full / incremental)
    uint8_t *cls;              // class per page (full / incremental)
    TileInfo *tile_info;       // per tile (full / incremental)
    unsigned long long *verify_count;
    unsigned long long *first_bad;
    const CrcTables *tables;
    uint32_t prefetch;         // bytes: each warp keeps [cursor + prefetch, + block) requested into L2
    const uint64_t *chunk_groups;  // K1g: n_chunks + 1 global page-group boundaries (device)
    unsigned long long *warp_times;  // optional (GCR_SCAN_TIMES): kScanStamps globaltimer ns per warp
    uint32_t grp_pf_block;     // K1g: block of a group (0..7) at which the next group is prefetched
    // Every table is linear in its byte index (tab[k][e] = adv(e << 8k)), so
    // the kernel rebuilds it in shared memory from 8 basis values per k:
    // basis[t][8k + i] = tab_t[k][1 << i], t = 0: the braid table of this
    // launch (adv_512; K1g: adv_128 / adv_256), 1..6: t4, a16 .. a256.  Kernel
    // parameters live in the constant bank: no 148-SM burst on the same L2
    // lines at launch (the global-table staging cost ~4.8 us per launch).
    uint32_t basis[7][32];
    InScanPack isp;            // f1 (img == nullptr: off)
    uint32_t t4rep;            // K1g: 8x-replicated raw16 table (see kernels.cu kT4RepBytes)
    const uint32_t *isp_page_alloc;  // f1: page -> allocation (K0's table)
    uint32_t *sb_probe;        // scan_probe(): the kernel writes its dynamic-smem base here and exits
    // 0, or the first chunk of a tail that K1 splits over its warps as ONE range
    // and publishes at once (full checkpoints: the drain needs chunk 0 early,
    // the rest long before the link frees up; one range start per warp instead
    // of one per chunk).  Never with the f1 in-scan pack (per-chunk lists).
    uint32_t merge_from;
};

struct ScatterDesc {
    uint64_t dst;      // device address
    uint64_t src_off;  // offset in the staging slot
    uint64_t bytes;    // multiple of 16
};

struct ZeroDesc {
    uint64_t dst;
    uint64_t bytes;
};

// f4 restore: one PRESENT page's stored form in a staging slot -> its page.
struct DecodeDesc {
    uint64_t dst;      // device address of the page
    uint64_t src_off;  // offset of the stored form in the slot (multiple of 16)
    uint32_t len;      // page length (multiple of 16)
    uint32_t stored;   // stored length (== len: raw)
};

// ---- kernel launchers (kernels.cu); all asynchronous on `st` -------------
// Each returns the number of kernels it launched (for stats) or -1 on a
// launch error (cudaGetLastError holds it).
int launch_build_page_table(const AllocDev *allocs, uint32_t n_allocs, uint32_t *page_alloc,
                            uint32_t *tile_alloc, uint32_t tiles_per_page, uint32_t pages_per_tile,
                            cudaStream_t st);
int scan_free_sms(bool incremental);                                // SMs K1 leaves to K2 / K4
uint64_t scan_workers(int n_sms, int free_sms);                      // K1 warps (a full persistent grid)
uint32_t scan_prefetch_bytes();                                     // K1 L2 prefetch distance (GCR_SCAN_PREFETCH)
uint32_t grp_prefetch_block();                                      // K1g prefetch trigger block (GCR_GRP_PF_BLOCK)
bool grp_t4rep();                                                   // K1g 8x raw16 table (GCR_GRP_T4REP)
int launch_scan(const ScanParams &p, int n_sms, cudaStream_t st);  // K1 (K1g when p.chunk_groups is set)
bool scan_uses_groups(uint32_t page_size);                          // K1g for this page size?
// K2 of one chunk: first waits (bounded) until chunk_done[chunk] == epoch.
// f1: if isp_base is set, K2(c) also writes isp_base[c + 1] = isp_base[c] +
// the chunk's PRESENT bytes and isp_ready[c + 1] = epoch.
int launch_tile_scan(TileInfo *tile_info, uint64_t tile_begin, uint64_t tile_end, const uint32_t *chunk_done,
                     uint32_t chunk, uint32_t epoch, TileRec *host_rec, unsigned long long *rec_count,
                     ChunkTotals *totals_host, unsigned long long *isp_base, uint32_t *isp_ready, cudaStream_t st);
int launch_pack(const AllocDev *allocs, const uint32_t *tile_alloc, const uint8_t *cls, uint64_t tile_begin,
                uint32_t page_size, uint32_t log2_page, uint8_t *slot, const StageItem *items, uint32_t n_items,
                int n_sms, int scan_free, const uint32_t *scan_done, uint32_t epoch, uint32_t *decision,
                cudaStream_t st);
// Pagemap over all pages: phase 1 counts run starts per block and scans them,
// writing the entry count to *n_entries_dev; phase 2 writes the entries.
int launch_pagemap_count(const uint8_t *cls, uint64_t n_pages, uint32_t *blk_cnt, uint32_t *blk_off,
                         unsigned long long *n_entries_dev, cudaStream_t st);
int launch_pagemap_write(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls,
                         uint64_t n_pages, uint32_t log2_page, const uint32_t *blk_off,
                         uint32_t *run_start, uint64_t n_entries, void *entries_dev, cudaStream_t st);
int launch_scatter(const ScatterDesc *desc, uint64_t n_desc, const uint8_t *slot, int n_sms,
                   cudaStream_t st);
int launch_zero_fill(const ZeroDesc *desc, uint64_t n_desc, int n_sms, cudaStream_t st);
size_t scan_smem_bytes();
uint64_t scan_warps_per_cta();  // K1 / K8 warps per CTA (GCR_SCAN_TIMES summaries)
// Once per device (gcr_create): launch K1g in probe mode to read its dynamic
// shared-memory base; K1g's immediate-base braid variant is used when the low
// 16 bits match the compile-time value (kernels.cu kGrpSbLo).  Returns 0 / -1.
int scan_probe();

// ---- f4 page codec (codec.cu, R-19) -------------------------------
// KA over the chunk's pages [page_begin, page_begin + n_pages): stored length
// per page (0 if not PRESENT) and presence masks (32 u32 per page).
int launch_codec_plan(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls, uint64_t page_begin,
                      uint32_t n_pages, uint32_t page_size, uint32_t log2_page, uint32_t *plan, uint32_t *masks,
                      uint32_t *done, int n_sms, cudaStream_t st);
// KB: slot offsets (from slot_base), the image's compact stored-length table
// from present_base on, {stored total, PRESENT count} into mapped host memory.
int launch_codec_offsets(const uint32_t *plan, uint32_t n_pages, uint32_t *off, uint32_t *stored_compact,
                         uint64_t present_base, uint64_t slot_base, unsigned long long *total_host, cudaStream_t st);
// KC: stored forms of the chunk's PRESENT pages into the slot.
int launch_codec_encode(const AllocDev *allocs, const uint32_t *page_alloc, const uint8_t *cls, uint64_t page_begin,
                        uint32_t n_pages, uint32_t page_size, uint32_t log2_page, const uint32_t *plan,
                        const uint32_t *off, const uint32_t *masks, uint8_t *slot, int n_sms, cudaStream_t st);
// KD: restore a staged group of stored pages.
int launch_codec_decode(const DecodeDesc *desc, uint64_t n_desc, const uint8_t *slot, uint32_t page_size, int n_sms,
                        cudaStream_t st);

// ---- host CRC32C math (crc_host.cpp), independent of oracle/ --------------
void build_tables(CrcTables *out);
// basis[8k + i] = tab[k][1 << i] of a 4x256 table (see ScanParams::basis)
void table_basis(const uint32_t (&tab)[4][256], uint32_t *basis32);
uint32_t zero_digest(uint64_t n);                 // Z(n)
uint32_t crc_shift(uint32_t reg, uint64_t nbytes);  // adv_nbytes(reg): reg(s, A|B) = crc_shift(reg(s, A), |B|) ^ reg(0, B)
uint32_t host_crc32c_update(uint32_t state, const void *p, uint64_t n);  // raw register update
bool crc_self_test();                            // "123456789" -> 0xE3069283 through the tables

}  // namespace gcr
