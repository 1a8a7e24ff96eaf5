/*
 * include/gcr.h -- C-ABI of libgcr.so, the B200-native device-memory
 * snapshot engine built from arXiv 2502.16631 (CRIUgpu).
 *
 * The paper's CUDA plugin drives four driver actions (§3.1.1,
 * P:157-173): "Locking all CUDA APIs affecting the GPU state ... waiting for
 * active operations ... to complete" with "a timeout (10 seconds by
 * default)"; "Checkpointing the GPU state of CUDA tasks into host
 * memory allocations"; "Restore resources such as device memory back
 * to the GPU, memory mappings to their original addresses"; "Unlock
 * driver APIs", invoked in the order PAUSE_DEVICES -> CHECKPOINT_DEVICES
 * -> RESUME_DEVICES_LATE (§3.1.3).  This library realises the
 * device-memory part of that protocol over an explicitly REGISTERED set of
 * device allocations: lock -> checkpoint -> (restore) -> unlock.
 *
 * Conventions (apply to every call):
 *  - Every call returns gcr_status.  No exception crosses the ABI; the
 *    library never calls exit()/abort().  On error, gcr_last_error(ctx) holds
 *    a one-line message (owned by ctx, valid until the next call on ctx).
 *  - Pointers named `dptr` are CUDA device addresses of the ctx's device; every
 *    other pointer is a host pointer.  The caller owns everything it passes in.
 *  - A gcr_ctx is single-threaded: one per (process, device).  Every call does
 *    cudaSetDevice(device) and shares the primary context (PyTorch's).
 *  - Byte layouts are little-endian, fixed width, naturally aligned; see
 *    DESIGN.md §3 for the format contract.
 *  - Phase machine (SPEC S:161 analog):
 *        register/unregister/watch_stream/reserve_host : RUNNING
 *        lock       : RUNNING -> LOCKED           (TIMEOUT: stays RUNNING)
 *        checkpoint : LOCKED -> CHECKPOINTED      (failure: stays LOCKED)
 *        release    : CHECKPOINTED -> RELEASED   (device memory freed, VAs kept)
 *        restore    : LOCKED|CHECKPOINTED|RELEASED -> LOCKED
 *        unlock     : LOCKED|CHECKPOINTED -> RUNNING   (not from RELEASED)
 *    Any other (phase, call) pair returns GCR_E_STATE and changes nothing.
 */
#ifndef GCR_H
#define GCR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gcr_ctx gcr_ctx;
typedef struct gcr_image gcr_image;

typedef enum {
    GCR_OK = 0,
    GCR_E_INVAL = 1,    /* bad argument: null pointer, bytes == 0, dptr or bytes not a
                           multiple of 16 (reading R-2), overlap with a registered
                           allocation, pointer not device memory of the ctx's
                           device, page size not a power of two in [4 KiB, 2 MiB] (R-1) */
    GCR_E_STATE = 2,    /* call not legal in the current phase (table above) */
    GCR_E_TIMEOUT = 3,  /* lock: watched streams not idle within lock_timeout_ms */
    GCR_E_PEER = 4,     /* reserved for multi-rank helpers: another rank failed */
    GCR_E_LAYOUT = 5,   /* image page size / allocation count / sizes differ from the
                           registry (SPEC S:145 TopologyMismatch; "same type/order") */
    GCR_E_CHAIN = 6,    /* chain does not start with a full image, parent_generation link
                           broken, PARENT page in a full image, or INCREMENTAL with no
                           parent digest state (reading R-8) */
    GCR_E_CORRUPT = 7,  /* meta_crc32c mismatch or inconsistent framing */
    GCR_E_VERSION = 8,  /* unknown image format version */
    GCR_E_VERIFY = 9,   /* restore: at least one page digest differs after the scatter */
    GCR_E_NOMEM = 10,   /* device or pinned host allocation failed */
    GCR_E_CUDA = 11,    /* a CUDA runtime call failed; message in gcr_last_error */
    GCR_E_IO = 12       /* storage tier: open/read/write/sync of an image file failed (errno
                           text in gcr_last_error) */
} gcr_status;

typedef enum { GCR_RUNNING = 0, GCR_LOCKED = 1, GCR_CHECKPOINTED = 2, GCR_RELEASED = 3 } gcr_phase;
typedef enum { GCR_FULL = 0, GCR_INCREMENTAL = 1 } gcr_mode;

/* Page classes and pagemap flags.  PARENT/PRESENT
 * sit at CRIU's PE_PARENT / PE_PRESENT bit positions; ZERO is ours (R-7). */
#define GCR_PE_PARENT (1u << 0)
#define GCR_PE_PRESENT (1u << 2)
#define GCR_PE_ZERO (1u << 3)

typedef struct {
    uint32_t page_size;       /* power of two in [4096, 2097152]; default 65536 (R-1) */
    uint32_t n_copy_streams;  /* copy streams for drain/restore; default 2, 1..8 */
    uint64_t chunk_bytes;     /* registry bytes scanned per pipeline chunk, also the staging slot
                                 size; default 1 GiB; multiple of page_size, <= 2 GiB */
    uint32_t n_staging_slots; /* device staging slots of chunk_bytes each; 0 (default) = one per
                                 copy stream, else n_copy_streams..16.  Checkpoint chunk i packs
                                 into slot i mod n, so its pack waits only for chunk i - n's
                                 drain; more slots let packs run further ahead of the drain. */
    uint32_t verify;          /* 1 (default) = restore re-reads every page and checks its digest
                                 (reading R-11); 0 = no verify pass (then restore never returns
                                 GCR_E_VERIFY) */
    uint64_t lock_timeout_ms; /* default 10000 -- "10 seconds by default" (R-12) */
    uint64_t direct_min_bytes;/* PRESENT runs of at least this many bytes move by DMA directly
                                 between the allocation and the pinned image (no staging, no
                                 pack/scatter kernel); shorter runs are packed (checkpoint) or
                                 scattered (restore) through the staging slots.  Checkpoint runs
                                 are built from whole 64 KiB tiles whose pages are all PRESENT
                                 (a tile mixing classes is always packed); restore runs are
                                 pagemap runs.  Default 16 MiB (shorter DMAs lose link
                                 efficiency); 0 = every eligible run direct;
                                 UINT64_MAX = every run staged.  The image bytes are identical
                                 either way. */
    uint32_t compress;        /* 0 (default) = PRESENT pages stored raw; 1 = f4 page codec: every
                                 PRESENT page is stored in its byte-plane dictionary form when that
                                 is shorter (R-19; "data compression"), encoded on
                                 the GPU before the drain and decoded on the GPU after the H2D.
                                 Digests, classes and the pagemap are unchanged; the image gets a
                                 stored-length table and header flag bit 1.  All PRESENT data then
                                 moves through the staging slots (direct_min_bytes is unused). */
    uint32_t in_scan_pack;    /* f1: 0 (default) = PRESENT pages reach the image
                                 through the staged / direct pipeline (K2 plan, K4 pack, copy-engine
                                 D2H); 1 = incremental checkpoints let the scan kernel itself write
                                 every PRESENT page straight into the pinned image (mapped memory;
                                 image offsets from per-CTA aggregates + a per-chunk base, no pack, no
                                 staging, no data D2H); 2 = every checkpoint does (full ones too).
                                 Measured: 1 is 3-7 % slower than 0 on C4 1-5 %
                                 dirty -- the scan's own PCIe stores couple it to the link -- so 0 is
                                 the default.  Ignored when compress = 1.  The image bytes are
                                 identical either way. */
} gcr_config;

/* Statistics of the most recent lock / checkpoint / restore / unlock
 * (SURVEY §5 "Metrics": the CRIU statistics of P:369-377 mapped to this path).
 * *_host_ns are host steady_clock durations of the whole ABI call; *_dev_ns are
 * sums of CUDA-event durations of the named kernels on the stream they ran on. */
typedef struct {
    uint64_t lock_ns, unlock_ns;                 /* host */
    uint64_t checkpoint_ns;                      /* host: gcr_checkpoint entry -> image in host memory */
    uint64_t restore_ns;                         /* host: gcr_restore entry -> verified */
    uint64_t scan_dev_ns;                        /* K1 scan_digest_classify, all chunks */
    uint64_t scan_launches;                      /* K1 launches in the last checkpoint */
    uint64_t scan_bytes;                         /* registered bytes K1 read (= R) */
    uint64_t compact_dev_ns;                     /* K2 compaction + K3 pagemap */
    uint64_t pack_dev_ns;                        /* K4 pack (sum over chunks) */
    uint64_t drain_ns;                           /* host: first D2H issued -> last D2H done */
    uint64_t restore_h2d_ns;                     /* host: first H2D issued -> last H2D done */
    uint64_t scatter_dev_ns;                     /* K6 scatter + K7 zero fill */
    uint64_t verify_dev_ns;                      /* K8 verify scan */
    uint64_t verify_launches;
    uint64_t pages_scanned, pages_zero, pages_parent, pages_written; /* last checkpoint */
    uint64_t image_bytes;                        /* last checkpoint: PRESENT bytes drained */
    uint64_t n_entries;                          /* last checkpoint: pagemap entries */
    uint64_t verify_failures;                    /* last restore */
    uint64_t first_bad_page;                     /* last restore: UINT64_MAX if none */
    uint64_t restore_h2d_bytes;                  /* last restore: image bytes copied H2D */
    uint64_t kernel_launches;                    /* cumulative: every kernel libgcr launched */
    uint64_t pinned_alloc_ns;                    /* cumulative: time spent in cudaHostAlloc */
    uint64_t direct_bytes;                       /* last checkpoint: image bytes drained straight from
                                                    the allocations (the rest was packed) */
    uint64_t restore_direct_bytes;               /* last restore: image bytes copied straight into
                                                    the allocations (the rest was scattered) */
    uint64_t release_ns;                         /* host: last gcr_release (unmap + release) */
    uint64_t remap_ns;                           /* host: last restore's re-create + re-map (0 if
                                                    the memory was resident) */
    uint64_t released_bytes;                     /* last gcr_release: physical bytes returned */
    uint64_t present_raw_bytes;                  /* last checkpoint: PRESENT bytes before coding (==
                                                    image_bytes unless compress) */
    uint64_t codec_dev_ns;                       /* last checkpoint: f4 plan + offsets + encode kernels */
    uint64_t decode_dev_ns;                      /* last restore: f4 decode kernels */
} gcr_stats;

/* gcr_image_hdr -- 96 bytes, offsets: magic 0, version 8, page_size 12,
 * generation 16, parent_generation 24, n_allocs 32, flags 36, n_pages 40,
 * n_present 48, n_zero 56, n_parent 64, n_entries 72, image_bytes 80,
 * meta_crc32c 88, reserved 92.  meta_crc32c = CRC32C over header (with this
 * field 0) || alloc table || pagemap || digests [|| stored lengths, f4]
 * (SPEC S:298 analog); image_bytes = length of the data section (for an f4
 * image the sum of the stored lengths).  This is
 * the analog of the paper's inventory flag "contains GPU state". */
typedef struct {
    char magic[8];               /* "GCRIMG\0\1" */
    uint32_t version;            /* 1 */
    uint32_t page_size;
    uint64_t generation;         /* 1, 2, ... per ctx */
    uint64_t parent_generation;  /* 0 for a full image */
    uint32_t n_allocs;
    uint32_t flags;              /* bit0 = incremental, bit1 = f4 coded (stored-length table present);
                                    other bits: GCR_E_VERSION */
    uint64_t n_pages, n_present, n_zero, n_parent, n_entries, image_bytes;
    uint32_t meta_crc32c;
    uint32_t reserved;           /* 0 */
} gcr_image_hdr;

/* alloc table record (24 B) -- registration order (reading R-3) */
typedef struct {
    uint64_t vaddr;
    uint64_t bytes;
    uint32_t alloc_id;
    uint32_t reserved;  /* 0 */
} gcr_alloc_rec;

/* pagemap entry (16 B) -- one per maximal run of equal class inside one
 * allocation (c.1 step 7); CRIU pagemap_entry analog. */
typedef struct {
    uint64_t vaddr;     /* device address of the run's first page at checkpoint time */
    uint32_t nr_pages;
    uint32_t flags;     /* exactly one of GCR_PE_PRESENT / GCR_PE_ZERO / GCR_PE_PARENT */
} gcr_pagemap_entry;

/* ---- context ------------------------------------------------------------ */

/* Fill *out with the defaults above.  GCR_E_INVAL if out is NULL. */
gcr_status gcr_config_default(gcr_config *out);

/* Create a context on CUDA device `cuda_device` (cfg may be NULL = defaults).
 * Allocates the device staging slots (n_copy_streams x chunk_bytes), the copy
 * streams and small pinned control buffers.  *out owned by the caller, freed
 * with gcr_destroy.  GCR_E_INVAL (bad config), GCR_E_NOMEM, GCR_E_CUDA. */
gcr_status gcr_create(int cuda_device, const gcr_config *cfg, gcr_ctx **out);

/* Free the context, its staging, device digest tables, pinned pool and every
 * gcr_image it still owns.  Never frees registered (caller-owned) memory. */
gcr_status gcr_destroy(gcr_ctx *ctx);

/* Register [dptr, dptr+bytes) as one allocation (RUNNING only).  The
 * allocation gets the next alloc_id; registration order is the page order
 * (R-3).  The memory stays caller-owned and must stay allocated while
 * registered.  Registering drops the incremental parent state (the layout
 * changed).  GCR_E_INVAL: see the enum. */
gcr_status gcr_register(gcr_ctx *ctx, uint64_t dptr, uint64_t bytes, uint32_t *alloc_id_out);

/* Remove a registered allocation (RUNNING only).  GCR_E_INVAL if unknown. */
gcr_status gcr_unregister(gcr_ctx *ctx, uint32_t alloc_id);

/* Add a CUDA stream (cudaStream_t, may be 0 = legacy default stream) that
 * lock must see idle (RUNNING only).  With no watched stream, lock waits for
 * the whole device: every stream of the process, blocking or non-blocking
 * (cudaDeviceSynchronize on a helper thread, bounded by lock_timeout_ms).
 * Not owned by the library. */
gcr_status gcr_watch_stream(gcr_ctx *ctx, void *cuda_stream);

/* Pre-pin `bytes` of host memory for images (RUNNING only), so checkpoints do
 * not pay cudaHostAlloc inside the locked window.  Cumulative.
 * GCR_E_NOMEM if pinning fails. */
gcr_status gcr_reserve_host(gcr_ctx *ctx, uint64_t bytes);

/* RUNNING -> LOCKED.  Waits (polling, no busy host spin beyond 50 us sleeps)
 * until every watched stream is idle, bounded by lock_timeout_ms ("waiting for
 * active operations ... to complete", "timeout (10 seconds by default)",
 * P:160).  On expiry returns GCR_E_TIMEOUT with phase RUNNING and nothing
 * changed (rollback, P:160 / SPEC S:126).  Cooperative contract (DESIGN.md,
 * deviation 1): between lock and unlock the caller enqueues no work that writes
 * registered memory. */
gcr_status gcr_lock(gcr_ctx *ctx);

/* LOCKED -> CHECKPOINTED: snapshot every registered allocation into a NEW
 * image in pinned host memory.  Steps (SURVEY §8(a)
 * A1-A7): page table, scan + CRC32C + zero test + dirty diff (K1), compaction
 * and pagemap (K2/K3), pack (K4) and multi-stream pinned drain (K5) overlapped
 * with the scan of the next chunk.  GCR_INCREMENTAL diffs against the digest
 * table of the ctx's last checkpoint or restore (R-8): GCR_E_CHAIN if there is
 * none.  *out is owned by the ctx until gcr_image_free (older images stay
 * valid: chains).  On any failure the phase stays LOCKED, no image is
 * returned and the parent digest state is unchanged. */
gcr_status gcr_checkpoint(gcr_ctx *ctx, gcr_mode mode, gcr_image **out);
/* (checkpoint and restore both first wait for caller work already enqueued on
 * the watched streams -- or, with none watched, on the whole device -- so they
 * are ordered after it even though the library's streams are non-blocking.) */

/* CHECKPOINTED -> LOCKED: undo the ctx's LAST checkpoint, whose image `img`
 * is freed, and restore the parent digest state it replaced (the next
 * incremental diffs against the previous parent again, generations are
 * re-issued).  Used by the multi-rank helpers when another rank's checkpoint
 * failed, so every rank is back where it was before the attempt (all or
 * nothing).  GCR_E_STATE if not CHECKPOINTED (e.g. after release or
 * unlock), GCR_E_INVAL if img is not the last checkpoint's image. */
gcr_status gcr_checkpoint_abort(gcr_ctx *ctx, gcr_image *img);

/* ---- releasable device memory ----------------------------
 * The paper's checkpoint action leaves the process "releasing all GPU
 * resources" and its restore maps device memory "back to the GPU,
 * memory mappings to their original addresses".  Memory from
 * gcr_mem_alloc is built from CUDA virtual-memory-management pieces (a
 * reserved VA range + a physical allocation mapped into it), so the library
 * can return the physical memory to the driver while keeping the VA range
 * reserved, and later back the SAME addresses with fresh physical memory:
 * pointers held by the application (tensors, pointer tables) stay valid. */

/* Allocate `bytes` (> 0) of device memory on the ctx's device, rounded up to
 * the driver's allocation granularity (2 MiB on B200), readable and writable
 * from the ctx's device (RUNNING only).  *dptr_out gets the address (2 MiB
 * aligned).  It is NOT registered: call gcr_register on it (or on sub-ranges)
 * as with any allocation.  Owned by the ctx: freed by gcr_mem_free or
 * gcr_destroy.  GCR_E_INVAL (null, bytes == 0), GCR_E_STATE, GCR_E_NOMEM,
 * GCR_E_CUDA (driver VMM entry points unavailable). */
gcr_status gcr_mem_alloc(gcr_ctx *ctx, uint64_t bytes, uint64_t *dptr_out);

/* Free memory from gcr_mem_alloc (RUNNING only).  GCR_E_INVAL if dptr is not
 * the start of such a block or any registered allocation lies inside it. */
gcr_status gcr_mem_free(gcr_ctx *ctx, uint64_t dptr);

/* CHECKPOINTED -> RELEASED: return the physical memory behind every registered
 * allocation to the driver, keeping the virtual address ranges reserved
 * (P:162-164).  Every registered allocation must lie in a gcr_mem_alloc block
 * and every block that holds one must be covered completely by registered
 * allocations (bytes outside the registry would be lost): otherwise
 * GCR_E_INVAL and nothing changes.  From RELEASED only gcr_restore (which first
 * re-backs the same addresses, then applies the chain) and gcr_destroy are
 * legal; unlock returns GCR_E_STATE (the memory is gone: SPEC S:180).
 * GCR_E_CUDA if the driver refuses an unmap (the phase is then RELEASED if any
 * block was released). */
gcr_status gcr_release(gcr_ctx *ctx);

/* LOCKED|CHECKPOINTED|RELEASED -> LOCKED: apply images chain[0..n) in order into the
 * registered allocations: PRESENT pages copied H2D and scattered (K6;
 * f4-coded images: decoded, KD), ZERO pages filled (K7), PARENT pages skipped.
 * For a coded chain[0] the first staging group (its data prefix) is copied into
 * the ctx's own staging memory before validation -- never into a registered
 * allocation -- so it overlaps the host's checks; entries map to allocations by
 * index, so allocations may live at new addresses (R-14).  Then every page's
 * CRC32C is recomputed and compared with chain[n-1]'s digests (K8, R-11).
 * Validation happens before any write, in order: meta CRC (CORRUPT), version
 * (VERSION), layout vs registry (LAYOUT), chain order (CHAIN).  After a
 * successful restore the ctx's parent digest state is chain[n-1]'s.  From
 * RELEASED, after validation, every released block is backed again at its
 * original address before the chain is applied -- the chain starts
 * with a full image, which writes every page.
 * Failure: a validation error (CORRUPT, VERSION, LAYOUT, CHAIN, INVAL) changes
 * nothing.  Once writes have begun, any failure (GCR_E_VERIFY with counts in
 * gcr_get_stats verify_failures / first_bad_page, GCR_E_NOMEM, GCR_E_CUDA)
 * leaves the memory content undefined and drops the parent digest state (an
 * incremental then returns GCR_E_CHAIN); the phase becomes LOCKED, or stays
 * RELEASED when the restore started from RELEASED (unlock refused until a
 * restore succeeds). */
gcr_status gcr_restore(gcr_ctx *ctx, gcr_image *const *chain, uint32_t n);

/* LOCKED|CHECKPOINTED -> RUNNING.  CHECKPOINTED keeps memory resident,
 * so unlock without restore is legal (deviation 2). */
gcr_status gcr_unlock(gcr_ctx *ctx);

gcr_status gcr_get_phase(const gcr_ctx *ctx, gcr_phase *out);
gcr_status gcr_get_stats(const gcr_ctx *ctx, gcr_stats *out);

/* The ctx's compute stream (cudaStream_t) on which K1/K2/K3/K8 run and into
 * which every copy stream is joined before checkpoint/restore return; lets a
 * caller bracket calls with its own CUDA events.  Not owned by the caller. */
gcr_status gcr_ctx_stream(const gcr_ctx *ctx, void **cuda_stream_out);

/* Host-link roofline probe (SURVEY §8(d) d.2 BW_d2h / BW_h2d) over the SAME
 * pinned memory images use: takes the pinned pool's first free range of
 * `bytes` (where the next image's data buffer lands; grows the pool if none),
 * times 3 copies between it and staging slot 0 in each direction on copy
 * stream 0 with CUDA events (after one warm-up copy), and returns the GB/s
 * (1e9 B/s).  Any phase; nothing else may run on the ctx meanwhile.
 * GCR_E_INVAL (null outputs, bytes == 0 or > chunk_bytes), GCR_E_NOMEM,
 * GCR_E_CUDA. */
gcr_status gcr_probe_link(gcr_ctx *ctx, uint64_t bytes, double *d2h_gbs, double *h2d_gbs);

/* Message of the last failed call on ctx ("" if none).  Owned by ctx. */
const char *gcr_last_error(const gcr_ctx *ctx);

/* ---- image accessors: every pointer is owned by the image and valid until
 * gcr_image_free / gcr_destroy.  GCR_E_INVAL on NULL arguments. ----------- */
gcr_status gcr_image_header(const gcr_image *img, gcr_image_hdr *out);
gcr_status gcr_image_allocs(const gcr_image *img, const gcr_alloc_rec **p, uint32_t *n);
gcr_status gcr_image_pagemap(const gcr_image *img, const gcr_pagemap_entry **p, uint64_t *n);
gcr_status gcr_image_digests(const gcr_image *img, const uint32_t **p, uint64_t *n);
/* PRESENT page bytes, concatenated in page order (c.1 step 6); pinned host.
 * For an f4 image (flags bit 1) every page's stored form (R-19). */
gcr_status gcr_image_data(const gcr_image *img, const uint8_t **p, uint64_t *bytes);
/* f4 images: the stored length of every PRESENT page, in page order (n =
 * n_present; raw pages have stored length == page length).  Other images:
 * *p = NULL, *n = 0. */
gcr_status gcr_image_stored(const gcr_image *img, const uint32_t **p, uint64_t *n);
gcr_status gcr_image_free(gcr_image *img);

/* Canonical byte stream = header(96) || alloc table || pagemap || digests ||
 * [stored lengths, f4 images only] || data: exactly what the oracle writes for
 * the same input.  meta_crc32c covers everything before the data. */
gcr_status gcr_image_stream_size(const gcr_image *img, uint64_t *bytes);
/* Write the stream into caller-owned dst of capacity cap (GCR_E_INVAL if too small). */
gcr_status gcr_image_serialize(const gcr_image *img, void *dst, uint64_t cap);
/* Copy a stream into a new ctx-owned image in pinned memory after checking
 * framing, meta CRC (CORRUPT) and version (VERSION).  Usable in any phase. */
gcr_status gcr_image_import(gcr_ctx *ctx, const void *stream, uint64_t bytes, gcr_image **out);

/* ---- storage tier: the paper's "memory write time -- the
 * time to save the memory state to persistent storage" and restore
 * "from storage".  The file holds exactly the canonical stream
 * (gcr_image_serialize); it is written and read by n_threads threads (0 = 8)
 * with positional I/O on disjoint ranges, straight from / into the image's
 * pinned buffers (no staging copy of the whole stream). ------------------- */
#define GCR_IO_SYNC 1u  /* fdatasync before returning (durable), then drop the file's page cache so a
                           later read comes from the device */

/* Create/truncate `path` and write img's canonical stream.  GCR_E_INVAL (null
 * arguments), GCR_E_IO (errno text in gcr_last_error of the image's ctx). */
gcr_status gcr_image_write_file(const gcr_image *img, const char *path, uint32_t n_threads, uint32_t flags);

/* Read a stream file into a new ctx-owned image in pinned memory (any phase):
 * framing, meta CRC (GCR_E_CORRUPT) and version (GCR_E_VERSION) are checked
 * as in gcr_image_import; the file size must equal the stream size
 * (GCR_E_CORRUPT otherwise).  GCR_E_IO if the file cannot be opened/read,
 * GCR_E_NOMEM if pinning fails. */
gcr_status gcr_image_read_file(gcr_ctx *ctx, const char *path, uint32_t n_threads, gcr_image **out);

#ifdef __cplusplus
}
#endif
#endif /* GCR_H */
