/*
 * oracle/gcr_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the
 * device-memory snapshot path (checkpoint -> page image + pagemap + digests,
 * and restore -> scatter + verify) of arXiv 2502.16631 (CRIUgpu).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (paper_2502_16631_b200/, libgcr.so) never links, imports or calls it,
 * and this file includes no header of the product: every struct layout below
 * is written out byte-by-byte from the format contract in DESIGN.md §3
 * (SURVEY.md §8(b)/(c)).
 *
 * What the paper fixes and what it does not.  PAPER.md §3.1.1
 * "Checkpointing the GPU state of CUDA tasks into host memory allocations"
 * and "Restore resources such as device memory back to the GPU" name
 * the operation; CRIU's page-granular memory dump ("pages scanned", P:432,
 * §5.3) and incremental/differential checkpointing (§7) name the
 * page scan and the dirty diff.  The paper prints no digest, page count or
 * byte of any image, so every rule here is the DESIGN.md reading (R-1..R-19)
 * and each one is pinned in tests/test_oracle_*.py against something other
 * than this file: RFC 3720 B.4 CRC32C vectors, the x86 SSE4.2 crc32
 * instruction, closed forms Z(n), brute force on tiny registries,
 * round-trip/chain/corruption invariants.
 *
 * Precision: all arithmetic is integer / GF(2); there is no floating point.
 *
 * Deliberately naive: byte-at-a-time Sarwate CRC, one page at a time, no
 * threads, no SIMD, no blocking or fusion beyond what c.1/c.2 state.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- status codes: numeric values fixed by the format contract */
enum {
    ORC_OK = 0, ORC_E_INVAL = 1, ORC_E_STATE = 2, ORC_E_TIMEOUT = 3, ORC_E_PEER = 4,
    ORC_E_LAYOUT = 5, ORC_E_CHAIN = 6, ORC_E_CORRUPT = 7, ORC_E_VERSION = 8,
    ORC_E_VERIFY = 9, ORC_E_NOMEM = 10
};
/* page classes (c.1 step 5) and pagemap flags (CRIU PE_PARENT=1<<0,
 * PE_PRESENT=1<<2; ZERO=1<<3 is ours, reading R-7) */
enum { ORC_CLASS_PRESENT = 0, ORC_CLASS_ZERO = 1, ORC_CLASS_PARENT = 2 };
enum { ORC_PE_PARENT = 1u << 0, ORC_PE_PRESENT = 1u << 2, ORC_PE_ZERO = 1u << 3 };
enum { ORC_FULL = 0, ORC_INCREMENTAL = 1 };

#define ORC_HEADER_BYTES 96u
#define ORC_ALLOC_REC_BYTES 24u
#define ORC_PAGEMAP_ENTRY_BYTES 16u
#define ORC_VERSION 1u
static const uint8_t ORC_MAGIC[8] = {'G', 'C', 'R', 'I', 'M', 'G', 0x00, 0x01};

/* ------------------------------------------------------------------------ */
/* CRC32C (Castagnoli), reading R-10: reflected polynomial 0x82F63B78, init
 * 0xFFFFFFFF, refin = refout = true, xorout 0xFFFFFFFF.  Sarwate byte table,
 * generated here from the polynomial by the textbook bit-at-a-time rule.   */
static uint32_t orc_table[256];
static int orc_table_ready = 0;

static void orc_init_table(void) {
    if (orc_table_ready) return;
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1u) ? (c >> 1) ^ 0x82F63B78u : (c >> 1);
        orc_table[i] = c;
    }
    orc_table_ready = 1;
}

static uint32_t orc_crc32c_update(uint32_t state, const uint8_t *p, uint64_t n) {
    for (uint64_t i = 0; i < n; i++) state = (state >> 8) ^ orc_table[(state ^ p[i]) & 0xFFu];
    return state;
}

/* CRC32C of n bytes. */
uint32_t orc_crc32c(const uint8_t *p, uint64_t n) {
    orc_init_table();
    return orc_crc32c_update(0xFFFFFFFFu, p, n) ^ 0xFFFFFFFFu;
}

/* ------------------------------------------------------------------------ */
/* c.1 steps 3-5 for ONE page: digest, zero test, classification.
 *   D = CRC32C(page bytes)                                   (step 3)
 *   Z = every byte == 0x00 (R-4: bytewise; -0.0f is not zero) (step 4)
 *   class = ZERO if Z; else PARENT if incremental and D == D_prev;
 *           else PRESENT                 (step 5; R-5 ZERO wins; R-6 dirty
 *                                          criterion is digest inequality) */
void orc_page_record(const uint8_t *page, uint64_t len, int mode, uint32_t d_prev,
                     uint32_t *digest_out, uint8_t *class_out) {
    uint32_t d = orc_crc32c(page, len);
    int all_zero = 1;
    for (uint64_t i = 0; i < len; i++) {
        if (page[i] != 0) { all_zero = 0; break; }
    }
    uint8_t cls;
    if (all_zero) cls = ORC_CLASS_ZERO;
    else if (mode == ORC_INCREMENTAL && d == d_prev) cls = ORC_CLASS_PARENT;
    else cls = ORC_CLASS_PRESENT;
    *digest_out = d;
    *class_out = cls;
}

static uint32_t orc_flag_of_class(uint8_t cls) {
    if (cls == ORC_CLASS_ZERO) return ORC_PE_ZERO;
    if (cls == ORC_CLASS_PARENT) return ORC_PE_PARENT;
    return ORC_PE_PRESENT;
}

/* little-endian fixed-width field writers/readers */
static void put_u32(uint8_t *p, uint32_t v) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static void put_u64(uint8_t *p, uint64_t v) { for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static uint32_t get_u32(const uint8_t *p) { uint32_t v = 0; for (int i = 0; i < 4; i++) v |= (uint32_t)p[i] << (8 * i); return v; }
static uint64_t get_u64(const uint8_t *p) { uint64_t v = 0; for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i); return v; }

/* page count of an allocation: m_a = ceil(bytes_a / P)            (c.1 step 2) */
static uint64_t pages_of(uint64_t bytes, uint32_t P) { return (bytes + P - 1) / P; }
/* true length of page p of an allocation: min(P, bytes_a - p*P)   (c.1 step 2) */
static uint64_t page_len(uint64_t bytes, uint32_t P, uint64_t p) {
    uint64_t rest = bytes - p * (uint64_t)P;
    return rest < P ? rest : P;
}

static int valid_page_size(uint32_t P) {
    return P >= 4096u && P <= 2097152u && (P & (P - 1u)) == 0;
}

/* ------------------------------------------------------------------------ */
/* f4 PAGE CODEC -- "data compression ... could further improve the efficiency
 * of checkpoint/restore operations" (§5.2; §7).  The paper names
 * the technique only; the code below is DESIGN.md reading R-19 ("byte-plane
 * dictionary code"), written out step by step:
 *
 *  A PRESENT page of L bytes (L % 16 == 0) is n = L/4 little-endian 32-bit
 *  words x_0..x_{n-1}.  Plane k (k = 0..3) is the sequence of byte k of every
 *  word.  For each plane: D_k = its distinct byte values in ascending order,
 *  d_k = |D_k|, b_k = ceil(log2 d_k) (0 when d_k == 1); packed section size
 *  S_p = pad16(d_k) + pad16(ceil(n*b_k/8)), raw section size S_r = pad16(n);
 *  mode_k = b_k if d_k <= 128 and S_p < S_r, else 8 (raw).
 *  Coded page = 16-byte header (byte k = mode_k; byte 4+k = d_k - 1 for a
 *  packed plane, 0 for a raw one; bytes 8..15 = 0) followed by the four plane
 *  sections in order: raw = the n plane bytes zero-padded to 16; packed = D_k
 *  zero-padded to 16, then code(i) = rank of plane value i in D_k as a b_k-bit
 *  field at bit position i*b_k (bit j of section byte m is bit 8m+j: LSB
 *  first), zero-padded to 16.  The page is stored coded iff its coded length C
 *  is < L, else raw: stored length == L <=> raw.
 *  Decoding a coded page: a MALFORMED header (a mode > 8; a raw plane with
 *  byte 4+k != 0; a packed plane with d_k > 128 or b_k != ceil(log2 d_k); a
 *  non-zero byte 8..15; section sizes not summing to the stored length)
 *  restores the page as zero bytes; a code >= d_k restores byte 0.  (Both
 *  sides implement this, so corrupted images restore identically; the
 *  restore's verify reports such pages.)                                     */
static uint64_t pad16(uint64_t x) { return (x + 15u) / 16u * 16u; }

static uint32_t ceil_log2(uint32_t d) {
    uint32_t b = 0;
    while ((1u << b) < d) b++;
    return b;
}

/* modes / dictionary sizes of a page's four planes; returns the coded length C */
static uint64_t orc_plan_page(const uint8_t *page, uint64_t len, uint8_t present[4][256], uint32_t d[4],
                              uint32_t mode[4]) {
    uint64_t n = len / 4, C = 16;
    for (int k = 0; k < 4; k++) {
        memset(present[k], 0, 256);
        for (uint64_t i = 0; i < n; i++) present[k][page[4 * i + k]] = 1;
        d[k] = 0;
        for (int v = 0; v < 256; v++) d[k] += present[k][v];
        uint32_t b = ceil_log2(d[k]);
        uint64_t sp = pad16(d[k]) + pad16((n * b + 7) / 8), sr = pad16(n);
        if (d[k] <= 128 && sp < sr) {
            mode[k] = b;
            C += sp;
        } else {
            mode[k] = 8;
            C += sr;
        }
    }
    return C;
}

/* Stored form of one page into out (capacity >= len); returns its length. */
uint64_t orc_encode_page(const uint8_t *page, uint64_t len, uint8_t *out) {
    uint8_t present[4][256];
    uint32_t d[4], mode[4];
    uint64_t n = len / 4;
    uint64_t C = orc_plan_page(page, len, present, d, mode);
    if (C >= len) {  /* raw */
        memcpy(out, page, len);
        return len;
    }
    memset(out, 0, C);
    for (int k = 0; k < 4; k++) {
        out[k] = (uint8_t)mode[k];
        out[4 + k] = mode[k] < 8 ? (uint8_t)(d[k] - 1) : 0;
    }
    uint64_t o = 16;
    for (int k = 0; k < 4; k++) {
        if (mode[k] == 8) {
            for (uint64_t i = 0; i < n; i++) out[o + i] = page[4 * i + k];
            o += pad16(n);
            continue;
        }
        uint8_t rank[256];
        uint32_t r = 0;
        for (int v = 0; v < 256; v++)
            if (present[k][v]) {
                out[o + r] = (uint8_t)v; /* dictionary, ascending */
                rank[v] = (uint8_t)r++;
            }
        o += pad16(d[k]);
        uint32_t b = mode[k];
        for (uint64_t i = 0; i < n; i++) {
            uint32_t code = rank[page[4 * i + k]];
            for (uint32_t j = 0; j < b; j++) {
                uint64_t pos = i * b + j;
                out[o + pos / 8] |= (uint8_t)(((code >> j) & 1u) << (pos % 8));
            }
        }
        o += pad16((n * b + 7) / 8);
    }
    return C;
}

/* Inverse of orc_encode_page: `stored` bytes (stored == len: raw) -> page. */
void orc_decode_page(const uint8_t *src, uint64_t stored, uint8_t *page, uint64_t len) {
    if (stored == len) {
        memcpy(page, src, len);
        return;
    }
    uint64_t n = len / 4;
    int malformed = stored < 16;
    uint64_t o = 16;
    uint64_t off[4];
    for (int k = 0; k < 4 && !malformed; k++) {
        uint32_t m = src[k], dm1 = src[4 + k];
        off[k] = o;
        if (m > 8) malformed = 1;
        else if (m == 8) {
            if (dm1 != 0) malformed = 1;
            o += pad16(n);
        } else {
            uint32_t dk = dm1 + 1;
            if (dk > 128 || ceil_log2(dk) != m) malformed = 1;
            o += pad16(dk) + pad16((n * m + 7) / 8);
        }
    }
    for (int j = 8; j < 16 && !malformed; j++)
        if (src[j] != 0) malformed = 1;
    if (!malformed && o != stored) malformed = 1;
    if (malformed) {
        memset(page, 0, len);
        return;
    }
    for (int k = 0; k < 4; k++) {
        uint32_t m = src[k];
        const uint8_t *sec = src + off[k];
        if (m == 8) {
            for (uint64_t i = 0; i < n; i++) page[4 * i + k] = sec[i];
            continue;
        }
        uint32_t dk = (uint32_t)src[4 + k] + 1;
        const uint8_t *codes = sec + pad16(dk);
        for (uint64_t i = 0; i < n; i++) {
            uint32_t code = 0;
            for (uint32_t j = 0; j < m; j++) {
                uint64_t pos = i * m + j;
                code |= (uint32_t)((codes[pos / 8] >> (pos % 8)) & 1u) << j;
            }
            page[4 * i + k] = code < dk ? sec[code] : 0;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* CHECKPOINT.
 *
 * Inputs: the registry in registration order (alloc_id[a], vaddr[a],
 * bytes[a]), page size P, the allocation contents, the mode, the parent
 * digest table d_prev (one u32 per page, required iff mode == INCREMENTAL),
 * the new generation and the parent generation (0 for FULL).
 *
 * Output: the canonical image stream
 *     header(96) || alloc table || pagemap || digests || data
 * malloc'ed into *out (caller frees with orc_free), length in *out_len.
 * Also, if digests_out != NULL, the new parent digest table (c.1 step 9),
 * which is the digest table in the stream.
 */
int orc_checkpoint_ex(uint32_t P, uint32_t n_allocs, const uint32_t *alloc_id,
                      const uint64_t *vaddr, const uint64_t *bytes,
                      const uint8_t *const *contents, int mode,
                      const uint32_t *d_prev, uint64_t n_prev,
                      uint64_t generation, uint64_t parent_generation, int compress,
                      uint8_t **out, uint64_t *out_len) {
    orc_init_table();
    *out = NULL;
    *out_len = 0;
    if (!valid_page_size(P) || n_allocs == 0) return ORC_E_INVAL;
    for (uint32_t a = 0; a < n_allocs; a++)
        if (bytes[a] == 0 || bytes[a] % 16 != 0 || vaddr[a] % 16 != 0) return ORC_E_INVAL; /* R-2 */

    /* step 2: enumerate pages, g over (a ascending, p ascending) */
    uint64_t n_pages = 0;
    for (uint32_t a = 0; a < n_allocs; a++) n_pages += pages_of(bytes[a], P);
    if (mode == ORC_INCREMENTAL && (d_prev == NULL || n_prev != n_pages)) return ORC_E_CHAIN; /* R-8 */

    uint32_t *D = (uint32_t *)malloc(n_pages * sizeof(uint32_t));
    uint8_t *cls = (uint8_t *)malloc(n_pages);
    uint64_t *stored = (uint64_t *)malloc(n_pages * sizeof(uint64_t)); /* f4: stored length per page */
    uint8_t *scratch = (uint8_t *)malloc(P);
    if (!D || !cls || !stored || !scratch) { free(D); free(cls); free(stored); free(scratch); return ORC_E_NOMEM; }

    /* steps 3-5: digest, zero test, classify every page */
    uint64_t g = 0, n_present = 0, n_zero = 0, n_parent = 0, image_bytes = 0;
    for (uint32_t a = 0; a < n_allocs; a++) {
        uint64_t m = pages_of(bytes[a], P);
        for (uint64_t p = 0; p < m; p++, g++) {
            uint64_t len = page_len(bytes[a], P, p);
            orc_page_record(contents[a] + p * (uint64_t)P, len, mode,
                            mode == ORC_INCREMENTAL ? d_prev[g] : 0u, &D[g], &cls[g]);
            if (cls[g] == ORC_CLASS_ZERO) n_zero++;
            else if (cls[g] == ORC_CLASS_PARENT) n_parent++;
            else {
                n_present++;
                /* step 6 with f4 (R-19): the page's stored form is its coded
                 * form if shorter, else its raw bytes */
                stored[g] = compress ? orc_encode_page(contents[a] + p * (uint64_t)P, len, scratch) : len;
                image_bytes += stored[g];
            }
        }
    }

    /* step 7: pagemap -- per allocation, maximal runs of equal class; runs
     * never cross allocations (even when contiguous in VA).  First count. */
    uint64_t n_entries = 0;
    g = 0;
    for (uint32_t a = 0; a < n_allocs; a++) {
        uint64_t m = pages_of(bytes[a], P);
        for (uint64_t p = 0; p < m; p++, g++)
            if (p == 0 || cls[g] != cls[g - 1]) n_entries++;
    }

    /* f4: one u32 stored length per PRESENT page after the digests (R-19) */
    uint64_t meta_bytes = ORC_HEADER_BYTES + (uint64_t)ORC_ALLOC_REC_BYTES * n_allocs +
                          ORC_PAGEMAP_ENTRY_BYTES * n_entries + 4u * n_pages + (compress ? 4u * n_present : 0u);
    uint64_t total = meta_bytes + image_bytes;
    uint8_t *s = (uint8_t *)calloc(total ? total : 1, 1);
    if (!s) { free(D); free(cls); free(stored); free(scratch); return ORC_E_NOMEM; }

    /* alloc table: {u64 vaddr; u64 bytes; u32 alloc_id; u32 reserved=0} */
    uint8_t *at = s + ORC_HEADER_BYTES;
    for (uint32_t a = 0; a < n_allocs; a++) {
        put_u64(at + 24u * a + 0, vaddr[a]);
        put_u64(at + 24u * a + 8, bytes[a]);
        put_u32(at + 24u * a + 16, alloc_id[a]);
        put_u32(at + 24u * a + 20, 0);
    }
    /* pagemap entries: {u64 vaddr; u32 nr_pages; u32 flags} */
    uint8_t *pm = at + (uint64_t)ORC_ALLOC_REC_BYTES * n_allocs;
    uint64_t e = 0;
    g = 0;
    for (uint32_t a = 0; a < n_allocs; a++) {
        uint64_t m = pages_of(bytes[a], P);
        uint64_t p = 0;
        while (p < m) {
            uint64_t q = p + 1;
            while (q < m && cls[g + (q - p)] == cls[g]) q++;
            put_u64(pm + 16u * e + 0, vaddr[a] + p * (uint64_t)P);
            put_u32(pm + 16u * e + 8, (uint32_t)(q - p));
            put_u32(pm + 16u * e + 12, orc_flag_of_class(cls[g]));
            e++;
            g += q - p;
            p = q;
        }
    }
    /* digests: one u32 LE per page, every class (R-9) */
    uint8_t *dg = pm + ORC_PAGEMAP_ENTRY_BYTES * n_entries;
    for (uint64_t i = 0; i < n_pages; i++) put_u32(dg + 4u * i, D[i]);

    /* f4 stored lengths, PRESENT pages in g order */
    uint8_t *cs = dg + 4u * n_pages;
    if (compress) {
        uint64_t i = 0;
        for (uint64_t q = 0; q < n_pages; q++)
            if (cls[q] == ORC_CLASS_PRESENT) put_u32(cs + 4u * i++, (uint32_t)stored[q]);
    }
    /* step 6: image data = concatenation in g order of PRESENT pages, true
     * lengths, no padding (f4: each page's stored form) */
    uint8_t *data = cs + (compress ? 4u * n_present : 0u);
    uint64_t cur = 0;
    g = 0;
    for (uint32_t a = 0; a < n_allocs; a++) {
        uint64_t m = pages_of(bytes[a], P);
        for (uint64_t p = 0; p < m; p++, g++) {
            if (cls[g] != ORC_CLASS_PRESENT) continue;
            uint64_t len = page_len(bytes[a], P, p);
            if (compress) cur += orc_encode_page(contents[a] + p * (uint64_t)P, len, data + cur);
            else {
                memcpy(data + cur, contents[a] + p * (uint64_t)P, len);
                cur += len;
            }
        }
    }

    /* step 8: header; meta_crc32c over header(with the field 0) || alloc
     * table || pagemap || digests */
    memcpy(s + 0, ORC_MAGIC, 8);
    put_u32(s + 8, ORC_VERSION);
    put_u32(s + 12, P);
    put_u64(s + 16, generation);
    put_u64(s + 24, mode == ORC_INCREMENTAL ? parent_generation : 0);
    put_u32(s + 32, n_allocs);
    put_u32(s + 36, (mode == ORC_INCREMENTAL ? 1u : 0u) | (compress ? 2u : 0u)); /* bit1: f4 coded */
    put_u64(s + 40, n_pages);
    put_u64(s + 48, n_present);
    put_u64(s + 56, n_zero);
    put_u64(s + 64, n_parent);
    put_u64(s + 72, n_entries);
    put_u64(s + 80, image_bytes);
    put_u32(s + 88, 0);
    put_u32(s + 92, 0);
    put_u32(s + 88, orc_crc32c(s, meta_bytes));

    free(D);
    free(cls);
    free(stored);
    free(scratch);
    *out = s;
    *out_len = total;
    return ORC_OK;
}

int orc_checkpoint(uint32_t P, uint32_t n_allocs, const uint32_t *alloc_id,
                   const uint64_t *vaddr, const uint64_t *bytes,
                   const uint8_t *const *contents, int mode,
                   const uint32_t *d_prev, uint64_t n_prev,
                   uint64_t generation, uint64_t parent_generation,
                   uint8_t **out, uint64_t *out_len) {
    return orc_checkpoint_ex(P, n_allocs, alloc_id, vaddr, bytes, contents, mode, d_prev, n_prev, generation,
                             parent_generation, 0, out, out_len);
}

void orc_free(void *p) { free(p); }

/* ------------------------------------------------------------------------ */
/* Parsed view of one stream (no copies). */
typedef struct {
    const uint8_t *s;
    uint64_t len;
    uint32_t page_size, n_allocs, flags;
    uint64_t generation, parent_generation, n_pages, n_present, n_zero, n_parent, n_entries,
        image_bytes;
    const uint8_t *allocs, *pagemap, *digests, *stored, *data; /* stored: f4 lengths or NULL */
} orc_view;

/* Validation, first part of c.2 step 1: framing, magic and meta CRC
 * (CORRUPT), then version (VERSION). */
static int orc_parse(const uint8_t *s, uint64_t len, orc_view *v) {
    if (len < ORC_HEADER_BYTES) return ORC_E_CORRUPT;
    if (memcmp(s, ORC_MAGIC, 8) != 0) return ORC_E_CORRUPT;
    v->s = s;
    v->len = len;
    v->page_size = get_u32(s + 12);
    v->generation = get_u64(s + 16);
    v->parent_generation = get_u64(s + 24);
    v->n_allocs = get_u32(s + 32);
    v->flags = get_u32(s + 36);
    v->n_pages = get_u64(s + 40);
    v->n_present = get_u64(s + 48);
    v->n_zero = get_u64(s + 56);
    v->n_parent = get_u64(s + 64);
    v->n_entries = get_u64(s + 72);
    v->image_bytes = get_u64(s + 80);
    /* declared sizes must frame the stream exactly (guard overflow first) */
    if (v->n_pages > len / 4 || v->n_entries > len / 16 || v->n_allocs > len / 24 || v->n_present > len / 4)
        return ORC_E_CORRUPT;
    uint64_t meta = ORC_HEADER_BYTES + 24ull * v->n_allocs + 16ull * v->n_entries + 4ull * v->n_pages +
                    ((v->flags & 2u) ? 4ull * v->n_present : 0ull);
    if (meta > len || len - meta != v->image_bytes) return ORC_E_CORRUPT;
    /* meta CRC with the field itself taken as 0 */
    uint32_t stored = get_u32(s + 88);
    uint8_t hdr[ORC_HEADER_BYTES];
    memcpy(hdr, s, ORC_HEADER_BYTES);
    put_u32(hdr + 88, 0);
    orc_init_table();
    uint32_t st = orc_crc32c_update(0xFFFFFFFFu, hdr, ORC_HEADER_BYTES);
    st = orc_crc32c_update(st, s + ORC_HEADER_BYTES, meta - ORC_HEADER_BYTES);
    if ((st ^ 0xFFFFFFFFu) != stored) return ORC_E_CORRUPT;
    if (get_u32(s + 8) != ORC_VERSION || (v->flags & ~3u) != 0) return ORC_E_VERSION; /* unknown flag bits */
    v->allocs = s + ORC_HEADER_BYTES;
    v->pagemap = v->allocs + 24ull * v->n_allocs;
    v->digests = v->pagemap + 16ull * v->n_entries;
    v->stored = (v->flags & 2u) ? v->digests + 4ull * v->n_pages : NULL;
    v->data = v->digests + 4ull * v->n_pages + ((v->flags & 2u) ? 4ull * v->n_present : 0ull);
    return ORC_OK;
}

/* Structural check of the pagemap against the image's own alloc table:
 * entries walk the pages in g order, each run inside one allocation, vaddr
 * at the run's first page, flags one of the three, counts and data length
 * consistent with the header.  Anything else is CORRUPT. */
static int orc_check_pagemap(const orc_view *v) {
    uint64_t e = 0, npres = 0, nzero = 0, npar = 0, bytes_present = 0, bytes_stored = 0;
    uint32_t P = v->page_size;
    if (!valid_page_size(P)) return ORC_E_CORRUPT;
    uint64_t total_pages = 0;
    for (uint32_t a = 0; a < v->n_allocs; a++) {
        uint64_t va = get_u64(v->allocs + 24ull * a), by = get_u64(v->allocs + 24ull * a + 8);
        if (by == 0) return ORC_E_CORRUPT;
        uint64_t m = pages_of(by, P);
        total_pages += m;
        uint64_t p = 0;
        while (p < m) {
            if (e >= v->n_entries) return ORC_E_CORRUPT;
            const uint8_t *pe = v->pagemap + 16ull * e;
            uint64_t eva = get_u64(pe);
            uint32_t nr = get_u32(pe + 8), fl = get_u32(pe + 12);
            if (eva != va + p * (uint64_t)P || nr == 0 || p + nr > m) return ORC_E_CORRUPT;
            if (fl != ORC_PE_PRESENT && fl != ORC_PE_ZERO && fl != ORC_PE_PARENT) return ORC_E_CORRUPT;
            for (uint64_t q = p; q < p + nr; q++) {
                if (fl == ORC_PE_PRESENT) {
                    uint64_t L = page_len(by, P, q);
                    bytes_present += L;
                    if (v->stored) { /* f4: raw (== L) or a coded form, a multiple of 16 shorter than L */
                        if (npres >= v->n_present) return ORC_E_CORRUPT;
                        uint64_t st = get_u32(v->stored + 4ull * npres);
                        if (st > L || (st != L && (st % 16 != 0 || st < 16))) return ORC_E_CORRUPT;
                        bytes_stored += st;
                    }
                    npres++;
                }
                else if (fl == ORC_PE_ZERO) nzero++;
                else npar++;
            }
            p += nr;
            e++;
        }
    }
    if (e != v->n_entries || total_pages != v->n_pages) return ORC_E_CORRUPT;
    if (npres != v->n_present || nzero != v->n_zero || npar != v->n_parent) return ORC_E_CORRUPT;
    if ((v->stored ? bytes_stored : bytes_present) != v->image_bytes) return ORC_E_CORRUPT;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* RESTORE of the chain streams[0..n_images) into the
 * registry (page size P, bytes[a]) whose contents are writable host buffers.
 *
 *  1. validate, in order: meta CRC, version, layout vs the registry, chain
 *     order (I_0 full; each parent_generation == previous generation);
 *  2. apply each image in chain order: PRESENT copies from the data cursor
 *     (true lengths), ZERO fills 0, PARENT skips (a PARENT in I_0 -> CHAIN);
 *     entries are mapped by allocation index (R-14);
 *  3. verify every page: CRC32C(page) == D_k[g]; count + first failing g.
 * Returns ORC_E_VERIFY iff the count is non-zero. */
int orc_restore(const uint8_t *const *streams, const uint64_t *lens, uint32_t n_images,
                uint32_t P, uint32_t n_allocs, const uint64_t *bytes,
                uint8_t *const *contents, uint64_t *verify_failures, uint64_t *first_bad) {
    orc_init_table();
    *verify_failures = 0;
    *first_bad = UINT64_MAX;
    if (n_images == 0 || n_images > 1024) return ORC_E_INVAL;
    orc_view views[1024];
    /* step 1: validate everything before writing anything */
    for (uint32_t k = 0; k < n_images; k++) {
        int st = orc_parse(streams[k], lens[k], &views[k]);
        if (st != ORC_OK) return st;
        st = orc_check_pagemap(&views[k]);
        if (st != ORC_OK) return st;
    }
    for (uint32_t k = 0; k < n_images; k++) {
        const orc_view *v = &views[k];
        if (v->page_size != P || v->n_allocs != n_allocs) return ORC_E_LAYOUT;
        for (uint32_t a = 0; a < n_allocs; a++)
            if (get_u64(v->allocs + 24ull * a + 8) != bytes[a]) return ORC_E_LAYOUT;
    }
    for (uint32_t k = 0; k < n_images; k++) {
        const orc_view *v = &views[k];
        if (k == 0) {
            if ((v->flags & 1u) != 0 || v->parent_generation != 0 || v->n_parent != 0) return ORC_E_CHAIN;
        } else {
            if ((v->flags & 1u) == 0 || v->parent_generation != views[k - 1].generation) return ORC_E_CHAIN;
        }
    }
    /* step 2: apply in chain order */
    for (uint32_t k = 0; k < n_images; k++) {
        const orc_view *v = &views[k];
        uint64_t e = 0, cursor = 0, ip = 0; /* ip: ordinal of the next PRESENT page */
        for (uint32_t a = 0; a < n_allocs; a++) {
            uint64_t m = pages_of(bytes[a], P);
            uint64_t p = 0;
            while (p < m) {
                const uint8_t *pe = v->pagemap + 16ull * e;
                uint32_t nr = get_u32(pe + 8), fl = get_u32(pe + 12);
                for (uint64_t q = p; q < p + nr; q++) {
                    uint64_t len = page_len(bytes[a], P, q);
                    uint8_t *dst = contents[a] + q * (uint64_t)P;
                    if (fl == ORC_PE_PRESENT) {
                        uint64_t st = v->stored ? get_u32(v->stored + 4ull * ip) : len;
                        orc_decode_page(v->data + cursor, st, dst, len); /* raw when st == len */
                        cursor += st;
                        ip++;
                    }
                    else if (fl == ORC_PE_ZERO) memset(dst, 0, len);
                    /* PARENT: skip */
                }
                p += nr;
                e++;
            }
        }
    }
    /* step 3: verify every page against the last image's digests */
    const orc_view *last = &views[n_images - 1];
    uint64_t g = 0;
    for (uint32_t a = 0; a < n_allocs; a++) {
        uint64_t m = pages_of(bytes[a], P);
        for (uint64_t p = 0; p < m; p++, g++) {
            uint64_t len = page_len(bytes[a], P, p);
            uint32_t d = orc_crc32c(contents[a] + p * (uint64_t)P, len);
            if (d != get_u32(last->digests + 4ull * g)) {
                if (*verify_failures == 0) *first_bad = g;
                (*verify_failures)++;
            }
        }
    }
    return *verify_failures ? ORC_E_VERIFY : ORC_OK;
}
