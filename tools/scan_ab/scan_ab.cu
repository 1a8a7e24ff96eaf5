// Same-box A/B of the scan kernel (K8 = k_scan in verify mode) between two
// source trees: compiled once per tree (SCAN_SRC = its csrc directory) into
// its own shared library exposing scan_ab_time(); tools/scan_ab.py loads both
// and alternates them on the same device buffer.  Diagnostics only.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <vector>

#include "kernels.cu"  // the tree's kernels + launchers (namespace gcr)

namespace gcr {
void build_tables(CrcTables *out);
uint32_t zero_digest(uint64_t n);
#ifndef SCAN_AB_R1
void table_basis(const uint32_t (&tab)[4][256], uint32_t *basis32);
#endif
}  // namespace gcr

extern "C" int scan_ab_time(uint64_t dptr, uint64_t bytes, uint32_t P, int iters, float *ms_out) {
    using namespace gcr;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    AllocDev a{};
    a.base = dptr;
    a.bytes = bytes;
    a.n_pages = (uint32_t)((bytes + P - 1) / P);
    a.n_tiles = P <= kTileBytes ? (uint32_t)((a.n_pages + kTileBytes / P - 1) / (kTileBytes / P)) : a.n_pages * (P / kTileBytes);
    a.tail_len = (uint32_t)(bytes - (uint64_t)(a.n_pages - 1) * P);
    a.z_tail = zero_digest(a.tail_len);
    a.n_rows = (uint64_t)(a.n_pages - 1) * (P / kRowBytes) + (a.tail_len + kRowBytes - 1) / kRowBytes;
    AllocDev *ad;
    cudaMalloc(&ad, sizeof a);
    cudaMemcpy(ad, &a, sizeof a, cudaMemcpyHostToDevice);
    uint64_t cr[2] = {0, a.n_rows};
    uint64_t *crd;
    cudaMalloc(&crd, 16);
    cudaMemcpy(crd, cr, 16, cudaMemcpyHostToDevice);
    CrcTables *th = new CrcTables;
    build_tables(th);
    CrcTables *td;
    cudaMalloc(&td, sizeof(CrcTables));
    cudaMemcpy(td, th, sizeof(CrcTables), cudaMemcpyHostToDevice);
    const uint64_t workers = scan_workers(nsm, 0);
    unsigned long long *fold, *misc;
    uint32_t *sync, *dref;
    cudaMalloc(&fold, 8 * workers);
    cudaMemset(fold, 0, 8 * workers);
    cudaMalloc(&sync, 16);
    cudaMemset(sync, 0, 16);
    cudaMalloc(&misc, 16);
    cudaMalloc(&dref, 4ull * a.n_pages);
    cudaMemset(dref, 0, 4ull * a.n_pages);
    ScanParams sp{};
    sp.allocs = ad;
    sp.n_allocs = 1;
    sp.chunk_rows = crd;
    sp.n_chunks = 1;
    sp.chunk_arrive = sync;
    sp.chunk_done = sync + 1;
    sp.workers = workers;
    sp.fold = FoldSlots{fold};
    sp.page_size = P;
    uint32_t lg = 0;
    while ((1u << lg) < P) lg++;
    sp.log2_page = lg;
    sp.z_page = zero_digest(P);
    sp.mode = kScanVerify;
    sp.d_ref = dref;
    sp.verify_count = misc;
    sp.first_bad = misc + 1;
    sp.tables = td;
    sp.prefetch = scan_prefetch_bytes();
#ifndef SCAN_AB_R1
    table_basis(th->braid, sp.basis[0]);
    table_basis(th->t4, sp.basis[1]);
    table_basis(th->a16, sp.basis[2]);
    table_basis(th->a32, sp.basis[3]);
    table_basis(th->a64, sp.basis[4]);
    table_basis(th->a128, sp.basis[5]);
    table_basis(th->a256, sp.basis[6]);
#endif
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float total = 0;
    for (int it = 0; it < iters + 1; it++) {
        sp.epoch = it + 1;
        cudaEventRecord(e0, st);
        if (launch_scan(sp, nsm, st) < 0) return -1;
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it) total += ms;  // first launch: warm-up
    }
    *ms_out = total / iters;
    cudaFree(ad); cudaFree(crd); cudaFree(td); cudaFree(fold); cudaFree(sync); cudaFree(misc); cudaFree(dref);
    delete th;
    cudaStreamDestroy(st);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
