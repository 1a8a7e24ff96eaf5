// tma_copy.cu -- standalone microbenchmark: device-to-device copy of 64 KiB
// pieces (the K4 pack / K6 scatter access pattern) by
//   (v) the 16-byte vector copy K6 uses (256 threads, 4 x 16 B in flight per thread),
//   (t) TMA bulk copies: per issuing lane a ring of NSTG shared-memory stages,
//       cp.async.bulk global->shared (mbarrier complete_tx) then
//       cp.async.bulk shared->global (bulk_group), the stage reloaded once the
//       store that read it has finished reading (wait_group.read),
//   (c) cudaMemcpyAsync D2D (copy engines), for context.
// Pieces are permuted (src piece k -> dst piece perm(k)) so both sides are
// gathers/scatters like the real kernels.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_copy/tma_copy tools/tma_copy/tma_copy.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) {                                                        \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                               \
        }                                                                               \
    } while (0)

constexpr uint64_t kPiece = 65536;

__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ uint64_t dst_piece(uint64_t k, uint64_t n) { return (k * 40503ull) % n; }  // n odd

__global__ void __launch_bounds__(256) k_vec(const uint8_t *src, uint8_t *dst, uint64_t n) {
    for (uint64_t u = blockIdx.x; u < n; u += gridDim.x) {
        const uint8_t *s = src + u * kPiece;
        uint8_t *d = dst + dst_piece(u, n) * kPiece;
        constexpr int U = 4;
        const uint32_t stride = blockDim.x * 16u;
        for (uint64_t off = threadIdx.x * 16u; off < kPiece; off += U * stride) {
            uint4 v[U];
#pragma unroll
            for (int w = 0; w < U; w++) v[w] = ldg_stream(s + off + w * stride);
#pragma unroll
            for (int w = 0; w < U; w++) *reinterpret_cast<uint4 *>(d + off + w * stride) = v[w];
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One issuing lane per warp; warp w of CTA b owns "lanes" (b * W + w) of the
// grid and takes sub-pieces (STG bytes) lane, lane + L, ... of the whole copy.
template <int STG, int NSTG>
__global__ void k_tma(const uint8_t *src, uint8_t *dst, uint64_t n) {
    extern __shared__ __align__(128) uint8_t sm[];
    const uint32_t W = blockDim.x >> 5, w = threadIdx.x >> 5;
    uint8_t *buf = sm + (size_t)w * NSTG * STG;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)W * NSTG * STG) + w * NSTG;
    if ((threadIdx.x & 31u) != 0) return;
    for (int s = 0; s < NSTG; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    constexpr uint64_t SPP = kPiece / STG;  // sub-pieces per piece
    const uint64_t L = (uint64_t)gridDim.x * W, me = (uint64_t)blockIdx.x * W + w, total = n * SPP;
    if (me >= total) return;
    const uint64_t cnt = (total - me + L - 1) / L;  // my sub-pieces
    auto srcp = [&](uint64_t k) {
        const uint64_t u = me + k * L;
        return src + u * STG;
    };
    auto dstp = [&](uint64_t k) {
        const uint64_t u = me + k * L;
        return dst + dst_piece(u / SPP, n) * kPiece + (u % SPP) * STG;
    };
    for (uint64_t k = 0; k < cnt && k < (uint64_t)NSTG; k++) {
        mbar_expect_tx(&bar[k], STG);
        bulk_load(buf + k * STG, srcp(k), STG, &bar[k]);
    }
    for (uint64_t k = 0; k < cnt; k++) {
        const uint32_t s = (uint32_t)(k % NSTG);
        mbar_wait(&bar[s], (uint32_t)((k / NSTG) & 1u));
        bulk_store(dstp(k), buf + s * STG, STG);
        bulk_commit();
        if (k >= 1 && k - 1 + NSTG < cnt) {  // stage of store k-1 is free once that store has read it
            bulk_wait_read<1>();
            const uint32_t s1 = (uint32_t)((k - 1) % NSTG);
            mbar_expect_tx(&bar[s1], STG);
            bulk_load(buf + s1 * STG, srcp(k - 1 + NSTG), STG, &bar[s1]);
        }
    }
    bulk_wait_all();
}

template <int STG, int NSTG>
static float run_tma(const uint8_t *s, uint8_t *d, uint64_t n, int ctas_per_sm, int warps, int sms, int reps) {
    const size_t smem = (size_t)warps * NSTG * STG + (size_t)warps * NSTG * 8;
    if (smem > 227 * 1024) return -1.f;
    CK(cudaFuncSetAttribute(k_tma<STG, NSTG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    k_tma<STG, NSTG><<<sms * ctas_per_sm, warps * 32, smem>>>(s, d, n);
    CK(cudaGetLastError());
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; r++) k_tma<STG, NSTG><<<sms * ctas_per_sm, warps * 32, smem>>>(s, d, n);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

static bool check(const uint8_t *s, const uint8_t *d, uint64_t n) {
    std::vector<uint8_t> hs(kPiece), hd(kPiece);
    for (uint64_t k : {0ull, 1ull, (unsigned long long)(n / 2), (unsigned long long)(n - 1)}) {
        CK(cudaMemcpy(hs.data(), s + k * kPiece, kPiece, cudaMemcpyDeviceToHost));
        const uint64_t dp = (k * 40503ull) % n;
        CK(cudaMemcpy(hd.data(), d + dp * kPiece, kPiece, cudaMemcpyDeviceToHost));
        if (std::memcmp(hs.data(), hd.data(), kPiece) != 0) return false;
    }
    return true;
}

int main(int argc, char **argv) {
    const uint64_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1024;
    uint64_t n = (mib << 20) / kPiece;
    if (n % 2 == 0) n--;  // the permutation k * 40503 mod n is a bijection when gcd(40503, n) = 1
    while (std::gcd<uint64_t>(40503ull, n) != 1) n -= 2;
    const uint64_t bytes = n * kPiece;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint8_t *s, *d;
    CK(cudaMalloc(&s, bytes));
    CK(cudaMalloc(&d, bytes));
    {
        std::vector<uint32_t> h(bytes / 4);
        uint32_t x = 12345;
        for (auto &v : h) v = (x = x * 1664525u + 1013904223u);
        CK(cudaMemcpy(s, h.data(), bytes, cudaMemcpyHostToDevice));
    }
    const int reps = 10;
    auto report = [&](const char *name, float ms, bool ok) {
        std::printf("{\"kernel\": \"%s\", \"bytes\": %llu, \"us\": %.1f, \"copy_TBps\": %.3f, \"ok\": %s}\n", name,
                    (unsigned long long)bytes, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e12, ok ? "true" : "false");
        std::fflush(stdout);
    };
    // (c) copy engine
    {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(a));
        for (int r = 0; r < reps; r++) CK(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        report("cudaMemcpyAsync D2D (contiguous)", ms / reps, true);
    }
    // (v) vector copy, grids of k x SMs
    for (int g : {2, 4, 8}) {
        CK(cudaMemset(d, 0, bytes));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        k_vec<<<sms * g, 256>>>(s, d, n);
        CK(cudaEventRecord(a));
        for (int r = 0; r < reps; r++) k_vec<<<sms * g, 256>>>(s, d, n);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        char nm[64];
        std::snprintf(nm, sizeof nm, "vec 256thr grid %dxSM", g);
        report(nm, ms / reps, check(s, d, n));
    }
    // (t) TMA variants
#define T(STG, NSTG, CPS, W)                                                          \
    {                                                                                 \
        CK(cudaMemset(d, 0, bytes));                                                  \
        const float ms = run_tma<STG, NSTG>(s, d, n, CPS, W, sms, reps);              \
        char nm[96];                                                                  \
        std::snprintf(nm, sizeof nm, "tma stage %dK x %d, %d warps, %d CTA/SM", STG / 1024, NSTG, W, CPS); \
        if (ms > 0) report(nm, ms, check(s, d, n));                                   \
    }
    T(16384, 4, 1, 3)
    T(16384, 4, 2, 1)
    T(16384, 3, 1, 4)
    T(8192, 6, 1, 4)
    T(8192, 8, 1, 3)
    T(8192, 4, 2, 3)
    T(32768, 3, 1, 2)
    T(32768, 2, 1, 3)
    T(4096, 8, 1, 6)
    T(16384, 6, 1, 2)
    T(8192, 12, 1, 2)
    T(16384, 2, 2, 3)
    return 0;
}
