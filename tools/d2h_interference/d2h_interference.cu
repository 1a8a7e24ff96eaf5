// d2h_interference.cu -- does SM load slow a D2H DMA?  A 256 MiB
// device -> pinned-host cudaMemcpyAsync timed alone and while a kernel streams
// HBM (read-only, or read + write) on K of the SMs, K in {8, 32, 148}.  The f4
// checkpoint encodes the next sub-chunk (KA/KC, ~2 TB/s of HBM traffic) while
// the previous one drains; this says whether that costs link throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/d2h_interference/d2h tools/d2h_interference/d2h_interference.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                   \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// stream src (and write dst if non-null) repeatedly for `ns` nanoseconds of
// the global timer (no host polling: a mapped-memory flag polled by every
// thread put ~10 GB/s of PCIe read requests on the link and wrecked the D2H)
__global__ void k_load(const uint4 *src, uint4 *dst, uint64_t n16, uint64_t ns, unsigned long long *sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t_end = gtimer() + ns;
    while (gtimer() < t_end) {
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldcs(src + i);
            if (dst) __stcs(dst + i, v);
            acc.x ^= v.x;
            acc.y ^= v.y;
        }
    }
    if (acc.x == 0x12345678u && acc.y == 0x9abcdef0u) atomicAdd(sink, 1ull);
}

int main() {
    const uint64_t D = 256ull << 20, L = 2048ull << 20;
    uint8_t *dsrc, *lsrc, *ldst, *host;
    CK(cudaMalloc(&dsrc, D));
    CK(cudaMalloc(&lsrc, L));
    CK(cudaMalloc(&ldst, L));
    CK(cudaMemset(dsrc, 1, D));
    CK(cudaMemset(lsrc, 2, L));
    CK(cudaHostAlloc(&host, D, cudaHostAllocDefault));
    unsigned long long *sink;
    CK(cudaMalloc(&sink, 8));
    cudaStream_t cs, ks;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto d2h = [&]() {
        float best = 1e9, sum = 0;
        for (int r = 0; r < 6; r++) {
            CK(cudaEventRecord(a, cs));
            CK(cudaMemcpyAsync(host, dsrc, D, cudaMemcpyDeviceToHost, cs));
            CK(cudaEventRecord(b, cs));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r) {
                sum += ms;
                best = ms < best ? ms : best;
            }
        }
        return std::make_pair(D / (sum / 5 * 1e-3) / 1e9, D / (best * 1e-3) / 1e9);
    };
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    auto alone = d2h();
    std::printf("{\"load\": \"none\", \"d2h_GBps_mean\": %.2f, \"best\": %.2f}\n", alone.first, alone.second);
    for (int rw = 0; rw < 2; rw++)
        for (int k : {8, 32, sms}) {
            k_load<<<k * 2, 1024, 0, ks>>>(reinterpret_cast<const uint4 *>(lsrc), rw ? reinterpret_cast<uint4 *>(ldst) : nullptr,
                                           L / 16, 200000000ull, sink);  // 200 ms: longer than the 6 D2Hs
            CK(cudaGetLastError());
            auto r = d2h();
            CK(cudaStreamSynchronize(ks));
            std::printf("{\"load\": \"%s on %d SMs\", \"d2h_GBps_mean\": %.2f, \"best\": %.2f}\n", rw ? "read+write" : "read", k,
                        r.first, r.second);
            std::fflush(stdout);
        }
    auto again = d2h();
    std::printf("{\"load\": \"none (after)\", \"d2h_GBps_mean\": %.2f, \"best\": %.2f}\n", again.first, again.second);
    return 0;
}
