// synth.cu -- libgcr_synth.so: seeded synthetic inputs (HARNESS; see
// include/gcr_synth.h).  No snapshot arithmetic lives here.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../../include/gcr_synth.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t f32_of(uint32_t b, uint32_t e0, bool sign) {
    return (sign ? (b & 0x80000000u) : 0u) | ((e0 + ((b >> 23) & 3u)) << 23) | (b & 0x7FFFFFu);
}

__device__ __forceinline__ uint64_t word_of(uint64_t r, uint32_t kind, uint32_t cb) {
    switch (kind) {
        case 0: return r;
        case 1: return (uint64_t)f32_of((uint32_t)r, 118, true) | ((uint64_t)f32_of((uint32_t)(r >> 32), 118, true) << 32);
        case 2: return (uint64_t)cb | ((uint64_t)cb << 32);
        case 3: return 0;
        case 4: return (uint64_t)f32_of((uint32_t)r, 113, true) | ((uint64_t)f32_of((uint32_t)(r >> 32), 113, true) << 32);
        case 5: return (uint64_t)f32_of((uint32_t)r, 103, false) | ((uint64_t)f32_of((uint32_t)(r >> 32), 103, false) << 32);
        case 6: {
            uint64_t w = 0;
            for (int k = 0; k < 4; k++) {
                const uint32_t h = (uint32_t)(r >> (16 * k)) & 0xFFFFu;
                const uint32_t v = (h & 0x8000u) | ((118u + ((h >> 7) & 3u)) << 7) | (h & 0x7Fu);
                w |= (uint64_t)v << (16 * k);
            }
            return w;
        }
    }
    return 0;
}

__global__ void k_fill(uint64_t *dst, uint64_t nwords, uint64_t ctr_base, uint32_t kind, uint32_t cb) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = (kind == 2 || kind == 3) ? 0 : splitmix64(ctr_base ^ i);
        dst[i] = word_of(r, kind, cb);
    }
}

__global__ void k_xor(uint32_t *p, uint32_t x) { *p ^= x; }

__global__ void k_xor_batch(const uint64_t *ptrs, const uint32_t *xs, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        *reinterpret_cast<uint32_t *>(ptrs[i]) ^= xs[i];
}

__global__ void k_spin(const volatile uint32_t *flag) {
    while (*flag == 0) {
        __nanosleep(1000);
    }
}

}  // namespace

extern "C" {

int gsy_fill(uint64_t dptr, uint64_t bytes, uint64_t seed, uint32_t key, uint32_t kind, uint32_t cb, void *stream) {
    if (bytes % 8 || kind > 6) return (int)cudaErrorInvalidValue;
    const uint64_t n = bytes / 8;
    if (n == 0) return 0;
    uint64_t grid = (n + 255) / 256;
    if (grid > 148ull * 32) grid = 148ull * 32;
    k_fill<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>((uint64_t *)dptr, n, seed ^ ((uint64_t)key << 40), kind, cb);
    return (int)cudaGetLastError();
}

int gsy_xor_u32(uint64_t dptr, uint32_t x, void *stream) {
    k_xor<<<1, 1, 0, (cudaStream_t)stream>>>((uint32_t *)dptr, x);
    return (int)cudaGetLastError();
}

int gsy_xor_u32_batch(const uint64_t *dptrs, const uint32_t *xs, uint64_t n, void *stream) {
    if (n == 0) return 0;
    uint64_t *dp = nullptr;
    uint32_t *dx = nullptr;
    cudaError_t e = cudaMalloc(&dp, n * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dx, n * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dp, dptrs, n * 8, cudaMemcpyHostToDevice, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dx, xs, n * 4, cudaMemcpyHostToDevice, (cudaStream_t)stream);
    if (e == cudaSuccess) {
        uint64_t grid = (n + 255) / 256;
        if (grid > 148ull * 16) grid = 148ull * 16;
        k_xor_batch<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(dp, dx, n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(dp);
    cudaFree(dx);
    return (int)e;
}

int gsy_flag_alloc(uint64_t *host_ptr, uint64_t *dev_ptr) {
    void *h = nullptr, *d = nullptr;
    cudaError_t e = cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return (int)e;
    *(volatile uint32_t *)h = 0;
    e = cudaHostGetDevicePointer(&d, h, 0);
    if (e != cudaSuccess) return (int)e;
    *host_ptr = (uint64_t)h;
    *dev_ptr = (uint64_t)d;
    return 0;
}

int gsy_flag_set(uint64_t host_ptr, uint32_t value) {
    *(volatile uint32_t *)host_ptr = value;
    return 0;
}

int gsy_flag_free(uint64_t host_ptr) { return (int)cudaFreeHost((void *)host_ptr); }

int gsy_spin_until_flag(uint64_t dev_flag, void *stream) {
    k_spin<<<1, 1, 0, (cudaStream_t)stream>>>((const volatile uint32_t *)dev_flag);
    return (int)cudaGetLastError();
}

}  // extern "C"
