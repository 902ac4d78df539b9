// microbench.cu -- B200 primitive throughput probes that shape the kernel design
// (shared/global atomics, scattered stores, random gathers, match.any).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench scripts/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void k_smem_atomic(uint32_t* out, int iters, uint32_t mask) {
    extern __shared__ uint32_t sh[];
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = hash32(x + it);
        if (MODE == 0) acc += atomicAdd(sh + (x & mask), 1u);
        else atomicAdd(sh + (x & mask), 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sh[0] + acc;
}

template <int MODE>
__global__ void k_gmem_atomic(uint32_t* arr, uint32_t* out, int iters, uint64_t mask) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = hash32(x + it);
        uint64_t a = (uint64_t(x) * 2654435761ULL) & mask;
        if (MODE == 0) acc += atomicAdd(arr + a, 1u);
        else atomicAdd(arr + a, 1u);
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

// Each thread: 8 independent atomics in flight, then uses results.
__global__ void k_gmem_atomic_ilp(uint32_t* arr, uint32_t* out, int iters, uint64_t mask) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
    for (int it = 0; it < iters; it += 8) {
        uint32_t r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x = hash32(x + it + k);
            r[k] = atomicAdd(arr + ((uint64_t(x) * 2654435761ULL) & mask), 1u);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += r[k];
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

template <typename T>
__global__ void k_scatter_store(T* arr, int iters, uint64_t mask) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        x = hash32(x + it);
        arr[(uint64_t(x) * 2654435761ULL) & mask] = T(x);
    }
}

template <typename T>
__global__ void k_gather(const T* arr, uint32_t* out, int iters, uint64_t mask) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    T acc = T(0);
    for (int it = 0; it < iters; it += 8) {
        T r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x = hash32(x + it + k);
            r[k] = arr[(uint64_t(x) * 2654435761ULL) & mask];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = acc + r[k];
    }
    if (acc == T(12345)) out[0] = 1;
}

__global__ void k_match(uint32_t* out, int iters) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = hash32(x + it);
        acc += __match_any_sync(0xffffffffu, x & 0xffff);
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 1 << 20);
    uint32_t* big;
    const size_t big_bytes = size_t(4) << 30;
    cudaMalloc(&big, big_bytes);
    cudaMemset(big, 0, big_bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, double ops, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("%-48s %9.3f ms  %8.2f Gop/s %s\n", name, ms, ops / ms / 1e6, e ? cudaGetErrorString(e) : "");
    };
    const int iters = 1024;
    for (int bs : {256, 1024}) {
        for (uint32_t entries : {4096u, 16384u, 32768u}) {
            int blocks = sms * (2048 / bs);
            size_t smem = entries * 4;
            if (smem > 48 * 1024) {
                cudaFuncSetAttribute(k_smem_atomic<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                cudaFuncSetAttribute(k_smem_atomic<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            }
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_smem_atomic<0>, bs, smem);
            blocks = sms * per;
            char name[128];
            double ops = double(blocks) * bs * iters;
            snprintf(name, sizeof name, "smem atomicAdd ret bs=%d tbl=%u (%d/SM)", bs, entries, per);
            timeit(name, ops, [&] { k_smem_atomic<0><<<blocks, bs, smem>>>(out, iters, entries - 1); });
            snprintf(name, sizeof name, "smem atomicAdd noret bs=%d tbl=%u", bs, entries);
            timeit(name, ops, [&] { k_smem_atomic<1><<<blocks, bs, smem>>>(out, iters, entries - 1); });
        }
    }
    for (uint64_t entries : {uint64_t(1) << 14, uint64_t(1) << 16, uint64_t(1) << 20, uint64_t(1) << 24, uint64_t(1) << 28}) {
        int blocks = sms * 8;
        double ops = double(blocks) * 256 * iters;
        char name[128];
        snprintf(name, sizeof name, "gmem atomicAdd ret (dep) tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_gmem_atomic<0><<<blocks, 256>>>(big, out, iters, entries - 1); });
        snprintf(name, sizeof name, "gmem atomicAdd ret ILP8 tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_gmem_atomic_ilp<<<blocks, 256>>>(big, out, iters, entries - 1); });
        snprintf(name, sizeof name, "gmem RED tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_gmem_atomic<1><<<blocks, 256>>>(big, out, iters, entries - 1); });
        snprintf(name, sizeof name, "scatter store u32 tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_scatter_store<uint32_t><<<blocks, 256>>>(big, iters, entries - 1); });
        snprintf(name, sizeof name, "scatter store u64 tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_scatter_store<unsigned long long><<<blocks, 256>>>((unsigned long long*)big, iters, entries - 1); });
        snprintf(name, sizeof name, "gather u32 tbl=2^%d", __builtin_ctzll(entries));
        timeit(name, ops, [&] { k_gather<uint32_t><<<blocks, 256>>>(big, out, iters, entries - 1); });
    }
    {
        uint64_t entries = uint64_t(1) << 29;
        int blocks = sms * 8;
        double ops = double(blocks) * 256 * iters;
        timeit("gather u64 tbl=2^29 (4GB)", ops, [&] { k_gather<unsigned long long><<<blocks, 256>>>((unsigned long long*)big, out, iters, entries - 1); });
    }
    {
        int blocks = sms * 8;
        double ops = double(blocks) * 256 * iters;
        timeit("match_any u32", ops, [&] { k_match<<<blocks, 256>>>(out, iters); });
    }
    {
        // copy bandwidth reference
        size_t n = size_t(1) << 30;
        timeit("memcpy D2D 2x1GiB (GB/s = 2*bytes)", double(n) * 2 / 1e3, [&] {
            cudaMemcpyAsync(big, (char*)big + n, n, cudaMemcpyDeviceToDevice);
        });
    }
    return 0;
}
