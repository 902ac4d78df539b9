// Microbenchmark: throughput of many small TMA bulk stores (shared -> global)
// issued by the digit-owner threads of a tile, as a multisplit write-out
// would: per tile, `runs` bulk copies of `bytes` each to scattered
// destinations (run r of tile t goes to region r, slot t). Compared with a
// plain coalesced STG write-out of the same tile.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1907_02900_b200/csrc/hg_common.cuh"
using namespace hg;

__global__ void __launch_bounds__(512) k_bulk(char* out, uint64_t region, int tiles, int runs, int bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x;
    for (int i = tid; i < runs * bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    fence_proxy_async();
    __syncthreads();
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int r = tid; r < runs; r += blockDim.x) {
            char* dst = out + uint64_t(r) * region + uint64_t(t) * bytes;
            tma_store_1d(dst, sm + r * bytes, bytes);
        }
        bulk_commit();
        bulk_wait_read();
        __syncthreads();
    }
    bulk_wait_all();
}

__global__ void __launch_bounds__(512) k_stg(uint2* out, uint64_t region, int tiles, int runs, int bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x;
    const int per = bytes / 8;
    for (int i = tid; i < runs * bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    __syncthreads();
    const uint2* s = reinterpret_cast<const uint2*>(sm);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int j = tid; j < runs * per; j += blockDim.x) {
            const int r = j / per, q = j - r * per;
            out[(uint64_t(r) * region + uint64_t(t) * bytes) / 8 + q] = s[j];
        }
        __syncthreads();
    }
}

int main() {
    const int runs = 256;
    for (int bytes : {64, 128, 256}) {
        const int tile_bytes = runs * bytes;
        const uint64_t total = uint64_t(2) << 30;  // 2 GB written
        const int tiles = int(total / tile_bytes);
        const uint64_t region = uint64_t(tiles) * bytes;
        char* out;
        cudaMalloc(&out, region * runs + 4096);
        cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_bytes);
        cudaFuncSetAttribute(k_stg, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_bytes);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int mode = 0; mode < 2; ++mode) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) k_bulk<<<148 * 2, 512, tile_bytes>>>(out, region, tiles, runs, bytes);
                else k_stg<<<148 * 2, 512, tile_bytes>>>(reinterpret_cast<uint2*>(out), region, tiles, runs, bytes);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s run=%4dB: %.3f ms  %.0f GB/s  (%s)\n", mode ? "STG " : "bulk", bytes, ms,
                   total / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(out);
    }
}
