// hg_scan.cuh -- single-pass decoupled look-back exclusive scan (sm_100a).
//
// Replaces the reference's chunked two-pass scan
// (proj/include/hashgraph/parallel.hpp:141-192 exclusive_scan_impl, called
// from core.hpp:135 and :205). Unsigned addition is exact, so the result is
// bit-identical to the sequential fold for any tiling.
//
// One pass over the data: each CTA scans a 4096-element tile in registers,
// publishes its aggregate in a 64-bit status word (2 flag bits + 62 value
// bits, so the payload travels with the flag in one single-copy-atomic
// store), and warp 0 looks back over up to 32 predecessors per step. Tile ids
// come from an atomic ticket so every predecessor tile is already resident
// (no deadlock). HBM traffic = read n + write n (+ 8 B per tile of status).
#pragma once

#include "hg_common.cuh"
#include "hg_internal.h"

namespace hg {

constexpr uint64_t kScanFlagAgg = uint64_t(1) << 62;
constexpr uint64_t kScanFlagIncl = uint64_t(2) << 62;
constexpr uint64_t kScanValMask = (uint64_t(1) << 62) - 1;
constexpr int kScanBlock = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanBlock * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T x) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, d);
        if (int(lane_id()) >= d) x += y;
    }
    return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
    if constexpr (sizeof(T) == 4) {
        return T(__reduce_add_sync(0xffffffffu, uint32_t(x)));  // one REDUX (sm_80+)
    } else {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        return x;
    }
}

// Loads kScanItems consecutive elements of `in` starting at element `base`
// (blocked arrangement); vectorised when the tile is full and aligned.
template <typename TI, typename TA>
__device__ __forceinline__ void scan_load(const TI* in, uint64_t n, uint64_t base, TA (&x)[kScanItems]) {
    const bool full = base + kScanItems <= n;
    if constexpr (sizeof(TI) == 4) {
        if (full && (reinterpret_cast<uintptr_t>(in + base) & 15) == 0) {
            const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
            for (int q = 0; q < kScanItems / 4; ++q) {
                const uint4 u = __ldcs(p + q);
                x[4 * q + 0] = u.x;
                x[4 * q + 1] = u.y;
                x[4 * q + 2] = u.z;
                x[4 * q + 3] = u.w;
            }
            return;
        }
    } else {
        if (full && (reinterpret_cast<uintptr_t>(in + base) & 15) == 0) {
            const ulonglong2* p = reinterpret_cast<const ulonglong2*>(in + base);
#pragma unroll
            for (int q = 0; q < kScanItems / 2; ++q) {
                const ulonglong2 u = __ldcs(p + q);
                x[2 * q + 0] = TA(u.x);
                x[2 * q + 1] = TA(u.y);
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) x[k] = base + k < n ? TA(in[base + k]) : TA(0);
}

template <typename TO>
__device__ __forceinline__ void scan_store(TO* out, uint64_t n, uint64_t base, const TO (&x)[kScanItems]) {
    const bool full = base + kScanItems <= n;
    if constexpr (sizeof(TO) == 4) {
        if (full && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
            uint4* p = reinterpret_cast<uint4*>(out + base);
#pragma unroll
            for (int q = 0; q < kScanItems / 4; ++q)
                p[q] = make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
            return;
        }
    } else {
        if (full && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
            ulonglong2* p = reinterpret_cast<ulonglong2*>(out + base);
#pragma unroll
            for (int q = 0; q < kScanItems / 2; ++q)
                p[q] = make_ulonglong2((unsigned long long)x[2 * q], (unsigned long long)x[2 * q + 1]);
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) out[base + k] = x[k];
}

// out[i] = sum(in[0..i)) for i < n; *total (nullable) = sum(in[0..n)).
// in == out (in place) is allowed. status[num_tiles] and *ticket must be
// zero on entry.
template <typename TI, typename TO>
__global__ void __launch_bounds__(kScanBlock)
k_scan_lookback(const TI* in, TO* out, uint64_t n, uint64_t* status, uint32_t* ticket, TO* total,
                const uint32_t* guard) {
    if (guard && !*guard) return;  // device-side skip (the exact fallback of partition_slack)
    __shared__ uint32_t s_tile;
    __shared__ TO s_warp[kScanBlock / 32];
    __shared__ TO s_prefix;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kScanTile + uint64_t(tid) * kScanItems;

    TO x[kScanItems];
    scan_load<TI, TO>(in, n, base, x);
    TO run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const TO v = x[k];
        x[k] = run;  // thread-local exclusive
        run += v;
    }
    const TO winc = warp_inclusive_sum(run);
    if (lane == 31) s_warp[warp] = winc;
    __syncthreads();
    if (warp == 0) {
        TO wt = lane < kScanBlock / 32 ? s_warp[lane] : TO(0);
        const TO wi = warp_inclusive_sum(wt);
        if (lane < kScanBlock / 32) s_warp[lane] = wi - wt;  // exclusive warp offsets
        const TO agg = __shfl_sync(0xffffffffu, wi, 31);
        // Look-back.
        TO prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed_u64(status, kScanFlagIncl | uint64_t(agg));
        } else {
            if (lane == 0) st_relaxed_u64(status + tile, kScanFlagAgg | uint64_t(agg));
            int64_t idx = int64_t(tile) - 1;
            while (true) {
                const int64_t j = idx - int64_t(lane);
                uint64_t s = kScanFlagIncl;
                if (j >= 0) {
                    do {
                        s = ld_relaxed_u64(status + j);
                    } while ((s >> 62) == 0);
                }
                const uint32_t incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                const uint32_t stop = incl ? uint32_t(__ffs(incl) - 1) : 32u;
                const TO val = lane <= stop ? TO(s & kScanValMask) : TO(0);
                prefix += warp_sum(val);
                if (incl) break;
                idx -= 32;
            }
            if (lane == 0) st_relaxed_u64(status + tile, kScanFlagIncl | uint64_t(prefix + agg));
        }
        if (lane == 0) {
            s_prefix = prefix;
            if (total && (tile + 1) * kScanTile >= n) *total = prefix + agg;
        }
    }
    __syncthreads();
    const TO off = s_prefix + s_warp[warp] + (winc - run);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) x[k] += off;
    scan_store<TO>(out, n, base, x);
}

inline uint64_t scan_num_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// Scratch bytes for one scan of n elements: status words + ticket.
inline size_t scan_scratch_bytes(uint64_t n) { return (scan_num_tiles(n) + 1) * sizeof(uint64_t); }

template <typename TI, typename TO>
cudaError_t launch_scan(const TI* in, TO* out, uint64_t n, void* scratch, TO* total, cudaStream_t s,
                        const char* name = "scan", const uint32_t* guard = nullptr) {
    if (n == 0) {
        if (total) return cudaMemsetAsync(total, 0, sizeof(TO), s);
        return cudaSuccess;
    }
    const uint64_t tiles = scan_num_tiles(n);
    uint64_t* status = static_cast<uint64_t*>(scratch);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(status + tiles);
    cudaError_t e = cudaMemsetAsync(scratch, 0, scan_scratch_bytes(n), s);
    if (e != cudaSuccess) return e;
    HG_LAUNCH(name, s, k_scan_lookback<TI, TO><<<unsigned(tiles), kScanBlock, 0, s>>>(in, out, n, status, ticket, total,
                                                                               guard));
    return cudaGetLastError();
}

}  // namespace hg
