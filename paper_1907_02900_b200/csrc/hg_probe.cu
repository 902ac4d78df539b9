// hg_probe.cu -- probe_standard on sm_100a.
//
// Replaces proj/include/hashgraph/join.hpp:110-136 (probe_standard) and its
// ProbeAccumulator (join.hpp:63-103):
//   K8  k_probe_count  per probe: hash, read offs[v], offs[v+1], compare every
//                      key of the segment (join.hpp:117-129); exact match
//                      count and key comparisons; optional per-probe counts
//   K9  scan           per-probe counts -> u64 pair offsets (deterministic slots)
//   K10 k_probe_write  re-walk probes with count > 0 and write
//                      (build entry index, probe position) pairs at exact
//                      slots, keeping slots < pair_cap (join.hpp:68-75)
// Segments longer than kLongSeg are walked warp-cooperatively (the 32 lanes
// stride one segment) so skewed, heavy vertices do not serialise one lane.
#include <algorithm>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_scan.cuh"

namespace hg {

int num_sms();

constexpr int kProbeBlock = 256;
constexpr uint64_t kLongSeg = 32;

template <bool POW2>
__device__ __forceinline__ uint64_t pvtx(uint64_t key, uint64_t seed, int hk, const Divisor& nv) {
    return hk == kHashIdentity ? vertex_of<kHashIdentity, POW2>(key, seed, nv)
                               : vertex_of<kHashMix64, POW2>(key, seed, nv);
}

// Loads the VEC probes of this lane for warp chunk `base` (VEC*32 probes per
// warp). valid[k] is false past the end.
template <typename K, int VEC>
__device__ __forceinline__ void load_probes(const K* probes, uint64_t m, uint64_t first, K (&pk)[VEC],
                                            bool (&valid)[VEC]) {
    using V = typename std::conditional<sizeof(K) == 4, uint4, ulonglong2>::type;
    if (first + VEC <= m && (reinterpret_cast<uintptr_t>(probes + first) & 15) == 0) {
        const V u = __ldcs(reinterpret_cast<const V*>(probes + first));
        const K* ku = reinterpret_cast<const K*>(&u);
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            pk[k] = ku[k];
            valid[k] = true;
        }
    } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            valid[k] = first + k < m;
            pk[k] = valid[k] ? probes[first + k] : K(0);
        }
    }
}

template <typename K, typename OffT, bool POW2, bool WRITE_COUNTS>
__global__ void __launch_bounds__(kProbeBlock)
k_probe_count(const K* __restrict__ probes, uint64_t m, uint64_t seed, int hk, Divisor nv,
              const OffT* __restrict__ offs, const K* __restrict__ tkeys,
              uint32_t* __restrict__ counts, uint64_t* __restrict__ totals) {
    constexpr int VEC = 16 / sizeof(K);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    uint64_t matches = 0, compared = 0;
    for (uint64_t base = warp * 32 * VEC; base < m; base += nwarps * 32 * VEC) {
        const uint64_t first = base + uint64_t(lane) * VEC;
        K pk[VEC];
        bool valid[VEC];
        load_probes<K, VEC>(probes, m, first, pk, valid);
        uint64_t b[VEC], e[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            b[k] = e[k] = 0;
            if (valid[k]) {
                const uint64_t v = pvtx<POW2>(pk[k], seed, hk, nv);
                b[k] = offs[v];
                e[k] = offs[v + 1];
            }
        }
        uint32_t c[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            c[k] = 0;
            const uint64_t len = e[k] - b[k];
            compared += len;
            if (len <= kLongSeg)
                for (uint64_t t = b[k]; t < e[k]; ++t) c[k] += tkeys[t] == pk[k];
            uint32_t longm = __ballot_sync(0xffffffffu, len > kLongSeg);
            while (longm) {
                const int src = __ffs(longm) - 1;
                longm &= longm - 1;
                const uint64_t kb = __shfl_sync(0xffffffffu, b[k], src);
                const uint64_t ke = __shfl_sync(0xffffffffu, e[k], src);
                const K kk = __shfl_sync(0xffffffffu, pk[k], src);
                uint32_t cc = 0;
                for (uint64_t t = kb + lane; t < ke; t += 32) cc += tkeys[t] == kk;
                cc = warp_sum(cc);
                if (int(lane) == src) c[k] = cc;
            }
            matches += c[k];
        }
        if constexpr (WRITE_COUNTS) {
            bool done = false;
            if constexpr (VEC == 4) {
                if (valid[3] && (reinterpret_cast<uintptr_t>(counts + first) & 15) == 0) {
                    *reinterpret_cast<uint4*>(counts + first) = make_uint4(c[0], c[1], c[2], c[3]);
                    done = true;
                }
            }
            if (!done) {
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (valid[k]) counts[first + k] = c[k];
            }
        }
    }
    // block reduction -> one pair of u64 atomics per CTA
    __shared__ unsigned long long s_m[kProbeBlock / 32], s_c[kProbeBlock / 32];
    matches = warp_sum(matches);
    compared = warp_sum(compared);
    if (lane == 0) {
        s_m[threadIdx.x >> 5] = matches;
        s_c[threadIdx.x >> 5] = compared;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long a = threadIdx.x < kProbeBlock / 32 ? s_m[threadIdx.x] : 0;
        unsigned long long d = threadIdx.x < kProbeBlock / 32 ? s_c[threadIdx.x] : 0;
        a = warp_sum(a);
        d = warp_sum(d);
        if (threadIdx.x == 0) {
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(totals), a);
            if (d) atomicAdd(reinterpret_cast<unsigned long long*>(totals + 1), d);
        }
    }
}

template <typename PT>
__device__ __forceinline__ void store_pair(void* pairs, uint64_t slot, uint64_t left, uint64_t right) {
    if constexpr (sizeof(PT) == 4) {
        reinterpret_cast<uint2*>(pairs)[slot] = make_uint2(uint32_t(left), uint32_t(right));
    } else {
        reinterpret_cast<ulonglong2*>(pairs)[slot] = make_ulonglong2(left, right);
    }
}

template <typename K, typename VT, typename OffT, typename PT, bool POW2>
__global__ void __launch_bounds__(kProbeBlock)
k_probe_write(const K* __restrict__ probes, uint64_t m, uint64_t seed, int hk, Divisor nv,
              const OffT* __restrict__ offs, const K* __restrict__ tkeys,
              const VT* __restrict__ tvals, const uint32_t* __restrict__ counts,
              const uint64_t* __restrict__ pair_off, void* __restrict__ pairs, uint64_t cap) {
    constexpr int VEC = 16 / sizeof(K);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t base = warp * 32 * VEC; base < m; base += nwarps * 32 * VEC) {
        const uint64_t first = base + uint64_t(lane) * VEC;
        K pk[VEC];
        bool valid[VEC];
        load_probes<K, VEC>(probes, m, first, pk, valid);
        uint64_t b[VEC], e[VEC], slot[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            b[k] = e[k] = slot[k] = 0;
            if (valid[k] && counts[first + k] != 0) {
                slot[k] = pair_off[first + k];
                if (slot[k] < cap) {
                    const uint64_t v = pvtx<POW2>(pk[k], seed, hk, nv);
                    b[k] = offs[v];
                    e[k] = offs[v + 1];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const uint64_t len = e[k] - b[k];
            if (len <= kLongSeg) {
                uint64_t sl = slot[k];
                for (uint64_t t = b[k]; t < e[k] && sl < cap; ++t) {
                    if (tkeys[t] == pk[k]) {
                        store_pair<PT>(pairs, sl, uint64_t(tvals[t]), first + k);
                        ++sl;
                    }
                }
            }
            uint32_t longm = __ballot_sync(0xffffffffu, len > kLongSeg);
            while (longm) {
                const int src = __ffs(longm) - 1;
                longm &= longm - 1;
                const uint64_t kb = __shfl_sync(0xffffffffu, b[k], src);
                const uint64_t ke = __shfl_sync(0xffffffffu, e[k], src);
                const K kk = __shfl_sync(0xffffffffu, pk[k], src);
                uint64_t sl = __shfl_sync(0xffffffffu, slot[k], src);
                const uint64_t pj = __shfl_sync(0xffffffffu, first + k, src);
                for (uint64_t t0 = kb; t0 < ke && sl < cap; t0 += 32) {
                    const uint64_t t = t0 + lane;
                    const bool hit = t < ke && tkeys[t] == kk;
                    const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                    const uint64_t my = sl + __popc(hm & lanemask_lt());
                    if (hit && my < cap) store_pair<PT>(pairs, my, uint64_t(tvals[t]), pj);
                    sl += __popc(hm);
                }
            }
        }
    }
}

template <typename K, typename VT, typename OffT, bool POW2>
static cudaError_t probe_impl(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    const Divisor nv = make_divisor(t.nv);
    const OffT* offs = static_cast<const OffT*>(t.offs);
    const K* probes = static_cast<const K*>(a.probes);
    const K* tkeys = static_cast<const K*>(t.keys);
    if (a.m == 0) {
        if (a.pairs && a.pair_offsets) return cudaMemsetAsync(a.pair_offsets, 0, 8, s);
        return cudaSuccess;
    }
    const int sms = num_sms();
    const bool need_counts = a.counts != nullptr;
    int per_sm = 0;
    cudaError_t e;
    if (need_counts) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_probe_count<K, OffT, POW2, true>,
                                                      kProbeBlock, 0);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_probe_count<K, OffT, POW2, false>,
                                                      kProbeBlock, 0);
    }
    constexpr int VEC = 16 / sizeof(K);
    const uint64_t warps_needed = (a.m + 32 * VEC - 1) / (32 * VEC);
    const uint64_t blocks_needed = (warps_needed * 32 + kProbeBlock - 1) / kProbeBlock;
    const unsigned grid = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>(blocks_needed, uint64_t(std::max(per_sm, 1)) * sms)));
    if (need_counts) {
        HG_LAUNCH("k8_probe_count", s, k_probe_count<K, OffT, POW2, true><<<grid, kProbeBlock, 0, s>>>(
            probes, a.m, t.seed, t.hash_kind, nv, offs, tkeys, a.counts, a.totals));
    } else {
        HG_LAUNCH("k8_probe_count", s, k_probe_count<K, OffT, POW2, false><<<grid, kProbeBlock, 0, s>>>(
            probes, a.m, t.seed, t.hash_kind, nv, offs, tkeys, nullptr, a.totals));
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (!a.pairs) return cudaSuccess;
    if (!need_counts || !a.pair_offsets) return cudaErrorInvalidValue;
    void* scratch = nullptr;
    if ((e = cudaMallocAsync(&scratch, scan_scratch_bytes(a.m), s)) != cudaSuccess) return e;
    e = launch_scan<uint32_t, uint64_t>(a.counts, a.pair_offsets, a.m, scratch,
                                        a.pair_offsets + a.m, s, "k9_pair_scan");
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return e;
    if (a.cap == 0) return cudaSuccess;
    if (a.pair_bytes == 4) {
        HG_LAUNCH("k10_probe_write", s, k_probe_write<K, VT, OffT, uint32_t, POW2><<<grid, kProbeBlock, 0, s>>>(
            probes, a.m, t.seed, t.hash_kind, nv, offs, tkeys, static_cast<const VT*>(t.vals),
            a.counts, a.pair_offsets, a.pairs, a.cap));
    } else {
        HG_LAUNCH("k10_probe_write", s, k_probe_write<K, VT, OffT, uint64_t, POW2><<<grid, kProbeBlock, 0, s>>>(
            probes, a.m, t.seed, t.hash_kind, nv, offs, tkeys, static_cast<const VT*>(t.vals),
            a.counts, a.pair_offsets, a.pairs, a.cap));
    }
    return cudaGetLastError();
}

template <typename K, typename VT, typename OffT>
static cudaError_t probe_pow(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return (t.nv & (t.nv - 1)) == 0 ? probe_impl<K, VT, OffT, true>(t, a, s)
                                    : probe_impl<K, VT, OffT, false>(t, a, s);
}
template <typename K, typename VT>
static cudaError_t probe_off(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.off_bytes == 4 ? probe_pow<K, VT, uint32_t>(t, a, s) : probe_pow<K, VT, uint64_t>(t, a, s);
}
template <typename K>
static cudaError_t probe_val(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.val_bytes == 4 ? probe_off<K, uint32_t>(t, a, s) : probe_off<K, uint64_t>(t, a, s);
}

cudaError_t probe_table(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.key_bytes == 4 ? probe_val<uint32_t>(t, a, s) : probe_val<uint64_t>(t, a, s);
}

}  // namespace hg
