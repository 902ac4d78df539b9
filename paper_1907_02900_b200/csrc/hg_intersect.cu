// hg_intersect.cu -- probe_new_prepared on sm_100a.
//
// Replaces proj/include/hashgraph/join.hpp:143-166 probe_new_prepared and
// its per-vertex nested loop intersect_adjacency (join.hpp:41-57). Two tables
// built over one vertex range hold, at vertex v, exactly the keys hashing to
// v, so every match lives in a segment pair (A_v, B_v). No hashing is needed:
// both CSRs are walked in vertex order, i.e. the kernel is a streaming merge
// of offsA, offsB, keysA, keysB (HBM-bound, every byte read once).
//
//   K12 k_intersect   persistent CTAs take vertex tiles (T = 2048 vertices)
//                     from an atomic ticket; thread 0 stages the tile's two
//                     offset slices and two key slices into shared memory
//                     with TMA bulk copies (one mbarrier); each thread owns
//                     T/256 consecutive vertices and compares every (a, b)
//                     pair of a short segment pair serially; segment pairs
//                     with |A_v|*|B_v| > kShortWork are flattened and strided
//                     over the warp (skewed keys do not serialise one lane).
//   pairs mode        the tile's match count is published with a decoupled
//                     look-back (status words as in hg_scan.cuh), so the
//                     pairs are written in the same pass at deterministic
//                     slots: vertex order, then A position, then B position
//                     -- exactly the sequential emission order of the
//                     reference (join.hpp:49-55), and a pair_cap keeps the
//                     first cap of them (join.hpp:71-74 keeps an arbitrary
//                     subset; ours is the sequential one).
// key_comparisons = sum_v |A_v|*|B_v| (join.hpp:52, test_join.cpp:189-205).
#include <algorithm>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_scan.cuh"

namespace hg {

constexpr int kIsBlock = 256;
constexpr uint32_t kIsTileShift = 11;  // 2048 vertices per tile
constexpr uint32_t kIsTile = 1u << kIsTileShift;
constexpr uint32_t kIsVpt = kIsTile / kIsBlock;  // vertices per thread
constexpr uint64_t kShortWork = 64;

struct IsArgs {
    const void* offa;
    const void* offb;
    const void* ka;
    const void* kb;
    const void* va;
    const void* vb;
    int off8a, off8b, val8a, val8b;
    uint64_t nv;
    uint64_t ntiles;
    uint32_t kcapa, kcapb;  // staged key-slice capacities (elements)
    uint64_t* status;       // pairs mode: look-back status word per tile
    void* pairs;
    int pair8;
    uint64_t cap;
    uint64_t* totals;  // [0] match_count, [1] key_comparisons
    uint32_t* ticket;
};

__device__ __forceinline__ uint64_t ld_off(const unsigned char* base, int off8, uint32_t i) {
    return off8 ? reinterpret_cast<const uint64_t*>(base)[i] : reinterpret_cast<const uint32_t*>(base)[i];
}
__device__ __forceinline__ uint64_t ld_goff(const void* p, int off8, uint64_t i) {
    return off8 ? static_cast<const uint64_t*>(p)[i] : static_cast<const uint32_t*>(p)[i];
}
__device__ __forceinline__ uint64_t ld_val(const void* p, int val8, uint64_t i) {
    return val8 ? static_cast<const uint64_t*>(p)[i] : static_cast<const uint32_t*>(p)[i];
}
__device__ __forceinline__ void st_pair(void* pairs, int pair8, uint64_t slot, uint64_t l, uint64_t r) {
    if (pair8) reinterpret_cast<ulonglong2*>(pairs)[slot] = make_ulonglong2(l, r);
    else reinterpret_cast<uint2*>(pairs)[slot] = make_uint2(uint32_t(l), uint32_t(r));
}

__host__ __device__ inline size_t is_span_bytes(size_t bytes) { return (bytes + 32 + 15) & ~size_t(15); }

template <typename K>
__host__ __device__ inline size_t is_smem_bytes(int off8a, int off8b, uint32_t kcapa, uint32_t kcapb) {
    return is_span_bytes(size_t(kIsTile + 1) * (off8a ? 8 : 4)) +
           is_span_bytes(size_t(kIsTile + 1) * (off8b ? 8 : 4)) +
           is_span_bytes(size_t(kcapa) * sizeof(K)) + is_span_bytes(size_t(kcapb) * sizeof(K));
}

// Block-wide exclusive sum of one u64 per thread; returns the thread's
// exclusive prefix and the block total in *total.
__device__ __forceinline__ uint64_t block_exclusive_u64(uint64_t x, uint64_t* s_warp, uint64_t* total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t inc = warp_inclusive_sum(x);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint64_t w = lane < kIsBlock / 32 ? s_warp[lane] : 0;
        const uint64_t wi = warp_inclusive_sum(w);
        if (lane < kIsBlock / 32) s_warp[lane] = wi - w;
        if (lane == 31) s_warp[kIsBlock / 32] = wi;
    }
    __syncthreads();
    const uint64_t r = s_warp[warp] + inc - x;
    *total = s_warp[kIsBlock / 32];
    return r;
}

template <typename K, bool PAIRS>
__global__ void __launch_bounds__(kIsBlock)
k_intersect(IsArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t s_bar;
    __shared__ uint64_t s_tile, s_ta, s_tb, s_na, s_nb, s_base;
    __shared__ uint32_t s_oa, s_ob, s_oka, s_okb, s_sta, s_stb;
    __shared__ uint64_t s_warp[kIsBlock / 32 + 1];
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const size_t offa_bytes = is_span_bytes(size_t(kIsTile + 1) * (a.off8a ? 8 : 4));
    const size_t offb_bytes = is_span_bytes(size_t(kIsTile + 1) * (a.off8b ? 8 : 4));
    unsigned char* const b_oa = smem;
    unsigned char* const b_ob = b_oa + offa_bytes;
    unsigned char* const b_ka = b_ob + offb_bytes;
    unsigned char* const b_kb = b_ka + is_span_bytes(size_t(a.kcapa) * sizeof(K));
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
    }
    uint32_t phase = 0;
    uint64_t matches = 0, compared = 0;
    while (true) {
        if (tid == 0) {
            const uint64_t p = atomicAdd(a.ticket, 1u);
            s_tile = p;
            if (p < a.ntiles) {
                const uint64_t vb = p << kIsTileShift;
                const uint32_t pv = uint32_t(a.nv - vb < kIsTile ? a.nv - vb : uint64_t(kIsTile));
                const uint64_t ta = ld_goff(a.offa, a.off8a, vb), tae = ld_goff(a.offa, a.off8a, vb + pv);
                const uint64_t tb = ld_goff(a.offb, a.off8b, vb), tbe = ld_goff(a.offb, a.off8b, vb + pv);
                s_ta = ta; s_tb = tb; s_na = tae - ta; s_nb = tbe - tb;
                const uint32_t sta = tae - ta <= a.kcapa, stb = tbe - tb <= a.kcapb;
                s_sta = sta; s_stb = stb;
                fence_proxy_async();
                auto span = [](uintptr_t ad, size_t bytes, uint32_t& lo_off) -> uint32_t {
                    const uintptr_t lo = ad & ~uintptr_t(15), hi = (ad + bytes + 15) & ~uintptr_t(15);
                    lo_off = uint32_t(ad - lo);
                    return uint32_t(hi - lo);
                };
                const int oba = a.off8a ? 8 : 4, obb = a.off8b ? 8 : 4;
                const uintptr_t aoa = reinterpret_cast<uintptr_t>(a.offa) + vb * oba;
                const uintptr_t aob = reinterpret_cast<uintptr_t>(a.offb) + vb * obb;
                const uintptr_t aka = reinterpret_cast<uintptr_t>(static_cast<const K*>(a.ka) + ta);
                const uintptr_t akb = reinterpret_cast<uintptr_t>(static_cast<const K*>(a.kb) + tb);
                uint32_t oa, ob, oka = 0, okb = 0;
                const uint32_t la = span(aoa, size_t(pv + 1) * oba, oa);
                const uint32_t lb = span(aob, size_t(pv + 1) * obb, ob);
                const uint32_t lka = (sta && tae > ta) ? span(aka, size_t(tae - ta) * sizeof(K), oka) : 0;
                const uint32_t lkb = (stb && tbe > tb) ? span(akb, size_t(tbe - tb) * sizeof(K), okb) : 0;
                s_oa = oa; s_ob = ob; s_oka = oka; s_okb = okb;
                mbar_arrive_expect_tx(&s_bar, la + lb + lka + lkb);
                tma_load_1d(b_oa, reinterpret_cast<const void*>(aoa - oa), la, &s_bar);
                tma_load_1d(b_ob, reinterpret_cast<const void*>(aob - ob), lb, &s_bar);
                if (lka) tma_load_1d(b_ka, reinterpret_cast<const void*>(aka - oka), lka, &s_bar);
                if (lkb) tma_load_1d(b_kb, reinterpret_cast<const void*>(akb - okb), lkb, &s_bar);
            }
        }
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= a.ntiles) break;
        const uint64_t vb = tile << kIsTileShift;
        const uint32_t pv = uint32_t(a.nv - vb < kIsTile ? a.nv - vb : uint64_t(kIsTile));
        const uint64_t ta = s_ta, tb = s_tb;
        const unsigned char* soa = b_oa + s_oa;
        const unsigned char* sob = b_ob + s_ob;
        const K* kpa = s_sta ? reinterpret_cast<const K*>(b_ka + s_oka) : static_cast<const K*>(a.ka) + ta;
        const K* kpb = s_stb ? reinterpret_cast<const K*>(b_kb + s_okb) : static_cast<const K*>(a.kb) + tb;
        mbar_wait(&s_bar, phase);
        phase ^= 1;

        // this thread's vertices [v0, v1) (tile-local)
        const uint32_t v0 = min(tid * kIsVpt, pv), v1 = min(v0 + kIsVpt, pv);
        uint64_t ab[kIsVpt + 1], bb[kIsVpt + 1];
#pragma unroll
        for (uint32_t j = 0; j <= kIsVpt; ++j) {
            const uint32_t v = min(v0 + j, v1);
            ab[j] = ld_off(soa, a.off8a, v) - ta;
            bb[j] = ld_off(sob, a.off8b, v) - tb;
        }
        uint32_t longm = 0;
        uint64_t cnt[PAIRS ? kIsVpt : 1];
#pragma unroll
        for (uint32_t j = 0; j < kIsVpt; ++j) {
            const uint64_t la = ab[j + 1] - ab[j], lb = bb[j + 1] - bb[j];
            const uint64_t work = la * lb;
            compared += work;
            uint64_t c = 0;
            if (work <= kShortWork) {
                for (uint64_t i = ab[j]; i < ab[j + 1]; ++i) {
                    const K x = kpa[i];
                    for (uint64_t q = bb[j]; q < bb[j + 1]; ++q) c += kpb[q] == x;
                }
            } else {
                longm |= 1u << j;
            }
            if constexpr (PAIRS) cnt[j] = c;
            else matches += c;
        }
        // long segment pairs: flattened p = i*lb + q, strided over the warp
#pragma unroll
        for (uint32_t j = 0; j < kIsVpt; ++j) {
            uint32_t wm = __ballot_sync(0xffffffffu, (longm >> j) & 1u);
            while (wm) {
                const int src = __ffs(wm) - 1;
                wm &= wm - 1;
                const uint64_t a0 = __shfl_sync(0xffffffffu, ab[j], src);
                const uint64_t la = __shfl_sync(0xffffffffu, ab[j + 1], src) - a0;
                const uint64_t b0 = __shfl_sync(0xffffffffu, bb[j], src);
                const uint64_t lb = __shfl_sync(0xffffffffu, bb[j + 1], src) - b0;
                const uint64_t work = la * lb;
                uint64_t c = 0;
                for (uint64_t p = lane; p < work; p += 32) {
                    const uint64_t i = p / lb, q = p - i * lb;
                    c += kpa[a0 + i] == kpb[b0 + q];
                }
                if constexpr (PAIRS) {
                    c = warp_sum(c);
                    if (int(lane) == src) cnt[j] = c;
                } else {
                    matches += c;
                }
            }
        }
        if constexpr (PAIRS) {
            uint64_t mine = 0;
#pragma unroll
            for (uint32_t j = 0; j < kIsVpt; ++j) mine += cnt[j];
            matches += mine;
            uint64_t tile_total;
            const uint64_t excl = block_exclusive_u64(mine, s_warp, &tile_total);
            // decoupled look-back over tiles (ticket order = tile order)
            if (tid < 32) {
                uint64_t prefix = 0;
                if (tile == 0) {
                    if (lane == 0) st_relaxed_u64(a.status, kScanFlagIncl | tile_total);
                } else {
                    if (lane == 0) st_relaxed_u64(a.status + tile, kScanFlagAgg | tile_total);
                    int64_t idx = int64_t(tile) - 1;
                    while (true) {
                        const int64_t jj = idx - int64_t(lane);
                        uint64_t s = kScanFlagIncl;
                        if (jj >= 0) {
                            do {
                                s = ld_relaxed_u64(a.status + jj);
                            } while ((s >> 62) == 0);
                        }
                        const uint32_t incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                        const uint32_t stop = incl ? uint32_t(__ffs(incl) - 1) : 32u;
                        prefix += warp_sum(lane <= stop ? (s & kScanValMask) : uint64_t(0));
                        if (incl) break;
                        idx -= 32;
                    }
                    if (lane == 0) st_relaxed_u64(a.status + tile, kScanFlagIncl | (prefix + tile_total));
                }
                if (lane == 0) s_base = prefix;
            }
            __syncthreads();
            const uint64_t tbase = s_base;
            if (tbase < a.cap) {
                uint64_t slot = tbase + excl;
#pragma unroll
                for (uint32_t j = 0; j < kIsVpt; ++j) {
                    if (!((longm >> j) & 1u) && cnt[j]) {
                        uint64_t sl = slot;
                        for (uint64_t i = ab[j]; i < ab[j + 1] && sl < a.cap; ++i) {
                            const K x = kpa[i];
                            for (uint64_t q = bb[j]; q < bb[j + 1]; ++q) {
                                if (kpb[q] == x && sl < a.cap) {
                                    st_pair(a.pairs, a.pair8, sl, ld_val(a.va, a.val8a, ta + i),
                                            ld_val(a.vb, a.val8b, tb + q));
                                    ++sl;
                                }
                            }
                        }
                    }
                    uint32_t wm = __ballot_sync(0xffffffffu, ((longm >> j) & 1u) && cnt[j] && slot < a.cap);
                    while (wm) {
                        const int src = __ffs(wm) - 1;
                        wm &= wm - 1;
                        const uint64_t a0 = __shfl_sync(0xffffffffu, ab[j], src);
                        const uint64_t la = __shfl_sync(0xffffffffu, ab[j + 1], src) - a0;
                        const uint64_t b0 = __shfl_sync(0xffffffffu, bb[j], src);
                        const uint64_t lb = __shfl_sync(0xffffffffu, bb[j + 1], src) - b0;
                        uint64_t ws = __shfl_sync(0xffffffffu, slot, src);
                        const uint64_t work = la * lb;
                        for (uint64_t p0 = 0; p0 < work && ws < a.cap; p0 += 32) {
                            const uint64_t p = p0 + lane;
                            uint64_t i = 0, q = 0;
                            bool hit = false;
                            if (p < work) {
                                i = p / lb;
                                q = p - i * lb;
                                hit = kpa[a0 + i] == kpb[b0 + q];
                            }
                            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                            const uint64_t my = ws + __popc(hm & lanemask_lt());
                            if (hit && my < a.cap)
                                st_pair(a.pairs, a.pair8, my, ld_val(a.va, a.val8a, ta + a0 + i),
                                        ld_val(a.vb, a.val8b, tb + b0 + q));
                            ws += __popc(hm);
                        }
                    }
                    slot += cnt[j];
                }
            }
        }
        __syncthreads();
    }
    // block reduction -> one pair of u64 atomics per CTA
    __shared__ unsigned long long s_m[kIsBlock / 32], s_c[kIsBlock / 32];
    matches = warp_sum(matches);
    compared = warp_sum(compared);
    if (lane == 0) {
        s_m[tid >> 5] = matches;
        s_c[tid >> 5] = compared;
    }
    __syncthreads();
    if (tid < 32) {
        unsigned long long x = tid < kIsBlock / 32 ? s_m[tid] : 0;
        unsigned long long y = tid < kIsBlock / 32 ? s_c[tid] : 0;
        x = warp_sum(x);
        y = warp_sum(y);
        if (tid == 0) {
            if (x) atomicAdd(reinterpret_cast<unsigned long long*>(a.totals), x);
            if (y) atomicAdd(reinterpret_cast<unsigned long long*>(a.totals + 1), y);
        }
    }
}

template <typename K>
static cudaError_t intersect_impl(const TableDesc& A, const TableDesc& B, const IntersectArgs& ia,
                                  cudaStream_t s) {
    IsArgs a{};
    a.offa = A.offs;
    a.offb = B.offs;
    a.ka = A.keys;
    a.kb = B.keys;
    a.va = A.vals;
    a.vb = B.vals;
    a.off8a = A.off_bytes == 8;
    a.off8b = B.off_bytes == 8;
    a.val8a = A.val_bytes == 8;
    a.val8b = B.val_bytes == 8;
    a.nv = A.nv;
    a.ntiles = (A.nv + kIsTile - 1) >> kIsTileShift;
    a.pairs = ia.pairs;
    a.pair8 = ia.pair_bytes == 8;
    a.cap = ia.pairs ? ia.cap : 0;
    a.totals = ia.totals;
    // staged key capacity per side: ~1.5x the mean slice + slack, within a
    // ~100 KB per-CTA budget (2+ CTAs per SM); larger slices read global memory
    auto capfor = [&](uint64_t n) {
        const double mean = double(n) * double(kIsTile) / double(A.nv);
        const double lim = double((size_t(40) << 10) / sizeof(K));
        return uint32_t(std::min(lim, std::max(256.0, 1.5 * mean + 256.0)));
    };
    a.kcapa = capfor(A.n);
    a.kcapb = capfor(B.n);
    const bool pairs = ia.pairs != nullptr && ia.cap > 0;
    const size_t smem = is_smem_bytes<K>(a.off8a, a.off8b, a.kcapa, a.kcapb);
    const size_t st_bytes = pairs ? a.ntiles * sizeof(uint64_t) : 0;
    void* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, st_bytes + 16, s);
    if (e != cudaSuccess) return e;
    a.status = static_cast<uint64_t*>(scratch);
    a.ticket = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + st_bytes);
    do {
        if ((e = cudaMemsetAsync(scratch, 0, st_bytes + 16, s)) != cudaSuccess) break;
        auto kern = pairs ? k_intersect<K, true> : k_intersect<K, false>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
            cudaSuccess)
            break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kIsBlock, smem);
        const unsigned grid = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * num_sms(), a.ntiles)));
        HG_LAUNCH(pairs ? "k12_intersect_pairs" : "k12_intersect", s,
                  kern<<<grid, kIsBlock, smem, s>>>(a));
        e = cudaGetLastError();
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

cudaError_t intersect_tables(const TableDesc& A, const TableDesc& B, const IntersectArgs& ia,
                             cudaStream_t s) {
    if (A.key_bytes != B.key_bytes || A.nv != B.nv) return cudaErrorInvalidValue;
    return A.key_bytes == 4 ? intersect_impl<uint32_t>(A, B, ia, s) : intersect_impl<uint64_t>(A, B, ia, s);
}

}  // namespace hg
