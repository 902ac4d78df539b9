// hg_intersect.cu -- probe_new_prepared on sm_100a.
//
// Replaces proj/include/hashgraph/join.hpp:143-166 probe_new_prepared and
// its per-vertex nested loop intersect_adjacency (join.hpp:41-57). Two tables
// built over one vertex range hold, at vertex v, exactly the keys hashing to
// v, so every match lives in a segment pair (A_v, B_v). No hashing is needed:
// both CSRs are walked in vertex order, i.e. the kernel is a streaming merge
// of offsA, offsB, keysA, keysB (HBM-bound, every byte read once).
//
//   K12 k_intersect   warp-specialised persistent CTAs. A producer warp takes
//                     vertex tiles (T = 2048) from an atomic ticket and issues
//                     TMA bulk copies of the tile's two offset slices and two
//                     key slices into a 2-stage shared-memory ring (full /
//                     empty mbarriers); 16 consumer warps intersect one tile
//                     while the next is in flight. Consumer thread t owns
//                     the tile vertices j*512 + t (conflict-free offset reads).
//                     A segment pair with both sides <= kShort entries is
//                     compared in registers (B side preloaded, predicated);
//                     longer pairs are flattened (p = i*|B_v| + q) and strided
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

constexpr int kIsBlock = 512;  // consumer threads (16 warps) + 1 producer warp
constexpr uint32_t kIsWarps = kIsBlock / 32;
constexpr uint32_t kIsTileShift = 11;  // 2048 vertices per tile
constexpr uint32_t kIsTile = 1u << kIsTileShift;
constexpr uint32_t kIsVpt = kIsTile / kIsBlock;  // vertices per consumer thread
constexpr uint32_t kShort = 4;                   // short segment pair: both sides <= kShort
constexpr int kIsStages = 2;

struct IsArgs {
    const void* offa;
    const void* offb;
    const void* ka;
    const void* kb;
    const void* va;
    const void* vb;
    int val8a, val8b;
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

__device__ __forceinline__ uint64_t ld_val(const void* p, int val8, uint64_t i) {
    return val8 ? static_cast<const uint64_t*>(p)[i] : static_cast<const uint32_t*>(p)[i];
}
__device__ __forceinline__ void st_pair(void* pairs, int pair8, uint64_t slot, uint64_t l, uint64_t r) {
    if (pair8) reinterpret_cast<ulonglong2*>(pairs)[slot] = make_ulonglong2(l, r);
    else reinterpret_cast<uint2*>(pairs)[slot] = make_uint2(uint32_t(l), uint32_t(r));
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Consumer-side wait: back off between polls so waiting warps do not steal
// issue slots from the warps that are comparing.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    while (!mbar_try(bar, parity)) __nanosleep(64);
}

// Barrier among the kIsBlock consumer threads (the producer warp is not in it).
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kIsBlock) : "memory");
}

__host__ __device__ inline size_t is_span_bytes(size_t bytes) { return (bytes + 32 + 15) & ~size_t(15); }

template <typename K, typename OA, typename OB>
struct IsLayout {
    __host__ __device__ static size_t offa() { return is_span_bytes(size_t(kIsTile + 1) * sizeof(OA)); }
    __host__ __device__ static size_t offb() { return is_span_bytes(size_t(kIsTile + 1) * sizeof(OB)); }
    __host__ __device__ static size_t keys(uint32_t cap) { return is_span_bytes(size_t(cap) * sizeof(K)); }
    __host__ __device__ static size_t stage(uint32_t kcapa, uint32_t kcapb) {
        return offa() + offb() + keys(kcapa) + keys(kcapb);
    }
};

// Per-stage tile descriptor written by the producer before it arrives on the
// stage's full barrier (release), read by consumers after their wait (acquire).
struct TileInfo {
    uint64_t tile;
    uint64_t ta, tb;    // first A / B entry of the tile
    uint32_t oa, ob;    // byte offsets of the offsets slices inside their buffers
    uint32_t oka, okb;  // byte offsets of the key slices
    uint32_t sta, stb;  // key slice staged in shared memory (else read from global)
};

// Segment pair of tile-local vertex v relative to the tile's key slices.
template <typename OA, typename OB>
struct Seg {
    OA a0, la;
    OB b0, lb;
};

template <typename OA, typename OB>
__device__ __forceinline__ Seg<OA, OB> seg_of(const OA* soa, const OB* sob, uint32_t v, OA ta, OB tb) {
    Seg<OA, OB> s;
    const OA x0 = soa[v], x1 = soa[v + 1];
    const OB y0 = sob[v], y1 = sob[v + 1];
    s.a0 = x0 - ta;
    s.la = x1 - x0;
    s.b0 = y0 - tb;
    s.lb = y1 - y0;
    return s;
}

// Short segment pair (both sides <= kShort): the B side is preloaded into
// registers under predicates, then each A entry is compared against it.
// When EMIT, matches are written in (A position, B position) order from
// slot `sl`; ga0 / gb0 are the pair's first global entry indices.
template <typename K, bool EMIT>
__device__ __forceinline__ uint32_t short_pair(const K* __restrict__ pa, uint32_t la,
                                               const K* __restrict__ pb, uint32_t lb, uint64_t sl,
                                               const IsArgs& a, uint64_t ga0, uint64_t gb0) {
    K kb[kShort];
    bool in[kShort];
#pragma unroll
    for (uint32_t q = 0; q < kShort; ++q) {
        in[q] = q < lb;
        kb[q] = in[q] ? pb[q] : K(0);
    }
    uint32_t c = 0;
    for (uint32_t i = 0; i < la; ++i) {
        const K x = pa[i];
#pragma unroll
        for (uint32_t q = 0; q < kShort; ++q) {
            const bool hit = in[q] && x == kb[q];
            if constexpr (EMIT) {
                if (hit) {
                    if (sl < a.cap)
                        st_pair(a.pairs, a.pair8, sl, ld_val(a.va, a.val8a, ga0 + i),
                                ld_val(a.vb, a.val8b, gb0 + q));
                    ++sl;
                }
            }
            c += hit;
        }
    }
    return c;
}

// Count-only segment pair with the inner side <= kShort entries (preloaded
// under predicates) and an outer side of any (small) length.
template <typename K>
__device__ __forceinline__ uint32_t short_count(const K* __restrict__ po, uint32_t lo,
                                                const K* __restrict__ pi, uint32_t li) {
    K kb[kShort];
    bool in[kShort];
#pragma unroll
    for (uint32_t q = 0; q < kShort; ++q) {
        in[q] = q < li;
        kb[q] = in[q] ? pi[q] : K(0);
    }
    uint32_t neg = 0;
    for (uint32_t i = 0; i < lo; ++i) {
        const K x = po[i];
        neg += eq_and(x, kb[0], in[0]) + eq_and(x, kb[1], in[1]) + eq_and(x, kb[2], in[2]) +
               eq_and(x, kb[3], in[3]);
    }
    return 0u - neg;
}

// Long segment pair (a0, la, b0, lb already broadcast): the |A|*|B|
// comparisons are flattened (p = i*lb + q) and strided over the warp.
// Returns the warp-total match count (all lanes); when EMIT, pairs go to
// consecutive slots from `sl` in p order (ballot + popc ranks).
template <typename K, bool EMIT>
__device__ __forceinline__ uint64_t long_pair(const K* __restrict__ kpa, const K* __restrict__ kpb,
                                              uint64_t a0, uint64_t la, uint64_t b0, uint64_t lb,
                                              uint64_t sl, const IsArgs& a, uint64_t ta, uint64_t tb) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t work = la * lb;
    uint64_t c = 0;
    auto loop = [&](auto work_t) {
        using I = decltype(work_t);
        const I w = I(work), l = I(lb);
        if constexpr (!EMIT) {
            for (I p = lane; p < w; p += 32) {
                const I i = p / l, q = p - i * l;
                c += kpa[a0 + i] == kpb[b0 + q];
            }
        } else {
            for (I p0 = 0; p0 < w && sl < a.cap; p0 += 32) {
                const I p = p0 + lane;
                I i = 0, q = 0;
                bool hit = false;
                if (p < w) {
                    i = p / l;
                    q = p - i * l;
                    hit = kpa[a0 + i] == kpb[b0 + q];
                }
                const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                const uint64_t my = sl + __popc(hm & lanemask_lt());
                if (hit && my < a.cap)
                    st_pair(a.pairs, a.pair8, my, ld_val(a.va, a.val8a, ta + a0 + i),
                            ld_val(a.vb, a.val8b, tb + b0 + q));
                sl += __popc(hm);
                if (lane == 0) c += __popc(hm);
            }
        }
    };
    if (work + 32 < (uint64_t(1) << 32)) loop(uint32_t(0));
    else loop(uint64_t(0));
    return warp_sum(c);
}

// One tile, consumer side. kpa / kpb point at the tile's key slices (shared
// memory when staged: the instantiation with shared pointers compiles to LDS).
// Count mode accumulates into matches / compared; pairs mode also writes the
// tile's pairs (needs the consumer barrier and the look-back).
template <typename K, typename OA, typename OB, bool PAIRS>
__device__ __forceinline__ void intersect_tile(const IsArgs& a, const OA* soa, const OB* sob,
                                               const K* kpa, const K* kpb, uint64_t tile,
                                               uint64_t ta, uint64_t tb, uint64_t& matches,
                                               uint64_t& compared, uint32_t (*s_cnt)[kIsBlock],
                                               uint64_t* s_wt, uint64_t* s_base,
                                               uint32_t (*s_q)[kIsVpt * 32]) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t vb = tile << kIsTileShift;
    const uint32_t pv = uint32_t(a.nv - vb < kIsTile ? a.nv - vb : uint64_t(kIsTile));
    const OA tA = OA(ta);
    const OB tB = OB(tb);
    // Phase 1: every vertex's segment pair; comparisons; compact the vertices
    // with both sides non-empty (~40% at load 1) into this warp's queue, so
    // the compare loops run densely instead of over 60% idle lanes.
    uint32_t* const q = s_q[warp];
    uint32_t nq = 0;
    uint64_t cmp_tile = 0;
#pragma unroll
    for (uint32_t j = 0; j < kIsVpt; ++j) {
        const uint32_t v = j * kIsBlock + tid;
        Seg<OA, OB> sp{0, 0, 0, 0};
        if (v < pv) sp = seg_of(soa, sob, v, tA, tB);
        cmp_tile += uint64_t(sp.la) * uint64_t(sp.lb);
        const bool act = sp.la && sp.lb;
        const uint32_t m = __ballot_sync(0xffffffffu, act);
        if (act) q[nq + __popc(m & lanemask_lt())] = v;
        nq += __popc(m);
        if constexpr (PAIRS) s_cnt[j][tid] = 0;
    }
    __syncwarp();
    // Phase 2: the queued segment pairs, 32 at a time. Pairs mode re-queues
    // (in place) the vertices that matched, for the write pass.
    compared += cmp_tile;
    uint32_t nq2 = 0;
    for (uint32_t k0 = 0; k0 < nq; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool act = k < nq;
        const uint32_t v = act ? q[k] : 0;
        Seg<OA, OB> sp{0, 0, 0, 0};
        if (act) sp = seg_of(soa, sob, v, tA, tB);
        // short classes: B side <= kShort with A <= 2*kShort (A outer), or,
        // counting only, A side <= kShort with B <= 2*kShort (B outer)
        const bool sb = sp.lb <= kShort && sp.la <= 2 * kShort;
        const bool sa = !PAIRS && !sb && sp.la <= kShort && sp.lb <= 2 * kShort;
        const bool lg = act && !sb && !sa;
        uint32_t c = 0;
        if (act && sb) {
            if constexpr (PAIRS)
                c = short_pair<K, false>(kpa + sp.a0, uint32_t(sp.la), kpb + sp.b0, uint32_t(sp.lb), 0, a, 0, 0);
            else
                c = short_count<K>(kpa + sp.a0, uint32_t(sp.la), kpb + sp.b0, uint32_t(sp.lb));
        } else if (act && sa) {
            c = short_count<K>(kpb + sp.b0, uint32_t(sp.lb), kpa + sp.a0, uint32_t(sp.la));
        }
        uint32_t wl = __ballot_sync(0xffffffffu, lg);
        while (wl) {
            const int src = __ffs(wl) - 1;
            wl &= wl - 1;
            const uint64_t cl = long_pair<K, false>(
                kpa, kpb, __shfl_sync(0xffffffffu, uint64_t(sp.a0), src),
                __shfl_sync(0xffffffffu, uint64_t(sp.la), src), __shfl_sync(0xffffffffu, uint64_t(sp.b0), src),
                __shfl_sync(0xffffffffu, uint64_t(sp.lb), src), 0, a, ta, tb);
            if (int(lane) == src) c = uint32_t(cl);
        }
        if constexpr (PAIRS) {
            if (c) s_cnt[v / kIsBlock][v % kIsBlock] = c;
            const uint32_t mm = __ballot_sync(0xffffffffu, c != 0);
            __syncwarp();
            if (c) q[nq2 + __popc(mm & lanemask_lt())] = v;
            nq2 += __popc(mm);
            __syncwarp();
        } else {
            matches += c;
        }
    }
    if constexpr (PAIRS) {
        // exclusive rank of each (j, tid) in vertex order j*kIsBlock + tid
        __syncwarp();
#pragma unroll
        for (uint32_t j = 0; j < kIsVpt; ++j) {
            const uint32_t c = s_cnt[j][tid];
            const uint32_t inc = warp_inclusive_sum(c);
            s_cnt[j][tid] = inc - c;  // warp-exclusive
            if (lane == 31) s_wt[j * kIsWarps + warp] = inc;
            matches += c;
        }
        consumer_sync();
        constexpr uint32_t kPer = kIsVpt * kIsWarps / 32;  // (j, warp) totals per lane
        static_assert(kPer >= 1 && kIsVpt * kIsWarps == 32 * kPer, "scan layout");
        if (warp == 0) {
            uint64_t x[kPer], sum = 0;
#pragma unroll
            for (uint32_t e = 0; e < kPer; ++e) sum += (x[e] = s_wt[kPer * lane + e]);
            const uint64_t inc = warp_inclusive_sum(sum);
            uint64_t run = inc - sum;
#pragma unroll
            for (uint32_t e = 0; e < kPer; ++e) {
                s_wt[kPer * lane + e] = run;
                run += x[e];
            }
            const uint64_t tile_total = __shfl_sync(0xffffffffu, inc, 31);
            // decoupled look-back over tiles (ticket order = tile order)
            uint64_t prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_relaxed_u64(a.status, kScanFlagIncl | tile_total);
            } else {
                if (lane == 0) st_relaxed_u64(a.status + tile, kScanFlagAgg | tile_total);
                int64_t idx = int64_t(tile) - 1;
                while (true) {
                    const int64_t jj = idx - int64_t(lane);
                    uint64_t sw = kScanFlagIncl;
                    if (jj >= 0) {
                        do {
                            sw = ld_relaxed_u64(a.status + jj);
                        } while ((sw >> 62) == 0);
                    }
                    const uint32_t inclm = __ballot_sync(0xffffffffu, (sw >> 62) == 2);
                    const uint32_t stop = inclm ? uint32_t(__ffs(inclm) - 1) : 32u;
                    prefix += warp_sum(lane <= stop ? (sw & kScanValMask) : uint64_t(0));
                    if (inclm) break;
                    idx -= 32;
                }
                if (lane == 0) st_relaxed_u64(a.status + tile, kScanFlagIncl | (prefix + tile_total));
            }
            if (lane == 0) {
                s_base[0] = prefix;
                s_base[1] = tile_total;
            }
        }
        consumer_sync();
        const uint64_t tbase = s_base[0];
        if (tbase < a.cap && s_base[1]) {
            // write pass over the re-queued matching vertices
            for (uint32_t k0 = 0; k0 < nq2; k0 += 32) {
                const uint32_t k = k0 + lane;
                const bool act = k < nq2;
                const uint32_t v = act ? q[k] : 0;
                const uint32_t j = v / kIsBlock, t = v % kIsBlock;
                const uint64_t slot = tbase + s_wt[j * kIsWarps + warp] + s_cnt[j][t];
                Seg<OA, OB> sp{0, 0, 0, 0};
                if (act) sp = seg_of(soa, sob, v, tA, tB);
                const bool go = act && slot < a.cap;
                const bool lg = !(sp.lb <= kShort && sp.la <= 2 * kShort);
                if (go && !lg)
                    short_pair<K, true>(kpa + sp.a0, uint32_t(sp.la), kpb + sp.b0, uint32_t(sp.lb), slot,
                                        a, ta + sp.a0, tb + sp.b0);
                uint32_t wm = __ballot_sync(0xffffffffu, go && lg);
                while (wm) {
                    const int src = __ffs(wm) - 1;
                    wm &= wm - 1;
                    long_pair<K, true>(kpa, kpb, __shfl_sync(0xffffffffu, uint64_t(sp.a0), src),
                                       __shfl_sync(0xffffffffu, uint64_t(sp.la), src),
                                       __shfl_sync(0xffffffffu, uint64_t(sp.b0), src),
                                       __shfl_sync(0xffffffffu, uint64_t(sp.lb), src),
                                       __shfl_sync(0xffffffffu, slot, src), a, ta, tb);
                }
            }
        }
    }
}

template <typename K, typename OA, typename OB, bool PAIRS>
__global__ void __launch_bounds__(kIsBlock + 32, 2)
k_intersect(IsArgs a) {
    using L = IsLayout<K, OA, OB>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t s_full[kIsStages], s_empty[kIsStages];
    __shared__ TileInfo s_info[kIsStages];
    __shared__ uint64_t s_base[2];
    __shared__ uint64_t s_wt[kIsVpt * kIsWarps];
    __shared__ uint32_t s_cnt[PAIRS ? kIsVpt : 1][kIsBlock];
    __shared__ uint32_t s_q[kIsWarps][kIsVpt * 32];  // per-warp queues of tile-local vertices
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t stage_bytes = L::stage(a.kcapa, a.kcapb);
    if (tid == 0) {
        for (int st = 0; st < kIsStages; ++st) {
            mbar_init(&s_full[st], 1);
            mbar_init(&s_empty[st], kIsWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kIsWarps) {
        // ---------------- producer (one thread)
        if (lane == 0) {
            const OA* offa = static_cast<const OA*>(a.offa);
            const OB* offb = static_cast<const OB*>(a.offb);
            for (uint32_t it = 0;; ++it) {
                const int st = int(it % kIsStages);
                if (it >= uint32_t(kIsStages)) mbar_wait(&s_empty[st], ((it / kIsStages) - 1) & 1);
                TileInfo& ti = s_info[st];
                const uint64_t p = atomicAdd(a.ticket, 1u);
                ti.tile = p;
                if (p >= a.ntiles) {
                    mbar_arrive(&s_full[st]);
                    break;
                }
                unsigned char* const b_oa = smem + st * stage_bytes;
                unsigned char* const b_ob = b_oa + L::offa();
                unsigned char* const b_ka = b_ob + L::offb();
                unsigned char* const b_kb = b_ka + L::keys(a.kcapa);
                const uint64_t vb = p << kIsTileShift;
                const uint32_t pv = uint32_t(a.nv - vb < kIsTile ? a.nv - vb : uint64_t(kIsTile));
                const uint64_t ta = offa[vb], tae = offa[vb + pv];
                const uint64_t tb = offb[vb], tbe = offb[vb + pv];
                ti.ta = ta;
                ti.tb = tb;
                ti.sta = tae - ta <= a.kcapa;
                ti.stb = tbe - tb <= a.kcapb;
                auto span = [](uintptr_t ad, size_t bytes, uint32_t& lo_off) -> uint32_t {
                    const uintptr_t lo = ad & ~uintptr_t(15), hi = (ad + bytes + 15) & ~uintptr_t(15);
                    lo_off = uint32_t(ad - lo);
                    return uint32_t(hi - lo);
                };
                const uintptr_t aoa = reinterpret_cast<uintptr_t>(offa + vb);
                const uintptr_t aob = reinterpret_cast<uintptr_t>(offb + vb);
                const uintptr_t aka = reinterpret_cast<uintptr_t>(static_cast<const K*>(a.ka) + ta);
                const uintptr_t akb = reinterpret_cast<uintptr_t>(static_cast<const K*>(a.kb) + tb);
                uint32_t oa, ob, oka = 0, okb = 0;
                const uint32_t la = span(aoa, size_t(pv + 1) * sizeof(OA), oa);
                const uint32_t lb = span(aob, size_t(pv + 1) * sizeof(OB), ob);
                const uint32_t lka = (ti.sta && tae > ta) ? span(aka, size_t(tae - ta) * sizeof(K), oka) : 0;
                const uint32_t lkb = (ti.stb && tbe > tb) ? span(akb, size_t(tbe - tb) * sizeof(K), okb) : 0;
                ti.oa = oa;
                ti.ob = ob;
                ti.oka = oka;
                ti.okb = okb;
                fence_proxy_async();
                mbar_arrive_expect_tx(&s_full[st], la + lb + lka + lkb);
                tma_load_1d(b_oa, reinterpret_cast<const void*>(aoa - oa), la, &s_full[st]);
                tma_load_1d(b_ob, reinterpret_cast<const void*>(aob - ob), lb, &s_full[st]);
                if (lka) tma_load_1d(b_ka, reinterpret_cast<const void*>(aka - oka), lka, &s_full[st]);
                if (lkb) tma_load_1d(b_kb, reinterpret_cast<const void*>(akb - okb), lkb, &s_full[st]);
            }
        }
        return;
    }

    // ---------------- consumers
    uint64_t matches = 0, compared = 0;
    for (uint32_t it = 0;; ++it) {
        const int st = int(it % kIsStages);
        mbar_wait_backoff(&s_full[st], (it / kIsStages) & 1);
        const TileInfo& ti = s_info[st];
        const uint64_t tile = ti.tile;
        if (tile >= a.ntiles) break;
        unsigned char* const b_oa = smem + st * stage_bytes;
        const OA* soa = reinterpret_cast<const OA*>(b_oa + ti.oa);
        const OB* sob = reinterpret_cast<const OB*>(b_oa + L::offa() + ti.ob);
        const K* ska = reinterpret_cast<const K*>(b_oa + L::offa() + L::offb() + ti.oka);
        const K* skb = reinterpret_cast<const K*>(b_oa + L::offa() + L::offb() + L::keys(a.kcapa) + ti.okb);
        const uint64_t ta = ti.ta, tb = ti.tb;
        if (ti.sta && ti.stb) {
            intersect_tile<K, OA, OB, PAIRS>(a, soa, sob, ska, skb, tile, ta, tb, matches, compared,
                                             s_cnt, s_wt, s_base, s_q);
        } else {
            const K* gka = static_cast<const K*>(a.ka) + ta;
            const K* gkb = static_cast<const K*>(a.kb) + tb;
            intersect_tile<K, OA, OB, PAIRS>(a, soa, sob, ti.sta ? ska : gka, ti.stb ? skb : gkb, tile,
                                             ta, tb, matches, compared, s_cnt, s_wt, s_base, s_q);
        }
        // release the stage to the producer
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[st]);
        if constexpr (PAIRS) consumer_sync();  // s_cnt / s_wt / s_base reuse
    }
    // block reduction over the consumers -> one pair of u64 atomics per CTA
    __shared__ unsigned long long s_m[kIsWarps], s_c[kIsWarps];
    matches = warp_sum(matches);
    compared = warp_sum(compared);
    if (lane == 0) {
        s_m[warp] = matches;
        s_c[warp] = compared;
    }
    consumer_sync();
    if (tid < 32) {
        unsigned long long x = tid < kIsWarps ? s_m[tid] : 0;
        unsigned long long y = tid < kIsWarps ? s_c[tid] : 0;
        x = warp_sum(x);
        y = warp_sum(y);
        if (tid == 0) {
            if (x) atomicAdd(reinterpret_cast<unsigned long long*>(a.totals), x);
            if (y) atomicAdd(reinterpret_cast<unsigned long long*>(a.totals + 1), y);
        }
    }
}

template <typename K, typename OA, typename OB>
static cudaError_t intersect_impl(const TableDesc& A, const TableDesc& B, const IntersectArgs& ia,
                                  cudaStream_t s) {
    IsArgs a{};
    a.offa = A.offs;
    a.offb = B.offs;
    a.ka = A.keys;
    a.kb = B.keys;
    a.va = A.vals;
    a.vb = B.vals;
    a.val8a = A.val_bytes == 8;
    a.val8b = B.val_bytes == 8;
    a.nv = A.nv;
    a.ntiles = (A.nv + kIsTile - 1) >> kIsTileShift;
    a.pairs = ia.pairs;
    a.pair8 = ia.pair_bytes == 8;
    a.cap = ia.pairs ? ia.cap : 0;
    a.totals = ia.totals;
    // staged key capacity per side: ~1.25x the mean slice + slack (a uniform
    // tile exceeds it with negligible probability), within a 12 KB per side
    // and stage budget; larger slices are read from global memory
    auto capfor = [&](uint64_t n) {
        const double mean = double(n) * double(kIsTile) / double(A.nv);
        const double lim = double((size_t(12) << 10) / sizeof(K));
        return uint32_t(std::min(lim, std::max(128.0, 1.25 * mean + 128.0)));
    };
    a.kcapa = capfor(A.n);
    a.kcapb = capfor(B.n);
    const bool pairs = ia.pairs != nullptr && ia.cap > 0;
    const size_t smem = kIsStages * IsLayout<K, OA, OB>::stage(a.kcapa, a.kcapb);
    const size_t st_bytes = pairs ? a.ntiles * sizeof(uint64_t) : 0;
    void* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, st_bytes + 16, s);
    if (e != cudaSuccess) return e;
    a.status = static_cast<uint64_t*>(scratch);
    a.ticket = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + st_bytes);
    do {
        if ((e = cudaMemsetAsync(scratch, 0, st_bytes + 16, s)) != cudaSuccess) break;
        auto kern = pairs ? k_intersect<K, OA, OB, true> : k_intersect<K, OA, OB, false>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
            cudaSuccess)
            break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kIsBlock + 32, smem);
        const unsigned grid = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * num_sms(), a.ntiles)));
        HG_LAUNCH(pairs ? "k12_intersect_pairs" : "k12_intersect", s,
                  kern<<<grid, kIsBlock + 32, smem, s>>>(a));
        e = cudaGetLastError();
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

template <typename K>
static cudaError_t intersect_off(const TableDesc& A, const TableDesc& B, const IntersectArgs& ia,
                                 cudaStream_t s) {
    if (A.off_bytes == 4 && B.off_bytes == 4) return intersect_impl<K, uint32_t, uint32_t>(A, B, ia, s);
    if (A.off_bytes == 8 && B.off_bytes == 8) return intersect_impl<K, uint64_t, uint64_t>(A, B, ia, s);
    if (A.off_bytes == 4) return intersect_impl<K, uint32_t, uint64_t>(A, B, ia, s);
    return intersect_impl<K, uint64_t, uint32_t>(A, B, ia, s);
}

cudaError_t intersect_tables(const TableDesc& A, const TableDesc& B, const IntersectArgs& ia,
                             cudaStream_t s) {
    if (A.key_bytes != B.key_bytes || A.nv != B.nv) return cudaErrorInvalidValue;
    return A.key_bytes == 4 ? intersect_off<uint32_t>(A, B, ia, s) : intersect_off<uint64_t>(A, B, ia, s);
}

}  // namespace hg
