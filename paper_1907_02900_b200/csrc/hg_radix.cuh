// hg_radix.cuh -- vertex-range partitioning machinery shared by the binned
// build (V2) and the partitioned probe.
//
// The reference's V2 scatters entries into bins of consecutive vertex ranges
// (core.hpp:192-219) so that the per-vertex passes run cache-resident. On
// B200 the per-partition work runs in shared memory, which needs partitions
// of ~2^12 vertices -- 2^16 partitions at V = 2^28. A one-shot 65536-way
// scatter costs one global atomic and one uncoalesced store per key (measured
// 7.4 ms at 2^28). Instead, partition ids are split into two <= 8-bit digits
// and the entries go through two radix passes whose per-tile ranking runs on
// shared-memory atomics (~1.8 T op/s on B200 vs ~0.13 T op/s for L2
// atomics, profiles/r01_microbench_b200.txt):
//
//   k_part_hist    one pass over the keys; full 2^b partition histogram in
//                  shared memory (two 16-bit halves per word, spilled to the
//                  global histogram every 2^15 increments, so skew cannot
//                  overflow); one global add per (CTA, non-empty partition)
//   scan           exclusive scan of the histogram -> partition starts
//   k_multisplit   per 4096-entry tile: shared-memory rank by digit, one global
//                  atomic per (tile, digit) reserving a contiguous run, then
//                  the tile is written digit-sorted, so stores coalesce into
//                  runs of ~tile/256 entries. Pass 1 splits by the high digit
//                  (reads the raw keys), pass 2 by the low digit within each
//                  high-digit bucket (tiles never straddle a bucket).
#pragma once

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_scan.cuh"

namespace hg {

int num_sms();

// ------------------------------------------------------------ entry types
// An entry is what travels through the passes: (key, value) for the build
// and for probes that need their position; the bare key for count-only probes.
template <typename K, typename VT>
struct EntryT {
    using T = ulonglong2;
    static constexpr bool kHasVal = true;
    __device__ static T make(K k, VT v) { return make_ulonglong2(k, v); }
    __device__ static K key(const T& e) { return K(e.x); }
    __device__ static VT val(const T& e) { return VT(e.y); }
};
template <>
struct EntryT<uint32_t, uint32_t> {
    using T = uint2;
    static constexpr bool kHasVal = true;
    __device__ static T make(uint32_t k, uint32_t v) { return make_uint2(k, v); }
    __device__ static uint32_t key(const T& e) { return e.x; }
    __device__ static uint32_t val(const T& e) { return e.y; }
};
template <typename K>
struct EntryT<K, void> {
    using T = K;
    static constexpr bool kHasVal = false;
    __device__ static T make(K k, uint64_t) { return k; }
    __device__ static K key(const T& e) { return e; }
    __device__ static uint32_t val(const T&) { return 0; }
};

template <int POW2>
__device__ __forceinline__ uint64_t hv(uint64_t key, uint64_t seed, int hk, const Divisor& nv) {
    return vhash<POW2>(key, seed, nv);
}

// ------------------------------------------------------------ geometry

constexpr uint32_t kMaxPartShift = 15;

struct PartGeom {
    uint32_t pshift = 0;  // partition width P = 2^pshift vertices
    uint64_t nparts = 1;  // ceil(V / P)
    uint32_t bits = 0;    // ceil(log2(nparts))
    uint32_t b1 = 0, b2 = 0;  // digit widths (pass 1 high, pass 2 low), b1 + b2 = bits
};

inline uint32_t ceil_log2(uint64_t x) {
    uint32_t b = 0;
    while ((uint64_t(1) << b) < x) ++b;
    return b;
}

// Partition width: aim for ~target entries per partition (N/V * P), at most
// 2^16 partitions (two 8-bit digits) while P <= 2^15, never wider than 2^15
// (2^15 u32 counters + K7's staging fit one CTA's 227 KB for every entry
// type). Callers check g.bits <= 16 (2^31 < V: the binned build slices the
// vertex range first, see build_v2_sliced).
inline PartGeom make_geom(uint64_t nv, uint64_t n, uint64_t want_pv, double target) {
    PartGeom g;
    const uint32_t vbits = ceil_log2(nv);
    uint32_t ps;
    if (want_pv) {
        ps = ceil_log2(want_pv);
    } else {
        const double per_vertex = n ? double(n) / double(nv) : 1.0;
        ps = 0;
        while (ps < kMaxPartShift && per_vertex * double(uint64_t(2) << ps) <= target) ++ps;
    }
    if (vbits > 16 && ps < vbits - 16) ps = vbits - 16;
    if (ps > kMaxPartShift) ps = kMaxPartShift;
    if (ps > vbits) ps = vbits;
    g.pshift = ps;
    g.nparts = (nv + (uint64_t(1) << ps) - 1) >> ps;
    g.bits = ceil_log2(g.nparts);
    g.b2 = g.bits / 2;
    g.b1 = g.bits - g.b2;
    return g;
}

// ------------------------------------------------------------ histogram

constexpr int kHistBlock = 1024;

// In = K (raw keys) or a record type {key, value} (uint2 / ulonglong2: routed
// records of a sharded build, hg_build_records); the key is its first field.
template <typename K, typename In>
__device__ __forceinline__ K key_of(const In& x) {
    if constexpr (std::is_same<In, K>::value) {
        return x;
    } else {
        return K(x.x);
    }
}

template <typename K, typename OffT, int POW2, typename In = K>
__global__ void __launch_bounds__(kHistBlock)
k_part_hist(const In* __restrict__ keys, uint64_t n, uint64_t seed, int hk, Divisor nv,
            uint32_t pshift, uint32_t nparts, OffT* __restrict__ hist, const uint32_t* guard) {
    if (guard && !*guard) return;
    extern __shared__ uint32_t sh[];  // nparts/2 words, two 16-bit counters each
    const uint32_t words = (nparts + 1) >> 1;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    constexpr int VEC = 16 / sizeof(In);
    using V = typename std::conditional<sizeof(In) == 4, uint4, ulonglong2>::type;
    auto count = [&](K key) {
        const uint32_t p = uint32_t(hv<POW2>(key, seed, hk, nv) >> pshift);
        const uint32_t sft = (p & 1) << 4;
        const uint32_t old = atomicAdd(sh + (p >> 1), 1u << sft);
        if (((old >> sft) & 0xFFFFu) == 0x7FFFu) {
            // this increment crossed 2^15: move 2^15 to the global count
            atomicSub(sh + (p >> 1), 0x8000u << sft);
            red_add(hist + p, OffT(0x8000));
        }
    };
    uint64_t head = ((16 - (reinterpret_cast<uintptr_t>(keys) & 15)) & 15) / sizeof(In);
    if (head > n) head = n;
    const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gtid < head) count(key_of<K>(keys[gtid]));
    const uint64_t nvec = (n - head) / VEC;
    const V* body = reinterpret_cast<const V*>(keys + head);
    // two 16-byte vectors per step, software-pipelined one step ahead so the
    // loads of step i+1 are in flight while step i's keys are counted; vector
    // indices in 32 bits whenever they fit
    auto sweep = [&](auto idx_t) {
        using I = decltype(idx_t);
        const I nv_ = I(nvec), st = I(stride);
        I q = I(gtid);
        V a{}, b{};
        if (q + st < nv_) {
            a = __ldcs(body + q);
            b = __ldcs(body + q + st);
        }
        for (; q + st < nv_; q += 2 * st) {
            const V ca = a, cb = b;
            if (q + 3 * st < nv_) {
                a = __ldcs(body + q + 2 * st);
                b = __ldcs(body + q + 3 * st);
            }
            const In* ka = reinterpret_cast<const In*>(&ca);
            const In* kb = reinterpret_cast<const In*>(&cb);
#pragma unroll
            for (int k = 0; k < VEC; ++k) count(key_of<K>(ka[k]));
#pragma unroll
            for (int k = 0; k < VEC; ++k) count(key_of<K>(kb[k]));
        }
        if (q < nv_) {
            const V a1 = __ldcs(body + q);
            const In* ka = reinterpret_cast<const In*>(&a1);
#pragma unroll
            for (int k = 0; k < VEC; ++k) count(key_of<K>(ka[k]));
        }
    };
    if (nvec + 4 * stride < (uint64_t(1) << 32)) sweep(uint32_t(0));
    else sweep(uint64_t(0));
    const uint64_t done = head + nvec * VEC;
    if (gtid < n - done) count(key_of<K>(keys[done + gtid]));
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < nparts; p += blockDim.x) {
        const uint32_t c = (sh[p >> 1] >> ((p & 1) << 4)) & 0xFFFFu;
        if (c) red_add(hist + p, OffT(c));
    }
}

// ------------------------------------------------------------ multisplit

constexpr int kSplitBlock = 512;
#ifndef HG_SPLIT_STAGES
#define HG_SPLIT_STAGES 2
#endif
constexpr int kSplitStages = HG_SPLIT_STAGES;  // TMA input stages (one tile prefetched ahead)
#ifndef HG_P2_STAGES
#define HG_P2_STAGES kSplitStages
#endif
#ifndef HG_P2_ITEMS_Q
#define HG_P2_ITEMS_Q 4  // pass-2 items per thread = the pass-1 count * Q / 4
#endif
// TMA input stages of a pass
template <bool PASS2>
__host__ __device__ constexpr int split_stages() { return PASS2 ? HG_P2_STAGES : kSplitStages; }
constexpr int kMaxDigits = 256;
constexpr uint32_t kOwnerRun = 64;  // digit runs up to this long are filled by their owner
// Consumer threads of a pass: pass 2 runs one producer warp (TMA refills)
// beside 15 consumer warps, pass 1 lets thread 0 issue its (cheap) refills.
template <bool PASS2>
__host__ __device__ constexpr int split_cons() { return PASS2 ? kSplitBlock - 32 : kSplitBlock; }
// 16 / 8 / 4 entries per consumer thread for 4- / 8- / 16-byte entries.
template <typename E>
__host__ __device__ constexpr int split_items() { return sizeof(E) >= 16 ? 4 : sizeof(E) <= 4 ? 16 : 8; }
template <typename E, bool PASS2>
__host__ __device__ constexpr int pass_items() { return PASS2 ? split_items<E>() * HG_P2_ITEMS_Q / 4 : split_items<E>(); }
template <typename E, bool PASS2 = false>
__host__ __device__ constexpr int split_tile() { return split_cons<PASS2>() * pass_items<E, PASS2>(); }

// One radix pass. RAW: input is the raw key array (+ optional vals, else the
// input position is the value). Otherwise input is an entry array.
// Digit of an entry = (p >> dshift) & dmask with p = partition id; the run
// for digit d of a tile is reserved on cursor[cbase(tile) + d], where cbase is
// 0 for pass 1 and (bucket << b2) for pass 2.
// PASS2: tiles are laid out bucket by bucket; tile_prefix[b] = first tile of
// high-digit bucket b (nb1 + 1 entries, cached in shared memory), bucket b
// spans [part_start[b << b2], part_start[(b+1) << b2]).
// Input tiles are double-buffered in shared memory by TMA 1-D bulk copies
// (cp.async.bulk + mbarrier): tile i+1 streams in while tile i is ranked,
// staged digit-sorted in shared memory and written out in coalesced runs.
template <typename K, typename VT, bool RAW, bool PASS2 = false>
struct SplitLayout {
    using E = typename EntryT<K, VT>::T;
    using InT = typename std::conditional<RAW, K, E>::type;
    static constexpr int kItems = pass_items<E, PASS2>();
    static constexpr int kTile = split_tile<E, PASS2>();
    static constexpr int kStages = split_stages<PASS2>();
    static constexpr size_t kInBytes = (size_t(kTile) * sizeof(InT) + 32 + 15) & ~size_t(15);
    static constexpr size_t kBytes = kStages * kInBytes + size_t(kTile) * sizeof(E) + kTile + 16;
};

// CTAs per SM the layout allows (<= 227 KB of shared memory per SM): 3 when
// the tile buffers are small, else 2; the register cap follows from it.
template <typename K, typename VT, bool RAW, bool PASS2 = false>
constexpr int split_min_blocks() {
    return SplitLayout<K, VT, RAW, PASS2>::kBytes * 3 <= size_t(220) * 1024 ? 3 : 2;
}

template <typename K, typename VT, typename OffT, bool RAW, bool PASS2, int POW2>
__global__ void __launch_bounds__(kSplitBlock, (split_min_blocks<K, VT, RAW, PASS2>()))
k_multisplit(const void* __restrict__ in, const VT* __restrict__ vals, uint64_t val_base,
             uint64_t n, uint64_t seed,
             int hk, Divisor nv, uint32_t pshift, uint32_t dshift, uint32_t dmask, uint32_t b2,
             OffT* __restrict__ cursor, const OffT* __restrict__ part_start, uint32_t nb1,
             const uint64_t* __restrict__ tile_prefix, uint64_t ntiles, uint64_t nparts,
             typename EntryT<K, VT>::T* __restrict__ out, const uint32_t* guard, uint64_t out_cap,
             uint32_t* overflow, const OffT* __restrict__ in_end, uint64_t in_cap) {
    // guard: device-side skip (exact fallback of partition_slack).
    // out_cap > 0: digit region r = cbase + d of `out` starts at r * out_cap
    //   and holds out_cap entries; a run that would cross its end sets
    //   *overflow (the caller falls back to the exact path) and is written,
    //   in bounds, over the region's end instead.
    // in_end != nullptr (PASS2): input bucket b is [b * in_cap, in_end[b]).
    if (guard && !*guard) return;
    // slack pass 2 after an overflowing pass 1: the exact path redoes it
    // (or a slack pass 1 when k_skew_sample already predicted the overflow)
    if (out_cap && *reinterpret_cast<volatile const uint32_t*>(overflow)) return;
    using ET = EntryT<K, VT>;
    using E = typename ET::T;
    using L = SplitLayout<K, VT, RAW, PASS2>;
    constexpr int kSt = L::kStages;
    using InT = typename L::InT;
    constexpr int kItems = L::kItems;
    constexpr int kTile = L::kTile;
    // pass 2 is warp-specialised: a producer warp streams the input tiles
    // (full / empty mbarriers per stage), so its refill -- forward bucket
    // walk, bulk-copy issue, overflow poll -- never sits in front of the
    // consumers' barrier (with thread 0 issuing it did: ~15 % of K6b's stall
    // samples). Pass 1's refill is a multiply, so thread 0 keeps issuing it
    // and all 16 warps rank.
    constexpr bool kProd = PASS2;
    constexpr uint32_t kCons = split_cons<PASS2>();
    extern __shared__ __align__(128) unsigned char smem[];
    E* const s_ent = reinterpret_cast<E*>(smem + kSt * L::kInBytes);
    uint8_t* const s_dig = reinterpret_cast<uint8_t*>(s_ent + kTile);
    __shared__ uint64_t s_bar[kSt];    // stage full (TMA landed)
    __shared__ uint64_t s_empty[kSt];  // stage consumed (producer mode)
    __shared__ uint64_t s_t0[kSt], s_t1[kSt], s_cb[kSt];
    __shared__ uint32_t s_ofs[kSt], s_ok[kSt];
    __shared__ uint32_t s_cnt[kMaxDigits];
    __shared__ uint32_t s_long[kMaxDigits];  // digits whose run is filled cooperatively
    __shared__ uint32_t s_nlong;
    __shared__ uint32_t s_off[kMaxDigits];
    // reserved global base - tile offset of each digit, in the offsets' width
    // (modular: base - off + j is the exact output index for j >= off)
    __shared__ OffT s_gbo[kMaxDigits];
    __shared__ uint64_t s_tp[PASS2 ? kMaxDigits + 1 : 1];  // tile_prefix cache
    // bucket start cache (dense layout) / bucket end cache (slack layout,
    // where bucket b starts at b * in_cap)
    __shared__ uint64_t s_bs[PASS2 ? kMaxDigits + 1 : 1];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ndig = dmask + 1;

    if constexpr (PASS2) {
        for (uint32_t b = tid; b <= nb1; b += kSplitBlock) {
            s_tp[b] = tile_prefix[b];
            if (in_end) {
                const uint64_t e = b < nb1 ? uint64_t(in_end[b]) : 0, lim = uint64_t(b + 1) * in_cap;
                s_bs[b] = e < lim ? e : lim;
            } else {
                const uint64_t q = (uint64_t(b) << b2) < nparts ? (uint64_t(b) << b2) : nparts;
                s_bs[b] = part_start[q];
            }
        }
        __syncthreads();
    }
    // (thread 0) range of a tile; false when past the last real tile. A CTA's
    // tiles only increase, so its bucket is tracked by a forward walk (no
    // search, no global load: the refill sits in front of a block barrier).
    uint32_t lo = 0;
    auto tile_range = [&](uint64_t tile, uint64_t& t0, uint64_t& t1, uint64_t& cbase) -> bool {
        if constexpr (PASS2) {
            if (tile >= s_tp[nb1]) return false;
            while (s_tp[lo + 1] <= tile) ++lo;
            uint64_t be;
            if (in_end) {
                t0 = uint64_t(lo) * in_cap + (tile - s_tp[lo]) * kTile;
                be = s_bs[lo];
            } else {
                t0 = s_bs[lo] + (tile - s_tp[lo]) * kTile;
                be = s_bs[lo + 1];
            }
            t1 = be < t0 + kTile ? be : t0 + kTile;
            cbase = uint64_t(lo) << b2;
        } else {
            if (tile >= ntiles) return false;
            t0 = tile * kTile;
            t1 = n < t0 + kTile ? n : t0 + kTile;
            cbase = 0;
        }
        return true;
    };
    auto issue = [&](uint64_t tile, int st, uint32_t abort) {
        uint64_t t0 = 0, t1 = 0, cb = 0;
        // a slack layout that already overflowed (skewed keys) stops early:
        // the exact path redoes the pass. Stages issued before stay valid and
        // are consumed, so no bulk copy is in flight when the CTA exits.
        const bool ok = !abort && tile_range(tile, t0, t1, cb);
        s_ok[st] = ok;
        s_t0[st] = t0;
        s_t1[st] = t1;
        s_cb[st] = cb;
        if (ok) {
            // s_ofs is written before the arrive below releases the stage
            const uintptr_t a = reinterpret_cast<uintptr_t>(static_cast<const InT*>(in) + t0);
            const uintptr_t alo = a & ~uintptr_t(15);
            const uint32_t len = uint32_t(((a + (t1 - t0) * sizeof(InT) + 15) & ~uintptr_t(15)) - alo);
            s_ofs[st] = uint32_t(a - alo);
            fence_proxy_async();
            mbar_arrive_expect_tx(&s_bar[st], len);
            tma_load_1d(smem + st * L::kInBytes, reinterpret_cast<const void*>(alo), len, &s_bar[st]);
        }
    };

    if (tid == 0) {
        for (int st = 0; st < kSt; ++st) {
            mbar_init(&s_bar[st], 1);
            mbar_init(&s_empty[st], 1);
        }
        fence_mbar_init();
        if constexpr (!kProd)
            for (int st = 0; st < kSt - 1; ++st) issue(blockIdx.x + uint64_t(st) * gridDim.x, st, 0u);
    }
    __syncthreads();
    if constexpr (kProd) {
        if (tid >= kCons) {
            if (tid == kCons) {
                uint32_t abort = 0;
                for (uint64_t i = 0;; ++i) {
                    const int sp = int(i % kSt);
                    if (i >= uint64_t(kSt))
                        mbar_wait(&s_empty[sp], uint32_t((i / kSt - 1) & 1));
                    issue(blockIdx.x + i * gridDim.x, sp, abort);
                    if (!s_ok[sp]) {
                        mbar_arrive(&s_bar[sp]);  // releases s_ok = 0: the consumers stop
                        break;
                    }
                    if (out_cap) abort = *reinterpret_cast<volatile const uint32_t*>(overflow);
                }
            }
            return;
        }
    }
    // block barrier of the consumers (the producer warp never joins it)
    auto bsync = [] {
        if constexpr (kProd) asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
        else __syncthreads();
    };
    uint64_t tile = blockIdx.x;
    int st = 0;
    uint32_t phase = 0;
    // (thread 0) overflow flag, polled every 16th tile and used one tile
    // later, so the load's latency stays off the refill path. Only for 16-byte
    // entries (C3's u64 keys + values, where a wasted pass costs the most):
    // measured on the 8-byte passes of C2, even this poll costs K6a 2-4 %.
    constexpr bool kPoll = sizeof(E) >= 16;
    uint32_t ovf = 0, iter = 0;
    // digit counters are zeroed here for the first tile and during the
    // write-out of the previous tile for the others, so a tile starts without
    // a barrier (each thread waits on the stage's mbarrier itself)
    for (uint32_t d = tid; d < ndig; d += kCons) s_cnt[d] = 0;
    if (tid == 0) s_nlong = 0;
    bsync();
    for (;; tile += gridDim.x) {
        if constexpr (kProd) {
            mbar_wait(&s_bar[st], phase);
            if (!s_ok[st]) break;
        } else {
            if (!s_ok[st]) break;
            // refill the stage consumed in the previous iteration
            const int pf = st == 0 ? kSt - 1 : st - 1;
            if (tid == 0) {
                issue(tile + uint64_t(kSt - 1) * gridDim.x, pf, ovf);
                if (kPoll && out_cap && (++iter & 15) == 0) ovf = *reinterpret_cast<volatile const uint32_t*>(overflow);
            }
            mbar_wait(&s_bar[st], phase);
        }
        const uint64_t t0 = s_t0[st];
        const uint32_t cnt = uint32_t(s_t1[st] - t0);
        const uint64_t cbase = s_cb[st];
        const InT* src = reinterpret_cast<const InT*>(smem + st * L::kInBytes + s_ofs[st]);

        E ent[kItems];
        uint32_t dr[kItems];  // digit << 16 | rank
        // full tiles (all but each bucket's last) run the per-entry loops
        // without bounds checks: no divergent region per item (BSSY / BSYNC /
        // BRA were 15 % of K6b's instructions)
        const bool full = cnt == uint32_t(kTile);
        auto rank_items = [&](auto fullc) {
        constexpr bool F = decltype(fullc)::value;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const uint32_t j = tid + k * kCons;
            if (F || j < cnt) {
                K key;
                if constexpr (RAW) {
                    key = src[j];
                    if constexpr (ET::kHasVal) {
                        ent[k] = ET::make(key, vals ? VT(vals[t0 + j]) : VT(val_base + t0 + j));
                    } else {
                        ent[k] = ET::make(key, 0);
                    }
                } else {
                    ent[k] = src[j];
                    key = ET::key(ent[k]);
                }
                const uint32_t p = uint32_t(hv<POW2>(key, seed, hk, nv) >> pshift);
                const uint32_t d = (p >> dshift) & dmask;
                dr[k] = (d << 16) | atomicAdd(s_cnt + d, 1u);
            }
        }
        };
        if (full) rank_items(std::true_type{});
        else rank_items(std::false_type{});
        bsync();
        // exclusive scan of the <= 256 digit counts + run reservation
        const uint32_t c = tid < ndig ? s_cnt[tid] : 0;
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (int(lane) >= d) inc += y;
        }
        // counts of the digits below this warp's 32, summed by the warp itself
        // (no cross-warp partials, no barrier)
        uint32_t base = 0;
        if (warp * 32 < ndig) {
            for (uint32_t w = 0; w < warp; ++w) base += s_cnt[32 * w + lane];
            base = warp_sum(base);
        }
        OffT gb = 0;
        uint32_t off = 0;
        if (tid < ndig) {
            off = base + inc - c;
            s_off[tid] = off;
            // the run reservation is consumed only after the scatter below, so
            // its L2 round trip overlaps the scatter
            if (c) {
                gb = atom_add(cursor + cbase + tid, OffT(c));
                if (out_cap) {
                    const uint64_t lim = (cbase + tid + 1) * out_cap;
                    if (uint64_t(gb) + c > lim) {  // slack region full: exact fallback
                        *overflow = 1u;
                        gb = OffT(lim >= c ? lim - c : 0);
                    }
                }
            }
            // digit of every slot of this digit's run, written by the digit's
            // owner as a byte run (word stores in the middle) instead of one
            // random byte store per entry in the scatter; runs longer than
            // kOwnerRun (skewed keys) are filled by the whole CTA below
            if (c <= kOwnerRun) {
                uint32_t o = off;
                const uint32_t e = off + c;
                const uint8_t dd = uint8_t(tid);
                while (o < e && (o & 3)) s_dig[o++] = dd;
                const uint32_t w4 = uint32_t(dd) * 0x01010101u;
                for (; o + 4 <= e; o += 4) *reinterpret_cast<uint32_t*>(s_dig + o) = w4;
                while (o < e) s_dig[o++] = dd;
            } else {
                s_long[atomicAdd(&s_nlong, 1u)] = tid;
            }
        }
        bsync();
        if (full) {
#pragma unroll
            for (int k = 0; k < kItems; ++k) s_ent[s_off[dr[k] >> 16] + (dr[k] & 0xFFFFu)] = ent[k];
        } else {
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t j = tid + k * kCons;
                if (j < cnt) s_ent[s_off[dr[k] >> 16] + (dr[k] & 0xFFFFu)] = ent[k];
            }
        }
        for (uint32_t li = 0; li < s_nlong; ++li) {
            const uint32_t d = s_long[li];
            const uint32_t o = s_off[d], e = o + s_cnt[d];
            const uint32_t w0 = (o + 3) >> 2, w1 = e >> 2;  // whole words inside the run
            const uint32_t w4 = d * 0x01010101u;
            for (uint32_t w = w0 + tid; w < w1; w += kCons)
                reinterpret_cast<uint32_t*>(s_dig)[w] = w4;
            if (tid < 4) {
                if (o + tid < 4 * w0) s_dig[o + tid] = uint8_t(d);
                if (4 * w1 + tid < e) s_dig[4 * w1 + tid] = uint8_t(d);
            }
        }
        if (c) s_gbo[tid] = gb - OffT(off);
        bsync();
        // counters of the next tile (s_cnt is not read by the write-out)
        for (uint32_t d = tid; d < ndig; d += kCons) s_cnt[d] = 0;
        if (tid == 0) s_nlong = 0;
        if (full) {
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t j = tid + k * kCons;
                out[uint64_t(OffT(s_gbo[s_dig[j]] + OffT(j)))] = s_ent[j];
            }
        } else {
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t j = tid + k * kCons;
                if (j < cnt) out[uint64_t(OffT(s_gbo[s_dig[j]] + OffT(j)))] = s_ent[j];
            }
        }
        bsync();
        if constexpr (kProd) {
            if (tid == 0) mbar_arrive(&s_empty[st]);  // stage st free for the producer
        }
        if (++st == kSt) {
            st = 0;
            phase ^= 1;
        }
    }
}

// Pass-2 tile layout: tile_prefix[b] = sum over buckets < b of ceil(size/tile).
// One CTA of kMaxDigits threads: thread b sizes bucket b, then a block scan
// (round 1 ran this as one thread walking 256 dependent global loads:
// ~135 us per launch, twice per C2 step).
template <typename OffT>
__global__ void __launch_bounds__(kMaxDigits)
k_tile_prefix(const OffT* __restrict__ part_start, uint64_t nparts, uint32_t nb1, uint32_t b2,
              uint32_t kSplitTile, uint64_t* __restrict__ tile_prefix, const uint32_t* guard,
              const OffT* __restrict__ in_end, uint64_t in_cap) {
    // in_end != nullptr: bucket b holds in_end[b] - b * in_cap entries (slack layout)
    if (guard && !*guard) return;
    __shared__ uint64_t s_w[kMaxDigits / 32];
    const uint32_t b = threadIdx.x, lane = b & 31, warp = b >> 5;
    uint64_t c = 0;
    if (b < nb1) {
        uint64_t sz;
        if (in_end) {
            const uint64_t lo = uint64_t(b) * in_cap, e = uint64_t(in_end[b]);
            sz = (e < lo + in_cap ? e : lo + in_cap) - lo;
        } else {
            const uint64_t hi = (uint64_t(b + 1) << b2) < nparts ? (uint64_t(b + 1) << b2) : nparts;
            sz = uint64_t(part_start[hi]) - uint64_t(part_start[uint64_t(b) << b2]);
        }
        c = (sz + kSplitTile - 1) / kSplitTile;
    }
    uint64_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (int(lane) >= d) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint64_t base = 0;
    for (uint32_t w = 0; w < warp; ++w) base += s_w[w];
    if (b < nb1) tile_prefix[b] = base + inc - c;
    if (b == nb1 - 1) tile_prefix[nb1] = base + inc;
}

template <typename OffT>
__global__ void k_init_cursors(const OffT* __restrict__ part_start, uint64_t nparts, uint32_t b2,
                               uint32_t nb1, OffT* __restrict__ cur1, OffT* __restrict__ cur2,
                               const uint32_t* guard) {
    if (guard && !*guard) return;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nparts; p += stride) {
        cur2[p] = part_start[p];
        if ((p & ((uint64_t(1) << b2) - 1)) == 0 && (p >> b2) < nb1) cur1[p >> b2] = part_start[p];
    }
}

// Slack layout (partition_slack): pass-1 bucket b at b * cap1, partition p at
// p * cap2.
template <typename OffT>
__global__ void k_init_cursors_slack(uint64_t nparts, uint32_t b2, uint32_t nb1, uint64_t cap1,
                                     uint64_t cap2, OffT* __restrict__ cur1, OffT* __restrict__ cur2) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nparts; p += stride) {
        cur2[p] = OffT(p * cap2);
        if ((p & ((uint64_t(1) << b2) - 1)) == 0 && (p >> b2) < nb1) cur1[p >> b2] = OffT((p >> b2) * cap1);
    }
}

// Partition counts of the slack layout (cursor - region start) -> hist.
template <typename OffT>
__global__ void k_slack_counts(const OffT* __restrict__ cur2, uint64_t nparts, uint64_t cap2,
                               OffT* __restrict__ counts) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nparts; p += stride)
        counts[p] = OffT(uint64_t(cur2[p]) - p * cap2);
}

// Scratch for partition(): histogram, cursors, tile prefix, scan status and
// one intermediate entry array (pass-1 output).
template <typename K, typename VT, typename OffT>
struct PartitionScratch {
    using E = typename EntryT<K, VT>::T;
    static size_t up(size_t x) { return (x + 255) / 256 * 256; }
    // mid_entries: pass-1 output capacity (slack layout), at least n
    static size_t bytes(const PartGeom& g, uint64_t n, uint64_t mid_entries = 0) {
        return up((g.nparts + 1) * sizeof(OffT)) * 2 + up(((uint64_t(1) << g.b1) + 1) * sizeof(OffT)) +
               up(((uint64_t(1) << g.b1) + 2) * 8) + up(scan_scratch_bytes(g.nparts)) +
               (g.b2 ? up((mid_entries > n ? mid_entries : n) * sizeof(E)) : 0);
    }
};

// Reorders n entries (raw keys [+ vals] on input) into partition order:
// out[part_start[p] .. part_start[p+1]) holds the entries of partition p
// (p = h(key) >> pshift). part_start (nparts + 1 entries, device) receives
// the partition offsets; part_start[nparts] = n.
// Optimistic ("slack") layout of a two-pass partition: pass-1 bucket b is
// written to [b * cap1, b * cap1 + count_b) and partition p to
// [p * cap2, p * cap2 + count_p), capacities ~8 sigma above the mean of a
// uniform hash, so no histogram pass is needed; the exact partition starts
// come from a scan of the final cursors. A region that overflows (skewed
// keys) sets *flag, and the exact path (histogram, scan, two passes into the
// dense layout) then runs behind device-side guards -- its kernels exit at
// once when *flag is 0. Consumers read partition p at
// (*flag ? part_start[p] : p * cap2), part_start[p + 1] - part_start[p]
// entries.
struct Slack {
    uint64_t cap1 = 0, cap2 = 0;
    uint32_t* flag = nullptr;  // device, zeroed by the caller
};

// Slack capacity of a region expecting `mean` entries: `factor` x the mean
// (room for duplicated keys, e.g. multiplicity 32 widens a 4096-entry
// partition's spread from 64 to ~360) plus 8 sigma of a Poisson count.
inline uint64_t slack_cap(double mean, double factor) {
    return uint64_t(factor * mean + 8.0 * std::sqrt(mean > 1.0 ? mean : 1.0) + 64.0);
}

// Slack capacities for n entries over geometry g (two passes), or none
// (cap1 = cap2 = 0) when the slack layout would not fit the offsets' width.
template <typename OffT>
inline Slack make_slack(const PartGeom& g, uint64_t n, uint64_t nv, uint32_t* flag) {
    Slack sl;
    if (g.b2 == 0 || n < (uint64_t(1) << 20)) return sl;
    const uint32_t nb1 = uint32_t((g.nparts + (uint64_t(1) << g.b2) - 1) >> g.b2);
    const double per_vertex = double(n) / double(nv);
    sl.cap2 = slack_cap(per_vertex * double(uint64_t(1) << g.pshift), 1.5);
    sl.cap1 = slack_cap(per_vertex * double(uint64_t(1) << (g.pshift + g.b2)), 1.25);
    sl.flag = flag;
    const uint64_t lim = sizeof(OffT) == 4 ? (uint64_t(1) << 32) - 1 : ~uint64_t(0) >> 2;
    if (double(nb1) * double(sl.cap1) >= double(lim) || double(g.nparts) * double(sl.cap2) >= double(lim))
        return Slack{};
    return sl;
}

// Slack pre-check for 16-byte entries (C3's u64 keys + values, where a
// wasted optimistic pass costs the most): one CTA hashes a strided sample of
// kSkewSample keys into their pass-1 digits. A digit whose sampled count is
// above `thresh` (twice its slack region's share of the sample) means pass 1
// would overflow, so *flag is set before it starts and the exact path runs
// without the aborted optimistic pass (C3 at load 1: ~0.3 ms). Uniform keys
// sit ~12 sigma below the threshold; milder skew is still caught by the
// in-pass overflow check.
constexpr uint32_t kSkewSample = 16384;
constexpr int kSkewBlock = 1024;

template <typename K, int POW2, typename In>
__global__ void __launch_bounds__(kSkewBlock)
k_skew_sample(const In* __restrict__ keys, uint64_t n, uint64_t seed, int hk, Divisor nv,
              uint32_t shift, uint32_t ndig, uint32_t thresh, uint32_t* __restrict__ flag) {
    __shared__ uint32_t h[kMaxDigits];
    for (uint32_t d = threadIdx.x; d < ndig; d += kSkewBlock) h[d] = 0;
    __syncthreads();
    const uint64_t step = n / kSkewSample;
    constexpr int kPer = int(kSkewSample) / kSkewBlock;
    K key[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) key[k] = key_of<K>(keys[uint64_t(threadIdx.x + k * kSkewBlock) * step]);
#pragma unroll
    for (int k = 0; k < kPer; ++k) atomicAdd(h + uint32_t(hv<POW2>(key[k], seed, hk, nv) >> shift), 1u);
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < ndig; d += kSkewBlock)
        if (h[d] > thresh) *flag = 1u;
}

template <typename K, typename VT, typename OffT, int POW2>
cudaError_t partition(const K* keys, const VT* vals, uint64_t n, uint64_t seed, int hk,
                      const Divisor& nv, const PartGeom& g, OffT* part_start, void* scratch,
                      typename EntryT<K, VT>::T* out, cudaStream_t s, const char* const names[3],
                      const typename EntryT<K, VT>::T* rec = nullptr, uint64_t val_base = 0,
                      const Slack* slack = nullptr) {
    using PS = PartitionScratch<K, VT, OffT>;
    using E = typename EntryT<K, VT>::T;
    char* p = static_cast<char*>(scratch);
    OffT* hist = reinterpret_cast<OffT*>(p);
    p += PS::up((g.nparts + 1) * sizeof(OffT));
    OffT* cur2 = reinterpret_cast<OffT*>(p);
    p += PS::up((g.nparts + 1) * sizeof(OffT));
    OffT* cur1 = reinterpret_cast<OffT*>(p);
    p += PS::up(((uint64_t(1) << g.b1) + 1) * sizeof(OffT));
    uint64_t* tile_prefix = reinterpret_cast<uint64_t*>(p);
    p += PS::up(((uint64_t(1) << g.b1) + 2) * 8);
    void* scan_scr = p;
    p += PS::up(scan_scratch_bytes(g.nparts));
    E* mid = reinterpret_cast<E*>(p);

    const bool opt = slack && slack->cap1 && slack->cap2 && g.b2 > 0;
    const uint32_t* guard = opt ? slack->flag : nullptr;
    cudaError_t e = cudaSuccess;
    const int sms = num_sms();
    const uint32_t nb1 = uint32_t((g.nparts + (uint64_t(1) << g.b2) - 1) >> g.b2);
    constexpr int kSplitTile = split_tile<E>();         // pass 1
    constexpr int kSplitTile2 = split_tile<E, true>();  // pass 2 (15 consumer warps)
    const uint64_t tiles1 = (n + kSplitTile - 1) / kSplitTile;
    const uint64_t tiles2 = (n + kSplitTile2 - 1) / kSplitTile2 + nb1;  // upper bound; exact = tile_prefix[nb1]
    // pass 1 reads the raw keys (+ values), or routed records (entries already)
    auto ks1 = rec ? k_multisplit<K, VT, OffT, false, false, POW2>
                   : k_multisplit<K, VT, OffT, true, false, POW2>;
    auto ks2 = k_multisplit<K, VT, OffT, false, true, POW2>;
    const size_t sm1 = rec ? SplitLayout<K, VT, false>::kBytes : SplitLayout<K, VT, true>::kBytes;
    constexpr size_t sm2 = SplitLayout<K, VT, false, true>::kBytes;
    const void* in1 = rec ? static_cast<const void*>(rec) : static_cast<const void*>(keys);
    if ((e = cudaFuncSetAttribute(ks1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1))) !=
            cudaSuccess ||
        (e = cudaFuncSetAttribute(ks2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2))) !=
            cudaSuccess)
        return e;
    int occ1 = 0, occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, ks1, kSplitBlock, sm1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, ks2, kSplitBlock, sm2);
    const unsigned g1 = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>(tiles1, uint64_t(sms) * std::max(1, occ1))));
    const unsigned g2 = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>(tiles2, uint64_t(sms) * std::max(1, occ2))));
    const unsigned gi = unsigned(std::min<uint64_t>((g.nparts + 255) / 256, 1024));

    if (opt) {
        if constexpr (sizeof(E) >= 16) {
            if (n >= uint64_t(kSkewSample) * 64) {
                const double share = double(slack->cap1) / double(n) * double(kSkewSample);
                const uint32_t thresh = uint32_t(std::min(2.0 * share, double(kSkewSample)));
                const uint32_t shift = g.pshift + g.b2, ndig = 1u << g.b1;
                if (rec)
                    k_skew_sample<K, POW2, E><<<1, kSkewBlock, 0, s>>>(rec, n, seed, hk, nv, shift, ndig,
                                                                      thresh, slack->flag);
                else
                    k_skew_sample<K, POW2, K><<<1, kSkewBlock, 0, s>>>(keys, n, seed, hk, nv, shift, ndig,
                                                                      thresh, slack->flag);
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            }
        }
        // ---- optimistic: no histogram, slack regions
        k_init_cursors_slack<OffT><<<gi, 256, 0, s>>>(g.nparts, g.b2, nb1, slack->cap1, slack->cap2,
                                                      cur1, cur2);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        HG_LAUNCH(names[1], s,
                  (ks1<<<g1, kSplitBlock, sm1, s>>>(
                      in1, vals, val_base, n, seed, hk, nv, g.pshift, g.b2,
                      uint32_t((1u << g.b1) - 1), 0, cur1, part_start, 0, nullptr, tiles1,
                      g.nparts, mid, nullptr, slack->cap1, slack->flag, nullptr, 0)));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        k_tile_prefix<OffT><<<1, kMaxDigits, 0, s>>>(part_start, g.nparts, nb1, g.b2, kSplitTile2,
                                                     tile_prefix, nullptr, cur1, slack->cap1);
        HG_LAUNCH(names[2], s,
                  (ks2<<<g2, kSplitBlock, sm2, s>>>(
                      mid, nullptr, 0, n, seed, hk, nv, g.pshift, 0, uint32_t((1u << g.b2) - 1),
                      g.b2, cur2, part_start, nb1, tile_prefix, tiles2, g.nparts, out, nullptr,
                      slack->cap2, slack->flag, cur1, slack->cap1)));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        k_slack_counts<OffT><<<gi, 256, 0, s>>>(cur2, g.nparts, slack->cap2, hist);
        if ((e = launch_scan<OffT, OffT>(hist, part_start, g.nparts, scan_scr, part_start + g.nparts,
                                         s, "part_scan")) != cudaSuccess)
            return e;
        // ---- exact fallback below: every kernel exits at once unless *flag
    }

    if ((e = cudaMemsetAsync(hist, 0, g.nparts * sizeof(OffT), s)) != cudaSuccess) return e;
    const size_t hsmem = ((g.nparts + 1) / 2) * 4;
    auto launch_hist = [&](auto kh, const auto* in) -> cudaError_t {
        cudaError_t r;
        if (hsmem > 48 * 1024 &&
            (r = cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hsmem))) !=
                cudaSuccess)
            return r;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kh, kHistBlock, hsmem);
        unsigned grid = unsigned(std::max(1, per_sm) * sms);
        grid = unsigned(std::max<uint64_t>(
            1, std::min<uint64_t>(grid, (n + kHistBlock * 16 - 1) / (kHistBlock * 16))));
        HG_LAUNCH(guard ? "fallback_hist" : names[0], s,
                  kh<<<grid, kHistBlock, hsmem, s>>>(in, n, seed, hk, nv, g.pshift,
                                                     uint32_t(g.nparts), hist, guard));
        return cudaGetLastError();
    };
    if constexpr (EntryT<K, VT>::kHasVal) {
        e = rec ? launch_hist(k_part_hist<K, OffT, POW2, E>, rec)
                : launch_hist(k_part_hist<K, OffT, POW2>, keys);
    } else {
        e = launch_hist(k_part_hist<K, OffT, POW2>, keys);
    }
    if (e != cudaSuccess) return e;
    if ((e = launch_scan<OffT, OffT>(hist, part_start, g.nparts, scan_scr, part_start + g.nparts, s,
                                     guard ? "fallback_scan" : "part_scan", guard)) != cudaSuccess)
        return e;
    k_init_cursors<OffT><<<gi, 256, 0, s>>>(part_start, g.nparts, g.b2, nb1, cur1, cur2, guard);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (g.b2 == 0) {
        // single pass straight into partition order
        HG_LAUNCH(guard ? "fallback_split1" : names[1], s,
                  (ks1<<<g1, kSplitBlock, sm1, s>>>(
                      in1, vals, val_base, n, seed, hk, nv, g.pshift, 0, uint32_t((1u << g.b1) - 1),
                      0, cur2, part_start, 0, nullptr, tiles1, g.nparts, out, guard, 0, nullptr,
                      nullptr, 0)));
        return cudaGetLastError();
    }
    HG_LAUNCH(guard ? "fallback_split1" : names[1], s,
              (ks1<<<g1, kSplitBlock, sm1, s>>>(
                  in1, vals, val_base, n, seed, hk, nv, g.pshift, g.b2, uint32_t((1u << g.b1) - 1), 0,
                  cur1, part_start, 0, nullptr, tiles1, g.nparts, mid, guard, 0, nullptr, nullptr, 0)));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_tile_prefix<OffT><<<1, kMaxDigits, 0, s>>>(part_start, g.nparts, nb1, g.b2, kSplitTile2,
                                                 tile_prefix, guard, nullptr, 0);
    HG_LAUNCH(guard ? "fallback_split2" : names[2], s,
              (ks2<<<g2, kSplitBlock, sm2, s>>>(
                  mid, nullptr, 0, n, seed, hk, nv, g.pshift, 0, uint32_t((1u << g.b2) - 1), g.b2,
                  cur2, part_start, nb1, tile_prefix, tiles2, g.nparts, out, guard, 0, nullptr,
                  nullptr, 0)));
    return cudaGetLastError();
}

}  // namespace hg
