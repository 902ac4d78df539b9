// hg_probe_impl.cuh -- probe_standard on sm_100a (kernels + launchers; one
// translation unit per (key, value, offset) width instantiates them, see
// hg_probe.cu).
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
//
// Partitioned probe (large tables): a random probe costs two random HBM
// sector reads (offsets, then keys), which caps the direct kernels at the
// ~40 G random accesses/s of HBM (profiles/r01_microbench_b200.txt). When the
// table is far larger than L2, the probes are first radix-partitioned by
// vertex range with the build's machinery (hg_radix.cuh); k_probe_part then
// stages one partition's offsets and keys slice in shared memory (coalesced)
// and answers every probe of that partition from shared memory.
#pragma once

#include <algorithm>
#include <cmath>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_radix.cuh"
#include "hg_scan.cuh"

namespace hg {

int num_sms();

constexpr int kProbeBlock = 256;
constexpr uint64_t kLongSeg = 32;

template <int POW2>
__device__ __forceinline__ uint64_t pvtx(uint64_t key, uint64_t seed, int hk, const Divisor& nv) {
    return vhash<POW2>(key, seed, nv);
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

template <typename K, typename OffT, int POW2, bool WRITE_COUNTS>
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
            if (len <= kLongSeg) c[k] = seg_count(tkeys + b[k], len, pk[k]);
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

template <typename K, typename VT, typename OffT, typename PT, int POW2>
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

// ------------------------------------------------------------ partitioned

constexpr int kPartProbeBlock = 512;
static const char* const kProbePassNames[3] = {"p4_part_hist", "p6a_multisplit", "p6b_multisplit"};

// Shared memory per CTA: offsets slice (P+1) | table keys slice (kcap) |
// probe entries of the partition (pcap), all filled by TMA bulk copies.
template <typename K, typename OffT, typename PEnt>
struct ProbeLayout {
    __host__ __device__ static size_t off_bytes(uint32_t P) { return (size_t(P + 1) * sizeof(OffT) + 32 + 15) & ~size_t(15); }
    __host__ __device__ static size_t key_bytes(uint32_t kcap) { return (size_t(kcap) * sizeof(K) + 32 + 15) & ~size_t(15); }
    __host__ __device__ static size_t ent_bytes(uint32_t pcap) { return (size_t(pcap) * sizeof(PEnt) + 32 + 15) & ~size_t(15); }
    static size_t bytes(uint32_t P, uint32_t kcap, uint32_t pcap) {
        return off_bytes(P) + key_bytes(kcap) + ent_bytes(pcap);
    }
};

// ------------------------------------------------ heavy segments (skew)
// A probe whose segment is longer than kHeavySeg (a heavy key of a skewed
// table, e.g. C3's Zipf ranks: millions of entries under one vertex) would
// keep one warp of one CTA busy for the whole walk while the rest of the GPU
// idles. k_probe_part queues such walks instead as work items of at most
// kHeavyChunk comparisons, and k_heavy_walk runs them on the whole grid:
// one CTA per item, coalesced key loads, one atomic per item.
constexpr uint64_t kHeavySeg = uint64_t(1) << 13;
constexpr uint32_t kHeavyChunk = 1u << 15;

struct HeavyItem {
    uint64_t key;
    uint64_t begin;  // first table entry (global index) of the chunk
    uint64_t pidx;   // probe position (per-probe counts)
    uint32_t len;    // comparisons in the chunk (0: unused slot)
    uint32_t mult;   // probes sharing this (segment, key) walk (count-only; 0 = 1)
};

struct HeavyQueue {
    HeavyItem* items = nullptr;  // nullptr: walk every segment in place
    uint32_t* n = nullptr;
    uint32_t cap = 0;
};

// Warp-collective: queues the segment [gb, gb + len) of probe (key, pidx) as
// chunks and returns true, or returns false (the warp walks it itself) when
// it is short or the queue is full. Slots reserved past a full queue's end
// are never read (k_heavy_walk stops at cap); reserved slots below it are
// always written.
template <typename K>
__device__ __forceinline__ bool defer_heavy(const HeavyQueue& q, K key, uint64_t gb, uint64_t len,
                                            uint64_t pidx, uint32_t mult = 1) {
    if (q.items == nullptr || len <= kHeavySeg) return false;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nch = uint32_t((len + kHeavyChunk - 1) / kHeavyChunk);
    uint32_t slot = 0;
    if (lane == 0) slot = atomicAdd(q.n, nch);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    const bool ok = uint64_t(slot) + nch <= q.cap;
    for (uint32_t c = lane; c < nch && slot + c < q.cap; c += 32) {
        HeavyItem it;
        it.key = uint64_t(key);
        it.begin = gb + uint64_t(c) * kHeavyChunk;
        it.pidx = pidx;
        it.len = ok ? uint32_t(len - uint64_t(c) * kHeavyChunk < kHeavyChunk
                                   ? len - uint64_t(c) * kHeavyChunk : kHeavyChunk)
                    : 0u;
        it.mult = mult;
        q.items[slot + c] = it;
    }
    return ok;
}

constexpr int kHeavyBlock = 512;

// Matches go to totals[0] and, with COUNTS, to counts[pidx] (per-probe
// counts in probe order).
template <typename K, bool COUNTS>
__global__ void __launch_bounds__(kHeavyBlock)
k_heavy_walk(const HeavyItem* __restrict__ items, const uint32_t* __restrict__ n_items, uint32_t cap,
             const K* __restrict__ tkeys, uint64_t* __restrict__ totals,
             uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_w[kHeavyBlock / 32];
    const uint32_t n = *n_items < cap ? *n_items : cap;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        const HeavyItem it = items[i];
        const K key = K(it.key);
        const K* kp = tkeys + it.begin;
        uint32_t c = 0;
        for (uint32_t t = threadIdx.x; t < it.len; t += kHeavyBlock) c += kp[t] == key;
        c = warp_sum(c);
        if (lane == 0) s_w[warp] = c;
        __syncthreads();
        if (warp == 0) {
            uint32_t x = lane < kHeavyBlock / 32 ? s_w[lane] : 0;
            x = warp_sum(x);
            if (lane == 0 && x) {
                if constexpr (COUNTS) atomicAdd(counts + it.pidx, x);
                const unsigned long long mx = (unsigned long long)x * (it.mult ? it.mult : 1u);
                atomicAdd(reinterpret_cast<unsigned long long*>(totals), mx);
            }
        }
        __syncthreads();
    }
}

// MODE 0: totals only; 1: totals + per-probe count at the probe's partitioned
// position (pcount[pos]) or, with ORIG, at its original index; 2: pairs.
// One partition per CTA iteration: thread 0 issues TMA bulk loads of the
// partition's offsets slice, its table-key slice and its probe entries into
// shared memory (one mbarrier), then every probe is answered from shared
// memory. Slices larger than the caps are read from global memory instead.
template <typename K, typename VT, typename OffT, typename IT, int POW2, int MODE, bool ORIG,
          typename PT>
__global__ void __launch_bounds__(kPartProbeBlock, (MODE == 2 ? 2 : 3))
k_probe_part(const typename EntryT<K, IT>::T* __restrict__ pin, const OffT* __restrict__ ppart,
             uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
             uint32_t pshift, const OffT* __restrict__ offs, const K* __restrict__ tkeys,
             const VT* __restrict__ tvals, uint32_t kcap, uint32_t pcap,
             uint32_t* __restrict__ pcount, const uint64_t* __restrict__ pair_off,
             void* __restrict__ pairs, uint64_t cap, uint64_t* __restrict__ totals,
             uint32_t* ticket, HeavyQueue heavy, uint64_t in_cap,
             const uint32_t* __restrict__ slack_flag) {
    // probe entries of partition p: slack layout (p * in_cap) of
    // partition_slack unless it overflowed, else dense (ppart[p])
    const bool slack_in = in_cap && !*slack_flag;
    using PE = EntryT<K, IT>;
    using PEnt = typename PE::T;
    using L = ProbeLayout<K, OffT, PEnt>;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t P = 1u << pshift;
    unsigned char* const b_off = smem;
    unsigned char* const b_key = smem + L::off_bytes(P);
    unsigned char* const b_ent = b_key + L::key_bytes(kcap);
    __shared__ uint64_t s_bar;
    __shared__ uint64_t s_p, s_tb, s_te, s_q0, s_q1, s_qin;
    __shared__ uint32_t s_o0, s_o1, s_o2, s_kst, s_pst;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t nwarps = kPartProbeBlock / 32;
    // count-only: the partition's heavy (segment, key) walks, deduplicated --
    // every probe of a key gets the same count, so each distinct key's heavy
    // segment is queued once with its probe multiplicity (C3: the 16 probes
    // of a Zipf rank no longer re-read its segment 16 times). Full table:
    // queued per probe as before. Compiled for u64-key tables only: on the
    // u32 C2 probe the partition-end flush barrier alone cost k8p 2.4 %.
    constexpr bool kDedupOn = MODE == 0 && sizeof(K) == 8;
    constexpr uint32_t kDedup = kDedupOn ? 64 : 1;
    __shared__ uint64_t s_dk[kDedup];
    __shared__ uint32_t s_db[kDedup], s_dl[kDedup], s_dm[kDedup], s_dv[kDedup];
    __shared__ uint32_t s_dn;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        s_dn = 0;
    }
    if (tid < kDedup) s_dv[tid] = 0;
    uint32_t phase = 0;
    uint64_t matches = 0, compared = 0;
    // (thread 0) partitions are claimed two ahead and their bounds loaded one
    // ahead, so the ticket atomic and the dependent bound loads overlap the
    // previous partition's probes instead of sitting in front of the block
    // barrier (k8p's top stall)
    uint32_t p_cur = 0, p_nxt = 0;
    OffT m_tb = 0, m_te = 0, m_q0 = 0, m_q1 = 0;
    auto bounds = [&](uint32_t q) {
        if (q < nparts) {
            const uint64_t vb = uint64_t(q) << pshift;
            const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
            m_tb = offs[vb];
            m_te = offs[vb + pv];
            m_q0 = ppart[q];
            m_q1 = ppart[q + 1];
        }
    };
    // (count-only; the per-probe-count / pair modes keep their registers)
    constexpr bool kAhead = MODE == 0;
    if (kAhead && tid == 0) {
        p_cur = atomicAdd(ticket, 1u);
        p_nxt = atomicAdd(ticket, 1u);
        bounds(p_cur);
    }
    while (true) {
        if (tid == 0) {
            uint64_t p, tb = 0, te = 0, q0 = 0, q1 = 0;
            if constexpr (kAhead) {
                p = p_cur;
                tb = m_tb, te = m_te, q0 = m_q0, q1 = m_q1;
                p_cur = p_nxt;
                bounds(p_cur);
                if (p_nxt < nparts) p_nxt = atomicAdd(ticket, 1u);
            } else {
                p = atomicAdd(ticket, 1u);
                if (p < nparts) {
                    const uint64_t vb = p << pshift;
                    const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
                    tb = offs[vb];
                    te = offs[vb + pv];
                    q0 = ppart[p];
                    q1 = ppart[p + 1];
                }
            }
            s_p = p;
            if (p < nparts) {
                const uint64_t vb = p << pshift;
                const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
                const uint64_t qin = slack_in ? p * in_cap : q0;
                s_tb = tb; s_te = te; s_q0 = q0; s_q1 = q1; s_qin = qin;
                s_kst = te - tb <= kcap;
                s_pst = q1 - q0 <= pcap;
                fence_proxy_async();
                // three spans, one transaction barrier
                const uintptr_t ao = reinterpret_cast<uintptr_t>(offs + vb);
                const uintptr_t ak = reinterpret_cast<uintptr_t>(tkeys + tb);
                const uintptr_t ae = reinterpret_cast<uintptr_t>(pin + qin);
                auto span = [](uintptr_t a, size_t bytes, uint32_t& lo_off) -> uint32_t {
                    const uintptr_t lo = a & ~uintptr_t(15), hi = (a + bytes + 15) & ~uintptr_t(15);
                    lo_off = uint32_t(a - lo);
                    return uint32_t(hi - lo);
                };
                uint32_t o0, o1 = 0, o2 = 0;
                const uint32_t l0 = span(ao, size_t(pv + 1) * sizeof(OffT), o0);
                const uint32_t l1 = s_kst ? span(ak, size_t(te - tb) * sizeof(K), o1) : 0;
                const uint32_t l2 = s_pst ? span(ae, size_t(q1 - q0) * sizeof(PEnt), o2) : 0;
                s_o0 = o0; s_o1 = o1; s_o2 = o2;
                mbar_arrive_expect_tx(&s_bar, l0 + l1 + l2);
                tma_load_1d(b_off, reinterpret_cast<const void*>(ao - o0), l0, &s_bar);
                if (l1) tma_load_1d(b_key, reinterpret_cast<const void*>(ak - o1), l1, &s_bar);
                if (l2) tma_load_1d(b_ent, reinterpret_cast<const void*>(ae - o2), l2, &s_bar);
            }
        }
        __syncthreads();
        const uint64_t p = s_p;
        if (p >= nparts) break;
        const uint64_t vb = p << pshift;
        const uint64_t tb = s_tb;
        const uint64_t q0 = s_q0, qn = s_q1 - s_q0;
        const OffT* soff = reinterpret_cast<const OffT*>(b_off + s_o0);
        mbar_wait(&s_bar, phase);
        phase ^= 1;
        // Probe loop, instantiated for the common case (slices staged in
        // shared memory: LDS on 32-bit addresses) and for oversized slices
        // (generic loads from global memory).
        auto run = [&](const K* __restrict__ kp, const PEnt* __restrict__ ep) {
            if constexpr (MODE == 0) {
                // count-only (the C2 step): partition-relative indices in the
                // offsets' width (u32 at C2), fewer 64-bit address updates
                using I = OffT;
                const I qi = I(qn), tbi = I(tb);
                // whole-warp rounds run without the bounds check (no divergent
                // region per probe); the last, partial round checks
                auto round = [&](I base, auto chk) {
                    const I i = base + I(lane);
                    K key = 0;
                    I b = 0, e = 0;
                    if (!decltype(chk)::value || i < qi) {
                        key = PE::key(ep[i]);
                        const uint32_t lv = uint32_t(hv<POW2>(key, seed, hk, nv) - vb);
                        b = I(soff[lv]) - tbi;
                        e = I(soff[lv + 1]) - tbi;
                    }
                    const I len = e - b;
                    compared += len;
                    uint32_t c = 0;
                    if (len <= I(kLongSeg)) c = seg_count(kp + b, uint64_t(len), key);
                    uint32_t longm = __ballot_sync(0xffffffffu, len > I(kLongSeg));
                    while (longm) {
                        const int src = __ffs(longm) - 1;
                        longm &= longm - 1;
                        const I kb = __shfl_sync(0xffffffffu, b, src);
                        const I ke = __shfl_sync(0xffffffffu, e, src);
                        const K kk = __shfl_sync(0xffffffffu, key, src);
                        if (kDedupOn && heavy.items && uint64_t(ke - kb) > kHeavySeg && uint64_t(ke) < (uint64_t(1) << 32)) {
                            // known key: one more probe on its walk
                            const uint32_t dn = min(*reinterpret_cast<volatile uint32_t*>(&s_dn), kDedup);
                            uint32_t hit = 0;
                            for (uint32_t j0 = 0; j0 < dn && !hit; j0 += 32) {
                                const uint32_t j = j0 + lane;
                                const bool m = j < dn && reinterpret_cast<volatile uint32_t*>(s_dv)[j] &&
                                               reinterpret_cast<volatile uint64_t*>(s_dk)[j] == uint64_t(kk);
                                hit = __ballot_sync(0xffffffffu, m);
                                if (hit && lane == uint32_t(__ffs(hit) - 1)) atomicAdd(&s_dm[j], 1u);
                            }
                            if (hit) continue;
                            uint32_t slot = 0;
                            if (lane == 0) slot = atomicAdd(&s_dn, 1u);
                            slot = __shfl_sync(0xffffffffu, slot, 0);
                            if (slot < kDedup) {
                                if (lane == 0) {
                                    s_dk[slot] = uint64_t(kk);
                                    s_db[slot] = uint32_t(kb);
                                    s_dl[slot] = uint32_t(ke - kb);
                                    s_dm[slot] = 1;
                                    __threadfence_block();
                                    reinterpret_cast<volatile uint32_t*>(s_dv)[slot] = 1;
                                }
                                continue;
                            }
                        }
                        if (defer_heavy(heavy, kk, tb + uint64_t(kb), uint64_t(ke - kb), 0)) continue;
                        uint32_t cc = 0;
                        for (I t = kb + I(lane); t < ke; t += 32) cc += kp[t] == kk;
                        cc = warp_sum(cc);
                        if (int(lane) == src) c = cc;
                    }
                    matches += c;
                };
                I base = I(warp) * 32;
                for (; base + 32 <= qi; base += I(nwarps) * 32) round(base, std::false_type{});
                if (base < qi) round(base, std::true_type{});
                if (kDedupOn && heavy.items) {
                    // queue the partition's deduplicated heavy walks (warp 0)
                    __syncthreads();
                    if (warp == 0) {
                        const uint32_t dn = min(s_dn, kDedup);
                        for (uint32_t j = 0; j < dn; ++j) {
                            const K kk = K(s_dk[j]);
                            const I kb = I(s_db[j]), ke = kb + I(s_dl[j]);
                            const uint32_t mult = s_dm[j];
                            if (defer_heavy(heavy, kk, tb + uint64_t(kb), uint64_t(ke - kb), 0, mult)) continue;
                            uint32_t cc = 0;  // queue full: walk here
                            for (I t = kb + I(lane); t < ke; t += 32) cc += kp[t] == kk;
                            cc = warp_sum(cc);
                            if (lane == 0) matches += uint64_t(cc) * mult;
                        }
                        if (lane == 0) s_dn = 0;
                        for (uint32_t j = lane; j < kDedup; j += 32) s_dv[j] = 0;
                    }
                }
            } else {
                for (uint64_t base = uint64_t(warp) * 32; base < qn; base += uint64_t(nwarps) * 32) {
                    const uint64_t i = base + lane;
                    const bool valid = i < qn;
                    K key = 0;
                    typename std::conditional<std::is_void<IT>::value, uint32_t, IT>::type pidx = 0;
                    uint64_t b = 0, e = 0;
                    if (valid) {
                        const auto ent = ep[i];
                        key = PE::key(ent);
                        if constexpr (PE::kHasVal) pidx = PE::val(ent);
                        const uint32_t lv = uint32_t(hv<POW2>(key, seed, hk, nv) - vb);
                        b = uint64_t(soff[lv]) - tb;
                        e = uint64_t(soff[lv + 1]) - tb;
                    }
                    const uint64_t len = e - b;
                    compared += len;
                    uint32_t c = 0;
                    if (len <= kLongSeg) c = seg_count(kp + b, len, key);
                    uint32_t longm = __ballot_sync(0xffffffffu, len > kLongSeg);
                    while (longm) {
                        const int src = __ffs(longm) - 1;
                        longm &= longm - 1;
                        const uint64_t kb = __shfl_sync(0xffffffffu, b, src);
                        const uint64_t ke = __shfl_sync(0xffffffffu, e, src);
                        const K kk = __shfl_sync(0xffffffffu, key, src);
                        if constexpr (MODE == 1 && ORIG) {
                            // the deferred walk adds to counts[pidx] (and the totals below)
                            if (defer_heavy(heavy, kk, tb + kb, ke - kb,
                                            uint64_t(__shfl_sync(0xffffffffu, pidx, src))))
                                continue;
                        }
                        uint32_t cc = 0;
                        for (uint64_t t = kb + lane; t < ke; t += 32) cc += kp[t] == kk;
                        cc = warp_sum(cc);
                        if (int(lane) == src) c = cc;
                    }
                    matches += c;
                    if constexpr (MODE == 1) {
                        if (valid) {
                            if constexpr (ORIG) pcount[pidx] = c;
                            else pcount[q0 + i] = c;
                        }
                    }
                    if constexpr (MODE == 2) {
                        uint64_t sl = (valid && c) ? pair_off[q0 + i] : 0;
                        if (valid && c && len <= kLongSeg) {
                            for (uint64_t t = b; t < e && sl < cap; ++t) {
                                if (kp[t] == key) {
                                    store_pair<PT>(pairs, sl, uint64_t(tvals[tb + t]), uint64_t(pidx));
                                    ++sl;
                                }
                            }
                        }
                        uint32_t lm = __ballot_sync(0xffffffffu, valid && c && len > kLongSeg);
                        while (lm) {
                            const int src = __ffs(lm) - 1;
                            lm &= lm - 1;
                            const uint64_t kb = __shfl_sync(0xffffffffu, b, src);
                            const uint64_t ke = __shfl_sync(0xffffffffu, e, src);
                            const K kk = __shfl_sync(0xffffffffu, key, src);
                            uint64_t ws = __shfl_sync(0xffffffffu, sl, src);
                            const uint64_t pj = __shfl_sync(0xffffffffu, uint64_t(pidx), src);
                            for (uint64_t t0 = kb; t0 < ke && ws < cap; t0 += 32) {
                                const uint64_t t = t0 + lane;
                                const bool hit = t < ke && kp[t] == kk;
                                const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                                const uint64_t my = ws + __popc(hm & lanemask_lt());
                                if (hit && my < cap) store_pair<PT>(pairs, my, uint64_t(tvals[tb + t]), pj);
                                ws += __popc(hm);
                            }
                        }
                    }
                }
            }
        };
        if (s_kst && s_pst) {
            run(reinterpret_cast<const K*>(b_key + s_o1), reinterpret_cast<const PEnt*>(b_ent + s_o2));
        } else {
            run(s_kst ? reinterpret_cast<const K*>(b_key + s_o1) : tkeys + tb,
                s_pst ? reinterpret_cast<const PEnt*>(b_ent + s_o2) : pin + s_qin);
        }
        __syncthreads();
    }
    __shared__ unsigned long long s_m[nwarps], s_c[nwarps];
    matches = warp_sum(matches);
    compared = warp_sum(compared);
    if (lane == 0) {
        s_m[warp] = matches;
        s_c[warp] = compared;
    }
    __syncthreads();
    if (tid < 32) {
        unsigned long long x = tid < nwarps ? s_m[tid] : 0, y = tid < nwarps ? s_c[tid] : 0;
        x = warp_sum(x);
        y = warp_sum(y);
        if (tid == 0 && MODE != 2) {
            if (x) atomicAdd(reinterpret_cast<unsigned long long*>(totals), x);
            if (y) atomicAdd(reinterpret_cast<unsigned long long*>(totals + 1), y);
        }
    }
}

// ------------------------------------------------ single-pass pairs (K10p)
// Pairs without per-probe count arrays or a global scan: partitions are taken
// in ticket order; per partition (staged in shared memory as in
// k_probe_part) the CTA
//   A  counts the matches of every probe, keeping per-(chunk, warp) totals
//      (chunk = 512 consecutive probes) for the first kPairRound chunks,
//   -  publishes the partition total with a decoupled look-back over
//      partitions (hg_scan.cuh status words) -> the partition's first slot,
//   B  scans the (chunk, warp) totals and writes every probe's pairs at
//      slot = base + (chunk, warp) prefix + warp-exclusive count.
// HBM traffic = the count-only probe's + the pairs themselves. Pair order:
// partition, then probe within the partition, then table segment order (the
// reference's order is unspecified too, join.hpp:71-74).
constexpr uint32_t kPairRound = 24;  // chunks per scan round (24 * 512 = 12288 probes)

// Per-lane match count of probe `i` of the partition (valid < qn), with
// warp-cooperative walks of long segments; warp-collective. Positions are
// partition-relative in the offsets' width (u32 at C2/C4), probe indices in J.
template <typename K, typename OffT, typename PEnt, typename PE, int POW2, typename J>
__device__ __forceinline__ uint32_t pair_count(const K* __restrict__ kp, const PEnt& ent,
                                               const OffT* soff, J i, J qn, OffT tb,
                                               uint64_t vb, uint64_t seed, int hk, const Divisor& nv,
                                               uint64_t& compared, K& key, OffT& b, OffT& e,
                                               uint32_t& pos) {
    using I = OffT;
    const uint32_t lane = threadIdx.x & 31;
    I bi = 0, ei = 0;
    key = 0;
    if (i < qn) {
        key = PE::key(ent);
        const uint32_t lv = uint32_t(hv<POW2>(key, seed, hk, nv) - vb);
        bi = I(soff[lv]) - tb;
        ei = I(soff[lv + 1]) - tb;
    }
    const I len = ei - bi;
    compared += len;
    uint32_t c = 0;
    pos = 0;
    if (len <= I(kLongSeg)) c = seg_count_pos(kp + bi, uint64_t(len), key, pos);
    uint32_t longm = __ballot_sync(0xffffffffu, len > I(kLongSeg));
    while (longm) {
        const int src = __ffs(longm) - 1;
        longm &= longm - 1;
        const I kb = __shfl_sync(0xffffffffu, bi, src);
        const I ke = __shfl_sync(0xffffffffu, ei, src);
        const K kk = __shfl_sync(0xffffffffu, key, src);
        uint32_t cc = 0;
        for (I t = kb + I(lane); t < ke; t += 32) cc += kp[t] == kk;
        cc = warp_sum(cc);
        if (int(lane) == src) c = cc;
    }
    b = bi;
    e = ei;
    return c;
}

// Inclusive warp prefix of per-lane counts; one ballot when every count is
// 0 or 1 (unique build keys: C4), else the shuffle scan.
__device__ __forceinline__ uint32_t warp_incl_count(uint32_t c) {
    if (__all_sync(0xffffffffu, c <= 1u)) return __popc(__ballot_sync(0xffffffffu, c != 0) & lanemask_lt()) + c;
    return warp_inclusive_sum(c);
}

constexpr uint32_t kNeedWalk = 0xFFFFFFFFu;

// Shared bytes of the single-pass pairs kernel's staged table-value slice.
template <typename VT>
__host__ __device__ constexpr size_t pair_val_bytes(uint32_t kcap) {
    return (size_t(kcap) * sizeof(VT) + 32 + 15) & ~size_t(15);
}

// Pass-A summary of one probe for pass B: 0 (no match), (t << 16) | 1 (one
// match at tile key t = b + pos, short segment, t < 2^16) or kNeedWalk.
template <typename I>
__device__ __forceinline__ uint32_t pair_info(I b, I e, uint32_t c, uint32_t pos) {
    if (c == 0) return 0u;
    if (c != 1 || e - b > I(kLongSeg) || e > I(0xFFFFu)) return kNeedWalk;
    return (uint32_t(b + pos) << 16) | 1u;
}

template <typename K, typename VT, typename OffT, typename IT, int POW2, typename PT, typename PJ>
__global__ void __launch_bounds__(kPartProbeBlock)
k_probe_pairs(const typename EntryT<K, IT>::T* __restrict__ pin, const OffT* __restrict__ ppart,
              uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
              uint32_t pshift, const OffT* __restrict__ offs, const K* __restrict__ tkeys,
              const VT* __restrict__ tvals, uint32_t kcap, uint32_t pcap, uint64_t* __restrict__ status,
              void* __restrict__ pairs, uint64_t cap, uint64_t* __restrict__ totals,
              uint32_t* ticket, uint64_t in_cap, const uint32_t* __restrict__ slack_flag) {
    // probe entries of partition p: slack layout (p * in_cap) unless it
    // overflowed, else dense (ppart[p]); pairs carry probe positions, so only
    // the reads move
    const bool slack_in = in_cap && !*slack_flag;
    using PE = EntryT<K, IT>;
    using PEnt = typename PE::T;
    using L = ProbeLayout<K, OffT, PEnt>;
    constexpr uint32_t nwarps = kPartProbeBlock / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t P = 1u << pshift;
    unsigned char* const b_off = smem;
    unsigned char* const b_key = smem + L::off_bytes(P);
    unsigned char* const b_ent = b_key + L::key_bytes(kcap);
    // the partition's table values (build entry indices of the pairs) are
    // staged next to its keys: the pair writes read them from shared memory
    // instead of one random L2 gather per pair
    unsigned char* const b_val = b_ent + L::ent_bytes(pcap);
    // per-probe result of pass A for the current round: 0 = no match,
    // (t << 16) | 1 = exactly one match at tile key t, kNeedWalk = walk again
    uint32_t* const s_info = reinterpret_cast<uint32_t*>(b_val + pair_val_bytes<VT>(kcap));
    __shared__ uint64_t s_bar;
    __shared__ uint64_t s_p, s_tb, s_q0, s_q1, s_base;
    __shared__ uint32_t s_o0, s_o1, s_o2, s_o3, s_kst, s_pst;
    __shared__ uint64_t s_wt[kPairRound * nwarps];
    __shared__ uint64_t s_red[nwarps];
    __shared__ uint64_t s_rt;  // a round's pair total
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
    }
    uint32_t phase = 0;
    uint64_t matches = 0, compared = 0;
    while (true) {
        if (tid == 0) {
            const uint64_t p = atomicAdd(ticket, 1u);
            s_p = p;
            if (p < nparts) {
                const uint64_t vb = p << pshift;
                const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
                const uint64_t tb = offs[vb], te = offs[vb + pv];
                const uint64_t q0 = ppart[p], q1 = ppart[p + 1];
                s_tb = tb;
                s_q0 = slack_in ? p * in_cap : q0;  // input start
                s_q1 = s_q0 + (q1 - q0);
                s_kst = te - tb <= kcap;
                s_pst = pcap && q1 - q0 <= pcap;
                fence_proxy_async();
                const uintptr_t ao = reinterpret_cast<uintptr_t>(offs + vb);
                const uintptr_t ak = reinterpret_cast<uintptr_t>(tkeys + tb);
                const uintptr_t ae = reinterpret_cast<uintptr_t>(pin + s_q0);
                auto span = [](uintptr_t a, size_t bytes, uint32_t& lo_off) -> uint32_t {
                    const uintptr_t lo = a & ~uintptr_t(15), hi = (a + bytes + 15) & ~uintptr_t(15);
                    lo_off = uint32_t(a - lo);
                    return uint32_t(hi - lo);
                };
                const uintptr_t av = reinterpret_cast<uintptr_t>(tvals + tb);
                uint32_t o0, o1 = 0, o2 = 0, o3 = 0;
                const uint32_t l0 = span(ao, size_t(pv + 1) * sizeof(OffT), o0);
                const uint32_t l1 = s_kst ? span(ak, size_t(te - tb) * sizeof(K), o1) : 0;
                const uint32_t l2 = s_pst ? span(ae, size_t(q1 - q0) * sizeof(PEnt), o2) : 0;
                const uint32_t l3 = s_kst ? span(av, size_t(te - tb) * sizeof(VT), o3) : 0;
                s_o0 = o0;
                s_o1 = o1;
                s_o2 = o2;
                s_o3 = o3;
                mbar_arrive_expect_tx(&s_bar, l0 + l1 + l2 + l3);
                tma_load_1d(b_off, reinterpret_cast<const void*>(ao - o0), l0, &s_bar);
                if (l1) tma_load_1d(b_key, reinterpret_cast<const void*>(ak - o1), l1, &s_bar);
                if (l2) tma_load_1d(b_ent, reinterpret_cast<const void*>(ae - o2), l2, &s_bar);
                if (l3) tma_load_1d(b_val, reinterpret_cast<const void*>(av - o3), l3, &s_bar);
            }
        }
        __syncthreads();
        const uint64_t p = s_p;
        if (p >= nparts) break;
        const uint64_t vb = p << pshift;
        const uint64_t tb = s_tb;
        const uint64_t q0 = s_q0, qn = s_q1 - s_q0;
        const OffT* soff = reinterpret_cast<const OffT*>(b_off + s_o0);
        mbar_wait(&s_bar, phase);
        phase ^= 1;
        const VT* __restrict__ vp =
            s_kst ? reinterpret_cast<const VT*>(b_val + s_o3) : tvals + tb;  // partition's values
        // J = PJ: probe index type (u32 unless the probe set has >= 2^31 probes)
        auto run = [&](const K* __restrict__ kp, const PEnt* __restrict__ ep, auto jt) {
            using J = decltype(jt);
            using I = OffT;
            // (one warp) exclusive scan of a round's (chunk, warp) totals in
            // (chunk, warp) order, relative to the round's base; s_rt = total
            auto scan_round = [&]() {
                constexpr uint32_t per = kPairRound * nwarps / 32;
                uint64_t x[per];
                uint64_t sum = 0;
#pragma unroll
                for (uint32_t k = 0; k < per; ++k) sum += (x[k] = s_wt[lane * per + k]);
                const uint64_t inc = warp_inclusive_sum(sum);
                uint64_t run_ = inc - sum;
#pragma unroll
                for (uint32_t k = 0; k < per; ++k) {
                    s_wt[lane * per + k] = run_;
                    run_ += x[k];
                }
                if (lane == 31) s_rt = inc;
            };
            const I tbi = I(tb);
            const J qj = J(qn);
            // A: counts; (chunk, warp) totals of the first round
            uint64_t mine = 0;
            const J nchunks = (qj + J(kPartProbeBlock) - 1) / J(kPartProbeBlock);
            const J i0 = J(warp * 32 + lane);
            PEnt nxt = i0 < qj ? ep[i0] : PEnt{};
            for (J ch = 0; ch < nchunks; ++ch) {
                K key;
                I b, e;
                const J i = ch * J(kPartProbeBlock) + i0;
                const PEnt cur = nxt;  // entries are prefetched one chunk ahead
                if (i + J(kPartProbeBlock) < qj) nxt = ep[i + J(kPartProbeBlock)];
                uint32_t pos;
                const uint32_t c = pair_count<K, OffT, PEnt, PE, POW2, J>(kp, cur, soff, i, qj, tbi, vb, seed,
                                                                           hk, nv, compared, key, b, e, pos);
                const uint32_t cw = warp_sum(c);
                if (ch < J(kPairRound)) {
                    if (lane == 0) s_wt[uint32_t(ch) * nwarps + warp] = cw;
                    s_info[uint32_t(ch) * kPartProbeBlock + uint32_t(i0)] = pair_info(b, e, c, pos);
                }
                mine += cw;
            }
            if (lane == 0) s_red[warp] = mine;
            __syncthreads();
            if (warp == 0) {
                uint64_t tot = lane < nwarps ? s_red[lane] : 0;
                tot = warp_sum(tot);
                uint64_t prefix = 0;
                if (p == 0) {
                    if (lane == 0) st_relaxed_u64(status, kScanFlagIncl | tot);
                } else {
                    if (lane == 0) st_relaxed_u64(status + p, kScanFlagAgg | tot);
                    int64_t idx = int64_t(p) - 1;
                    while (true) {
                        const int64_t jj = idx - int64_t(lane);
                        uint64_t sw = kScanFlagIncl;
                        if (jj >= 0) {
                            do {
                                sw = ld_relaxed_u64(status + jj);
                            } while ((sw >> 62) == 0);
                        }
                        const uint32_t inclm = __ballot_sync(0xffffffffu, (sw >> 62) == 2);
                        const uint32_t stop = inclm ? uint32_t(__ffs(inclm) - 1) : 32u;
                        prefix += warp_sum(lane <= stop ? (sw & kScanValMask) : uint64_t(0));
                        if (inclm) break;
                        idx -= 32;
                    }
                    if (lane == 0) st_relaxed_u64(status + p, kScanFlagIncl | (prefix + tot));
                }
                if (lane == 0) {
                    s_base = prefix;
                    matches += tot;
                }
            } else if (warp == 1) {
                scan_round();  // round 0, overlapping warp 0's look-back
            }
            __syncthreads();
            uint64_t base = s_base;
            // B: rounds of kPairRound chunks
            for (J r0 = 0; r0 < nchunks && base < cap; r0 += J(kPairRound)) {
                const J r1 = r0 + J(kPairRound) < nchunks ? r0 + J(kPairRound) : nchunks;
                if (r0 > 0) {
                    __syncthreads();
                    for (J ch = r0; ch < r1; ++ch) {
                        K key;
                        I b, e;
                        uint64_t dummy = 0;
                        const J i = ch * J(kPartProbeBlock) + i0;
                        const PEnt cur = i < qj ? ep[i] : PEnt{};
                        uint32_t pos;
                        const uint32_t c = pair_count<K, OffT, PEnt, PE, POW2, J>(
                            kp, cur, soff, i, qj, tbi, vb, seed, hk, nv, dummy, key, b, e, pos);
                        const uint32_t cw = warp_sum(c);
                        if (lane == 0) s_wt[uint32_t(ch - r0) * nwarps + warp] = cw;
                        s_info[uint32_t(ch - r0) * kPartProbeBlock + uint32_t(i0)] = pair_info(b, e, c, pos);
                    }
                    __syncthreads();
                    if (warp == 0) scan_round();
                    __syncthreads();
                }
                const uint64_t round_total = s_rt;
                const J ib = r0 * J(kPartProbeBlock) + i0;
                PEnt nxtb = ib < qj ? ep[ib] : PEnt{};
                const uint64_t* wt = s_wt + warp;
                const uint32_t* inf = s_info + uint32_t(i0);
                for (J ch = r0; ch < r1; ++ch, wt += nwarps, inf += kPartProbeBlock) {
                    K key = 0;
                    I b = 0, e = 0;
                    uint64_t dummy = 0;
                    const J i = ch * J(kPartProbeBlock) + i0;
                    const PEnt cur = nxtb;
                    if (ch + 1 < r1 && i + J(kPartProbeBlock) < qj) nxtb = ep[i + J(kPartProbeBlock)];
                    const uint32_t info = i < qj ? *inf : 0u;
                    const bool walk = info == kNeedWalk;
                    uint32_t c = info & 1u;
                    if (__any_sync(0xffffffffu, walk)) {
                        // duplicates / long segments: count again (warp-collective)
                        uint32_t pos;
                        const uint32_t cc = pair_count<K, OffT, PEnt, PE, POW2, J>(
                            kp, cur, soff, i, qj, tbi, vb, seed, hk, nv, dummy, key, b, e, pos);
                        if (walk) c = cc;
                    }
                    if (!walk) b = e = 0;
                    const uint32_t incl = warp_incl_count(c);
                    uint64_t sl = base + *wt + (incl - c);
                    const I len = e - b;
                    const uint64_t pidx = PE::kHasVal && i < qj ? uint64_t(PE::val(cur)) : 0;
                    if (!walk && c == 1) {
                        // one match at a known tile key: one value gather + store
                        if (sl < cap) store_pair<PT>(pairs, sl, uint64_t(vp[info >> 16]), pidx);
                    } else if (c && len <= I(kLongSeg)) {
                        for (I t = b; t < e && sl < cap; ++t) {
                            if (kp[t] == key) {
                                store_pair<PT>(pairs, sl, uint64_t(vp[t]), pidx);
                                ++sl;
                            }
                        }
                    }
                    uint32_t lm = __ballot_sync(0xffffffffu, c && len > I(kLongSeg));
                    while (lm) {
                        const int src = __ffs(lm) - 1;
                        lm &= lm - 1;
                        const I kb = __shfl_sync(0xffffffffu, b, src);
                        const I ke = __shfl_sync(0xffffffffu, e, src);
                        const K kk = __shfl_sync(0xffffffffu, key, src);
                        uint64_t ws = __shfl_sync(0xffffffffu, sl, src);
                        const uint64_t pj = __shfl_sync(0xffffffffu, pidx, src);
                        for (I t0 = kb; t0 < ke && ws < cap; t0 += 32) {
                            const I t = t0 + I(lane);
                            const bool hit = t < ke && kp[t] == kk;
                            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                            const uint64_t my = ws + __popc(hm & lanemask_lt());
                            if (hit && my < cap) store_pair<PT>(pairs, my, uint64_t(vp[t]), pj);
                            ws += __popc(hm);
                        }
                    }
                }
                base += round_total;
            }
        };
        auto run_j = [&](const K* __restrict__ kp, const PEnt* __restrict__ ep) {
            run(kp, ep, PJ(0));
        };
        if (s_kst && s_pst) {
            run_j(reinterpret_cast<const K*>(b_key + s_o1), reinterpret_cast<const PEnt*>(b_ent + s_o2));
        } else {
            run_j(s_kst ? reinterpret_cast<const K*>(b_key + s_o1) : tkeys + tb,
                s_pst ? reinterpret_cast<const PEnt*>(b_ent + s_o2) : pin + q0);
        }
        __syncthreads();
    }
    // totals: matches accumulated by warp 0 lane 0; comparisons by everyone
    compared = warp_sum(compared);
    if (lane == 0) s_red[warp] = compared;
    __syncthreads();
    if (tid < 32) {
        unsigned long long y = tid < nwarps ? s_red[tid] : 0;
        y = warp_sum(y);
        if (tid == 0) {
            if (matches) atomicAdd(reinterpret_cast<unsigned long long*>(totals), matches);
            if (y) atomicAdd(reinterpret_cast<unsigned long long*>(totals + 1), y);
        }
    }
}

template <typename K, typename IT>
__global__ void k_scatter_counts(const typename EntryT<K, IT>::T* __restrict__ pin,
                                 const uint32_t* __restrict__ pcount, uint64_t m,
                                 uint32_t* __restrict__ counts) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
        counts[EntryT<K, IT>::val(pin[i])] = pcount[i];
}

template <typename K, typename VT, typename OffT, typename IT, int POW2>
static cudaError_t probe_partitioned(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    const Divisor nv = make_divisor(global_nv(t), t.vbase);
    const OffT* offs = static_cast<const OffT*>(t.offs);
    const K* tkeys = static_cast<const K*>(t.keys);
    const VT* tvals = static_cast<const VT*>(t.vals);
    const K* probes = static_cast<const K*>(a.probes);
    constexpr uint32_t kTarget = 4096;
    const PartGeom g = make_geom(t.nv, t.n, 0, double(kTarget));
    const uint32_t P = 1u << g.pshift;
    // table-key cap from the table's keys per partition, probe cap from the
    // probes' expected count per partition (both ~1.5x the mean)
    const double kmean = double(t.n) * double(P) / double(t.nv);
    const double pmean = double(a.m) * double(P) / double(t.nv);
    uint32_t kcap = uint32_t(std::min(12288.0, std::max(512.0, 1.5 * kmean + 256)));
    uint32_t pcap = uint32_t(std::min(12288.0, std::max(512.0, 1.5 * pmean + 256)));
    const bool want_counts = a.counts != nullptr && a.counts_requested;
    const bool need_idx = want_counts || a.pairs != nullptr;
    // shrink the staged caps until every layout this call may launch fits one
    // CTA (partitions above a cap are read from global memory instead)
    {
        using E1L = ProbeLayout<K, OffT, typename EntryT<K, IT>::T>;
        const size_t optin = smem_optin() - 8192;  // static shared memory of the kernels
        const size_t round = size_t(kPairRound) * kPartProbeBlock * sizeof(uint32_t);
        while (E1L::bytes(P, kcap, pcap) > optin && (kcap > 512 || pcap > 512)) {
            if (pcap > 512 && pcap >= kcap) pcap -= pcap / 4;
            else kcap -= kcap / 4;
        }
        while (E1L::bytes(P, kcap, 0) + round > optin && kcap > 512) kcap -= kcap / 4;
    }
    // single-pass pairs kernel: keys AND values of the partition staged, two
    // CTAs per SM -> a tighter key cap (mean + 6 sigma of a Poisson count)
    uint32_t kcap_pairs = uint32_t(std::min<double>(kcap, std::max(512.0, kmean + 6.0 * std::sqrt(kmean) + 64)));
    {
        using E1L = ProbeLayout<K, OffT, typename EntryT<K, IT>::T>;
        const size_t optin = smem_optin() - 8192;
        const size_t round = size_t(kPairRound) * kPartProbeBlock * sizeof(uint32_t);
        while (E1L::bytes(P, kcap_pairs, 0) + pair_val_bytes<VT>(kcap_pairs) + round > optin &&
               kcap_pairs > 512)
            kcap_pairs -= kcap_pairs / 4;
    }
    const int sms = num_sms();
    cudaError_t e;
    char* scratch = nullptr;
    const size_t ps_bytes = ((g.nparts + 1) * sizeof(OffT) + 255) & ~size_t(255);
    using E1 = typename EntryT<K, IT>::T;
    using E0 = typename EntryT<K, void>::T;
    const size_t ent = need_idx ? sizeof(E1) : sizeof(E0);
    const bool single = a.pairs && !want_counts && a.cap > 0;  // k_probe_pairs
    // slack (histogram-free) partition layout when it fits (partition_slack in
    // hg_radix.cuh; the flag word is ticket + 2): count-only probes, per-probe
    // counts in probe order and the single-pass pairs read their partitions
    // through it; the two-pass pairs address per-probe arrays by partitioned
    // position and keep the dense layout
    const bool slack_ok = !need_idx || (want_counts && !a.pairs) || single;
    const Slack sl_caps = slack_ok ? make_slack<OffT>(g, a.m, t.nv, nullptr) : Slack{};
    const uint64_t nb1 = (g.nparts + (uint64_t(1) << g.b2) - 1) >> g.b2;
    const size_t pscr = need_idx ? PartitionScratch<K, IT, OffT>::bytes(g, a.m, nb1 * sl_caps.cap1)
                                 : PartitionScratch<K, void, OffT>::bytes(g, a.m, nb1 * sl_caps.cap1);
    const size_t reorg_bytes =
        (std::max<uint64_t>(a.m, g.nparts * sl_caps.cap2) * ent + 255) & ~size_t(255);
    const size_t cnt_bytes = (a.pairs && !single) ? ((a.m * 4 + 255) & ~size_t(255)) : 0;
    const size_t po_bytes = single ? ((g.nparts * 8 + 255) & ~size_t(255))
                                   : a.pairs ? (((a.m + 1) * 8 + 255) & ~size_t(255)) : 0;
    const size_t scan_bytes = (a.pairs && !single) ? ((scan_scratch_bytes(a.m) + 255) & ~size_t(255)) : 0;
    // heavy-segment queue (count-only and per-probe counts): 2^20 items, 32 MB
    const bool use_heavy = !a.pairs;
    const uint32_t hcap = use_heavy ? (1u << 20) : 0;
    const size_t heavy_bytes = size_t(hcap) * sizeof(HeavyItem);
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                             ps_bytes + pscr + reorg_bytes + cnt_bytes + po_bytes + scan_bytes +
                                 heavy_bytes + 256,
                             s)) != cudaSuccess)
        return e;
    char* cur = scratch;
    OffT* ppart = reinterpret_cast<OffT*>(cur);
    cur += ps_bytes;
    void* pscratch = cur;
    cur += pscr;
    void* reorg = cur;
    cur += reorg_bytes;
    uint32_t* pcount = reinterpret_cast<uint32_t*>(cur);
    cur += cnt_bytes;
    uint64_t* pair_off = reinterpret_cast<uint64_t*>(cur);
    cur += po_bytes;
    void* scan_scr = cur;
    cur += scan_bytes;
    HeavyQueue hq;
    if (use_heavy) {
        hq.items = reinterpret_cast<HeavyItem*>(cur);
        cur += heavy_bytes;
        hq.cap = hcap;
    }
    uint32_t* ticket = reinterpret_cast<uint32_t*>(cur);  // ticket, heavy count, slack flag
    if (use_heavy) hq.n = ticket + 1;
    Slack sl = sl_caps;
    sl.flag = ticket + 2;
    const uint64_t in_cap = sl.cap1 && sl.cap2 && g.b2 > 0 ? sl.cap2 : 0;
    // deferred heavy walks, after the partitioned kernel (per-probe counts: COUNTS)
    auto run_heavy = [&](bool counts) -> cudaError_t {
        const unsigned gh = unsigned(num_sms() * 2);
        if (counts) {
            HG_LAUNCH("k8h_heavy_walk", s,
                      (k_heavy_walk<K, true><<<gh, kHeavyBlock, 0, s>>>(hq.items, hq.n, hq.cap, tkeys,
                                                                        a.totals, a.counts)));
        } else {
            HG_LAUNCH("k8h_heavy_walk", s,
                      (k_heavy_walk<K, false><<<gh, kHeavyBlock, 0, s>>>(hq.items, hq.n, hq.cap,
                                                                         tkeys, a.totals, nullptr)));
        }
        return cudaGetLastError();
    };
    do {
        if (need_idx) {
            if ((e = cudaMemsetAsync(ticket, 0, 16, s)) != cudaSuccess) break;
            e = partition<K, IT, OffT, POW2>(probes, static_cast<const IT*>(nullptr), a.m, t.seed,
                                             t.hash_kind, nv, g, ppart, pscratch,
                                             static_cast<E1*>(reorg), s, kProbePassNames,
                                             static_cast<const E1*>(a.records), 0, &sl);
        } else {
            if ((e = cudaMemsetAsync(ticket, 0, 16, s)) != cudaSuccess) break;
            e = partition<K, void, OffT, POW2>(probes, static_cast<const void*>(nullptr), a.m,
                                               t.seed, t.hash_kind, nv, g, ppart, pscratch,
                                               static_cast<E0*>(reorg), s, kProbePassNames, nullptr,
                                               0, &sl);
        }
        if (e != cudaSuccess) break;
        const size_t smem = ProbeLayout<K, OffT, E1>::bytes(P, kcap, pcap);
        auto launch = [&](auto kern, const char* name, uint32_t* pc, const uint64_t* po, void* pr,
                          uint64_t cap) -> cudaError_t {
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(smem));
            if (r != cudaSuccess) return r;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPartProbeBlock, smem);
            const unsigned gk = unsigned(
                std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * sms, g.nparts));
            if ((r = cudaMemsetAsync(ticket, 0, 8, s)) != cudaSuccess) return r;
            HG_LAUNCH(name, s,
                      kern<<<gk, kPartProbeBlock, smem, s>>>(
                          static_cast<const E1*>(reorg), ppart, g.nparts, t.nv, t.seed,
                          t.hash_kind, nv, g.pshift, offs, tkeys, tvals, kcap, pcap, pc, po, pr,
                          cap, a.totals, ticket, (pc == a.counts && pc) ? hq : HeavyQueue{},
                          (pc == a.counts && pc) ? in_cap : 0, sl.flag));
            return cudaGetLastError();
        };
        // the pairs kernel reads its probe entries straight from global memory
        // (coalesced; its second pass hits L2), so only the offsets and table
        // keys are staged and more CTAs fit per SM
        const size_t smem_pairs = ProbeLayout<K, OffT, E1>::bytes(P, kcap_pairs, 0) +
                                  pair_val_bytes<VT>(kcap_pairs) +
                                  size_t(kPairRound) * kPartProbeBlock * sizeof(uint32_t);
        auto launch_pairs = [&](auto kern, uint64_t* status) -> cudaError_t {
            const size_t smem = smem_pairs;
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(smem));
            if (r != cudaSuccess) return r;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPartProbeBlock, smem);
            const unsigned gk = unsigned(
                std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * sms, g.nparts));
            if ((r = cudaMemsetAsync(ticket, 0, 4, s)) != cudaSuccess) return r;
            HG_LAUNCH("k10p_probe_pairs", s,
                      kern<<<gk, kPartProbeBlock, smem, s>>>(
                          static_cast<const E1*>(reorg), ppart, g.nparts, t.nv, t.seed,
                          t.hash_kind, nv, g.pshift, offs, tkeys, tvals, kcap_pairs, 0, status,
                          a.pairs, a.cap, a.totals, ticket, in_cap, sl.flag));
            return cudaGetLastError();
        };
        if (!need_idx) {
            // count-only: key-only entries
            auto kern = k_probe_part<K, VT, OffT, void, POW2, 0, false, uint32_t>;
            const size_t smem0 = ProbeLayout<K, OffT, E0>::bytes(P, kcap, pcap);
            cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(smem0));
            if (r != cudaSuccess) { e = r; break; }
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPartProbeBlock, smem0);
            const unsigned gk = unsigned(
                std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * sms, g.nparts));
            if ((e = cudaMemsetAsync(ticket, 0, 8, s)) != cudaSuccess) break;  // not the flag
            HG_LAUNCH("k8p_probe_part", s,
                      kern<<<gk, kPartProbeBlock, smem0, s>>>(
                          static_cast<const E0*>(reorg), ppart, g.nparts, t.nv, t.seed,
                          t.hash_kind, nv, g.pshift, offs, tkeys, tvals, kcap, pcap, nullptr,
                          nullptr, nullptr, 0, a.totals, ticket, hq, in_cap, sl.flag));
            if ((e = cudaGetLastError()) != cudaSuccess) break;
            e = run_heavy(false);
            break;
        }
        if (!a.pairs) {
            // per-probe counts in the caller's (original) order
            e = launch(k_probe_part<K, VT, OffT, IT, POW2, 1, true, uint32_t>, "k8p_probe_part",
                       a.counts, nullptr, nullptr, 0);
            if (e == cudaSuccess) e = run_heavy(true);
            break;
        }
        if (single) {
            // single pass: counts, look-back over partitions, pairs
            uint64_t* status = pair_off;  // nparts status words
            if ((e = cudaMemsetAsync(status, 0, g.nparts * sizeof(uint64_t), s)) != cudaSuccess) break;
            // probe indices inside a partition in 32 bits unless the whole
            // probe set could put 2^31 probes into one partition
            const bool wide = a.m >= (uint64_t(1) << 31);
            if (a.pair_bytes == 4) {
                e = wide ? launch_pairs(k_probe_pairs<K, VT, OffT, IT, POW2, uint32_t, uint64_t>, status)
                         : launch_pairs(k_probe_pairs<K, VT, OffT, IT, POW2, uint32_t, uint32_t>, status);
            } else {
                e = wide ? launch_pairs(k_probe_pairs<K, VT, OffT, IT, POW2, uint64_t, uint64_t>, status)
                         : launch_pairs(k_probe_pairs<K, VT, OffT, IT, POW2, uint64_t, uint32_t>, status);
            }
            break;
        }
        // pairs: counts in partition order -> pair slots -> pairs
        e = launch(k_probe_part<K, VT, OffT, IT, POW2, 1, false, uint32_t>, "k8p_probe_part",
                   pcount, nullptr, nullptr, 0);
        if (e != cudaSuccess) break;
        if (want_counts) {
            HG_LAUNCH("p_counts_scatter", s,
                      (k_scatter_counts<K, IT><<<unsigned(std::min<uint64_t>((a.m + 255) / 256,
                                                                             uint64_t(sms) * 16)),
                                                 256, 0, s>>>(static_cast<const E1*>(reorg),
                                                              pcount, a.m, a.counts)));
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        if ((e = launch_scan<uint32_t, uint64_t>(pcount, pair_off, a.m, scan_scr, pair_off + a.m, s,
                                                 "k9_pair_scan")) != cudaSuccess)
            break;
        if (a.cap == 0) break;
        if (a.pair_bytes == 4) {
            e = launch(k_probe_part<K, VT, OffT, IT, POW2, 2, false, uint32_t>, "k10p_probe_write",
                       nullptr, pair_off, a.pairs, a.cap);
        } else {
            e = launch(k_probe_part<K, VT, OffT, IT, POW2, 2, false, uint64_t>, "k10p_probe_write",
                       nullptr, pair_off, a.pairs, a.cap);
        }
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

// Tables whose vertex range is too wide for the partitioned probe (its
// offsets slice must fit shared memory within 2^16 partitions: V > 2^30 at
// load 1, e.g. 2^31-key tables or C5's 2^32 vertices on one GPU): the probes
// are first split into power-of-two vertex-range slices (one pass of the
// partition machinery; keys only when counting, records {key, probe
// position} for per-probe counts) and each slice is probed by the
// partitioned probe against its view of the table (offsets of the slice's
// range, global entry positions).
template <typename K, typename VT, typename OffT, typename IT, int POW2>
static cudaError_t probe_sliced(const TableDesc& t, const ProbeArgs& a, uint32_t sshift,
                                cudaStream_t s) {
    using E = typename EntryT<K, IT>::T;
    const uint64_t S = uint64_t(1) << sshift;
    const uint64_t G = (t.nv + S - 1) / S;
    if (G > 256) return cudaErrorInvalidValue;
    const bool idx = a.counts != nullptr && a.counts_requested;
    PartGeom sg;  // one split pass: "partition" = slice of 2^sshift vertices
    sg.pshift = sshift;
    sg.nparts = G;
    sg.bits = sg.b1 = ceil_log2(G);
    sg.b2 = 0;
    const size_t bytes = (a.m * (idx ? sizeof(E) : sizeof(K)) + 255) & ~size_t(255);
    const size_t sbytes = ((G + 1) * 8 + 255) & ~size_t(255);
    const size_t pbytes = idx ? PartitionScratch<K, IT, uint64_t>::bytes(sg, a.m)
                              : PartitionScratch<K, void, uint64_t>::bytes(sg, a.m);
    char* scratch = nullptr;
    cudaError_t e = cudaSuccess;
    if (huge_allocation(bytes + sbytes + pbytes)) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes + sbytes + pbytes, s);
    if (e != cudaSuccess) return e;
    uint64_t* dstart = reinterpret_cast<uint64_t*>(scratch + bytes);
    uint64_t cnt[257];
    static const char* const kNames[3] = {"slice_hist", "slice_split", "slice_split2"};
    do {
        const Divisor nv = make_divisor(global_nv(t), t.vbase);
        const K* probes = static_cast<const K*>(a.probes);
        if (idx) {  // records {key, probe position}
            e = partition<K, IT, uint64_t, POW2>(probes, static_cast<const IT*>(nullptr), a.m, t.seed,
                                                 t.hash_kind, nv, sg, dstart,
                                                 scratch + bytes + sbytes,
                                                 reinterpret_cast<E*>(scratch), s, kNames);
        } else {    // keys only
            e = partition<K, void, uint64_t, POW2>(probes, static_cast<const void*>(nullptr), a.m,
                                                   t.seed, t.hash_kind, nv, sg, dstart,
                                                   scratch + bytes + sbytes,
                                                   reinterpret_cast<K*>(scratch), s, kNames);
        }
        if (e != cudaSuccess) break;
        if ((e = cudaMemcpyAsync(cnt, dstart, (G + 1) * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess)
            break;
        for (uint64_t g = 0; g < G; ++g) cnt[g] = cnt[g + 1] - cnt[g];
        uint64_t start = 0;
        for (uint64_t g = 0; g < G && e == cudaSuccess; ++g) {
            TableDesc sub = t;
            sub.nv = t.nv - g * S < S ? t.nv - g * S : S;
            sub.gnv = global_nv(t);
            sub.vbase = t.vbase + g * S;
            sub.offs = static_cast<OffT*>(t.offs) + g * S;  // global entry positions
            sub.n = uint64_t(double(t.n) * double(sub.nv) / double(t.nv));  // density estimate
            ProbeArgs sa = a;
            sa.m = cnt[g];
            sa.method = 2;
            if (idx) {
                sa.probes = nullptr;
                sa.records = reinterpret_cast<const E*>(scratch) + start;
            } else {
                sa.probes = reinterpret_cast<const K*>(scratch) + start;
                sa.counts = nullptr;
            }
            if (sa.m) e = probe_partitioned<K, VT, OffT, IT, POW2>(sub, sa, s);
            start += cnt[g];
        }
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

template <typename K, typename VT, typename OffT, int POW2>
static cudaError_t probe_impl(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    const Divisor nv = make_divisor(global_nv(t), t.vbase);
    const OffT* offs = static_cast<const OffT*>(t.offs);
    const K* probes = static_cast<const K*>(a.probes);
    const K* tkeys = static_cast<const K*>(t.keys);
    if (a.m == 0) {
        if (a.pairs && a.pair_offsets) return cudaMemsetAsync(a.pair_offsets, 0, 8, s);
        return cudaSuccess;
    }
    const uint64_t table_bytes = (t.nv + 1) * sizeof(OffT) + t.n * sizeof(K);
    // partitioned probes need the partition's offsets slice in shared memory
    const PartGeom pg = make_geom(t.nv, t.n, 0, 4096.0);
    const bool fits = (size_t(1) << pg.pshift) * sizeof(OffT) <= size_t(64) << 10 && pg.bits <= 16;
    const bool part = fits && (a.method == 2 || (a.method == 0 && table_bytes > (uint64_t(96) << 20) &&
                                                 a.m >= (uint64_t(1) << 20)));
    if (part) {
        if (a.m <= (uint64_t(1) << 32))
            return probe_partitioned<K, VT, OffT, uint32_t, POW2>(t, a, s);
        return probe_partitioned<K, VT, OffT, uint64_t, POW2>(t, a, s);
    }
    // too wide for one partitioned pass: slices of 2^(16 + ps) vertices, ps the
    // widest partition whose offsets slice fits (count-only / per-probe counts)
    if (!fits && !a.pairs && a.method != 1 && table_bytes > (uint64_t(96) << 20) &&
        a.m >= (uint64_t(1) << 20)) {
        const double per_vertex = double(t.n) / double(t.nv);
        uint32_t ps = 0;  // make_geom's natural width (~4096 entries per partition)
        while (ps < kMaxPartShift && per_vertex * double(uint64_t(2) << ps) <= 4096.0) ++ps;
        while (ps > 0 && (size_t(1) << ps) * sizeof(OffT) > size_t(64) << 10) --ps;
        if (a.m <= (uint64_t(1) << 32))
            return probe_sliced<K, VT, OffT, uint32_t, POW2>(t, a, 16 + ps, s);
        return probe_sliced<K, VT, OffT, uint64_t, POW2>(t, a, 16 + ps, s);
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
cudaError_t probe_pow(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return dispatch_hash_mode(hash_mode(global_nv(t), t.hash_kind), [&](auto hm) {
        return probe_impl<K, VT, OffT, decltype(hm)::value>(t, a, s);
    });
}

}  // namespace hg
