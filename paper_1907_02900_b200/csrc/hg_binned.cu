// hg_binned.cu -- binned ("advanced", V2) HashGraph build on sm_100a.
//
// Replaces proj/include/hashgraph/core.hpp:183-230 (build_v2): keys are first
// scattered into contiguous vertex-range partitions ("bins",
// bin = v / bin_size, core.hpp:192-197), then every partition is built on
// chip. B200 mapping (the partition passes are in hg_radix.cuh):
//   K4 k_part_hist     partition histogram            (core.hpp:195-203)
//   K5 scan            partition starts               (core.hpp:205)
//   K6 k_multisplit x2 two 8-bit radix passes: (key,val) -> partition order
//                      (core.hpp:207-219)
//   K7 k_part_build    per partition, in shared memory: count, scan, place,
//                      then coalesced stores of offsets / keys / vals
//                      (core.hpp:221-223: create_table over the reorg array)
// The partition width P is a power of two sized so one partition's vertex
// counters plus its staged entries fit one CTA's shared memory; this is the
// B200 analogue of the reference's "bins sized to the LLC".
// The reference's bin_count only tunes CPU cache locality and never changes
// the output (hashgraph_bench.cpp:471), so P is chosen for the hardware.
#include <algorithm>
#include <cstdlib>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_radix.cuh"
#include "hg_scan.cuh"

namespace hg {

// ---------------------------------------------------------------- K7

// K7: partitions are assigned round-robin to CTAs (two CTAs per SM). Per
// partition:
//   * its entries arrive by one TMA bulk copy, issued while the previous
//     partition is still being processed (the partition bounds are loaded two
//     partitions ahead), and are moved into registers (kItems per thread);
//   * each entry's rank within its vertex is the old value returned by its
//     shared-memory count atomic, so placement needs no second atomic;
//   * keys / values are placed into shared-memory staging arrays and written
//     back with TMA bulk stores (cp.async.bulk global<-shared) that overlap
//     the next partition; offsets go out as 16-byte vector stores.
// Shared memory: cnt[P] u32 | in[cap] entries | keys[cap+4] | vals[cap+4].
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

constexpr int kBuildBlock = 512;
static const char* const kBuildPassNames[3] = {"k4_part_hist", "k6a_multisplit", "k6b_multisplit"};

// 8-byte entries (u32 key + u32 value): the partition's entries arrive by
// TMA into an input stage (prefetched during the previous partition). 16-byte
// entries: no input stage -- each thread loads its entries straight from
// global memory (16-byte coalesced loads) -- so that 9 entries per thread
// (cap 4608, C3's u64 partitions at load 1 hold ~4096) still fit two CTAs per
// SM; round 1 staged them with a cap of 3072, which sent every C3 load-1
// partition to K7b.
template <typename K, typename VT>
struct BuildLayout {
    using E = typename EntryT<K, VT>::T;
    static constexpr bool kStageIn = sizeof(E) < 16;
    static constexpr int kItems = sizeof(E) >= 16 ? 9 : 11;
    // items past kBase are touched only by partitions larger than kBase * 512
    // (a warp-uniform branch), so the common case pays for kBase items
    static constexpr int kBase = sizeof(E) >= 16 ? 9 : 9;
    static constexpr uint32_t kCap = kBuildBlock * kItems;  // entries per partition built here
    __host__ __device__ static size_t in_bytes() {
        return kStageIn ? align16(size_t(kCap) * sizeof(E) + 32) : 0;
    }
    __host__ __device__ static size_t k_bytes() { return align16(size_t(kCap + 4) * sizeof(K)); }
    __host__ __device__ static size_t v_bytes() { return align16(size_t(kCap + 4) * sizeof(VT)); }
    static size_t bytes(uint32_t P) { return align16(size_t(P) * 4) + in_bytes() + k_bytes() + v_bytes(); }
};

template <typename K, typename VT, typename OffT, int POW2>
__global__ void __launch_bounds__(kBuildBlock, 2)
k_part_build(const typename EntryT<K, VT>::T* __restrict__ reorg,
             const OffT* __restrict__ part_start /* nparts + 1 partition offsets */,
             uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
             uint32_t pshift, uint64_t obase, OffT* __restrict__ offs, K* __restrict__ okeys,
             VT* __restrict__ ovals, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_n,
             uint64_t in_cap, const uint32_t* __restrict__ slack_flag) {
    // partition p's input: the slack layout (p * in_cap) of partition_slack
    // unless it overflowed, else the dense layout (part_start[p])
    const bool slack_in = in_cap && !*slack_flag;
    using PE = EntryT<K, VT>;
    using E = typename PE::T;
    using L = BuildLayout<K, VT>;
    constexpr int kItems = L::kItems;
    constexpr uint32_t cap = L::kCap;
    constexpr uint32_t KA = 16 / sizeof(K), VA = 16 / sizeof(VT);
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t P = 1u << pshift;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    unsigned char* inb = smem + align16(size_t(P) * 4);
    K* sk = reinterpret_cast<K*>(inb + L::in_bytes());
    VT* sv = reinterpret_cast<VT*>(reinterpret_cast<unsigned char*>(sk) + L::k_bytes());
    __shared__ uint64_t s_bar;
    __shared__ uint64_t s_s, s_e;
    __shared__ uint32_t s_ofs;
    __shared__ uint32_t s_warp[kBuildBlock / 32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t step = gridDim.x;

    // thread 0: bounds of the partition after the next one (prefetched)
    uint64_t n_s = 0, n_e = 0;
    auto in_of = [&](uint64_t p, uint64_t s) -> uint64_t { return slack_in ? p * in_cap : s; };
    auto issue = [&](uint64_t p, uint64_t s, uint64_t e) {  // thread 0
        if constexpr (L::kStageIn) {
            if (e - s <= cap) {
                fence_proxy_async();
                s_ofs = tma_load_span(inb, reorg + in_of(p, s), uint32_t((e - s) * sizeof(E)), &s_bar);
            }
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const uint64_t p0 = blockIdx.x;
        if (p0 < nparts) {
            s_s = part_start[p0];
            s_e = part_start[p0 + 1];
            issue(p0, s_s, s_e);
        }
        if (p0 + step < nparts) {
            n_s = part_start[p0 + step];
            n_e = part_start[p0 + step + 1];
        }
    }
    // vertex counters: zeroed here for the first partition, then during the
    // bulk stores of the previous one (no barrier at a partition's start)
    auto zero_cnt = [&] {
        if ((P & 3) == 0) {
            for (uint32_t j = 4 * tid; j < P; j += 4 * kBuildBlock) sts128(cnt + j, make_uint4(0, 0, 0, 0));
        } else {
            for (uint32_t j = tid; j < P; j += kBuildBlock) cnt[j] = 0;
        }
    };
    zero_cnt();
    __syncthreads();
    // (thread 0, once every thread has read this partition's bounds and
    // staged input) next partition's entries stream in while this one is built
    auto advance = [&](uint64_t p) {
        const uint64_t pn = p + step;
        if (pn < nparts) issue(pn, n_s, n_e);
        s_s = n_s;
        s_e = n_e;
        if (pn + step < nparts) {
            n_s = part_start[pn + step];
            n_e = part_start[pn + step + 1];
        }
    };
    uint32_t phase = 0;
    for (uint64_t p = blockIdx.x; p < nparts; p += step) {
        const uint64_t s = s_s, e = s_e;
        const uint32_t cntp = uint32_t(e - s);
        const bool staged = cntp <= cap;
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
        // per-item loops: kBase items unrolled, the rest only for large
        // partitions. f(k, check): items below kFull of a partition holding
        // at least kFull * kBuildBlock entries (nearly all of them: 3584 of a
        // 4096 mean) run without the bounds check, so without a divergent
        // region per item (BSSY / BSYNC / BRA were 15 % of K7's instructions)
        constexpr int kFull = L::kBase - 2;
        auto for_items = [&](auto&& f) {
            if (cntp >= uint32_t(kFull) * kBuildBlock) {
#pragma unroll
                for (int k = 0; k < kFull; ++k) f(k, std::false_type{});
#pragma unroll
                for (int k = kFull; k < L::kBase; ++k) f(k, std::true_type{});
            } else {
#pragma unroll
                for (int k = 0; k < L::kBase; ++k) f(k, std::true_type{});
            }
            if (cntp > uint32_t(L::kBase) * kBuildBlock) {
#pragma unroll
                for (int k = L::kBase; k < kItems; ++k) f(k, std::true_type{});
            }
        };
        E ent[kItems];
        if (staged) {
            if constexpr (L::kStageIn) {
                mbar_wait(&s_bar, phase);
                phase ^= 1;
                const E* src = reinterpret_cast<const E*>(inb + s_ofs);
                for_items([&](int k, auto chk) {
                    const uint32_t i = tid + k * kBuildBlock;
                    if (!decltype(chk)::value || i < cntp) ent[k] = src[i];
                });
            } else {
                const E* src = reorg + in_of(p, s);
                for_items([&](int k, auto chk) {
                    const uint32_t i = tid + k * kBuildBlock;
                    if (!decltype(chk)::value || i < cntp) ent[k] = __ldcs(src + i);
                });
            }
        }
        // count: the second hash evaluation of V2's create_table pass
        // (core.hpp:126-133); the returned count is the entry's rank
        uint32_t lr[kItems];
        if (staged) {
            for_items([&](int k, auto chk) {
                const uint32_t i = tid + k * kBuildBlock;
                if (!decltype(chk)::value || i < cntp) {
                    const uint32_t lv = uint32_t(hv<POW2>(PE::key(ent[k]), seed, hk, nv) - vb);
                    lr[k] = (lv << 16) | atomicAdd(cnt + lv, 1u);
                }
            });
        } else {
            // oversized (skewed) partition: built by the grid-wide K7b
            // kernels; here only its counters (offs[vb+1 .. vb+pv]) are zeroed
            for (uint32_t j = tid; j < pv; j += kBuildBlock) offs[vb + j + 1] = OffT(0);
            if (p == 0 && tid == 0) offs[0] = OffT(obase);
            if (tid == 0) big_list[atomicAdd(big_n, 1u)] = uint32_t(p);
            __syncthreads();  // bounds read by every thread
            if (tid == 0) advance(p);
            __syncthreads();
            continue;
        }
        __syncthreads();  // counts final; staged input and bounds consumed
        if (tid == 0) advance(p);
        // exclusive scan of cnt[0..pv): thread owns `per` consecutive counters
        // (vectorised 16-byte shared loads/stores when per is a multiple of 4)
        const uint64_t so = s + obase;  // offsets are written with the table's entry base
        const uint32_t per = (pv + kBuildBlock - 1) / kBuildBlock;
        const uint32_t j0 = min(pv, tid * per), j1 = min(pv, j0 + per);
        const bool vec = (per & 3) == 0 && j1 - j0 == per && per <= 16;
        // u32 offsets of a partition whose width is a multiple of 4 are written
        // after the scan as lane-contiguous 16-byte stores (block-uniform)
        const bool coal = sizeof(OffT) == 4 && (pv & 3) == 0;
        uint32_t run = 0;
        if (vec) {
            for (uint32_t q = 0; q < per; q += 4) {
                const uint4 c4 = lds128(cnt + j0 + q);
                run += c4.x + c4.y + c4.z + c4.w;
            }
        } else {
            for (uint32_t j = j0; j < j1; ++j) run += cnt[j];
        }
        uint32_t inc = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (int(lane) >= d) inc += y;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        // each warp sums the totals of the warps before it (one load per
        // lane + a warp reduction; no second barrier)
        const uint32_t wbase = warp_sum(lane < warp ? s_warp[lane] : 0u);
        uint32_t acc = wbase + inc - run;
        if (vec) {
            for (uint32_t q = 0; q < per; q += 4) {
                const uint4 c4 = lds128(cnt + j0 + q);
                const uint4 st = make_uint4(acc, acc + c4.x, acc + c4.x + c4.y,
                                            acc + c4.x + c4.y + c4.z);
                sts128(cnt + j0 + q, st);
                const uint32_t nxt = st.w + c4.w;
                if (!coal) {
                    offs[vb + j0 + q + 1] = OffT(so + st.y);
                    offs[vb + j0 + q + 2] = OffT(so + st.z);
                    offs[vb + j0 + q + 3] = OffT(so + st.w);
                    offs[vb + j0 + q + 4] = OffT(so + nxt);
                }
                acc = nxt;
            }
        } else {
            for (uint32_t j = j0; j < j1; ++j) {
                const uint32_t c = cnt[j];
                cnt[j] = acc;  // exclusive start
                acc += c;
                if (!coal) offs[vb + j + 1] = OffT(so + acc);  // end(j)
            }
        }
        if (p == 0 && tid == 0) offs[0] = OffT(obase);
        // the previous partition's bulk stores must have read the staging arrays
        if (tid == 0) bulk_wait_read();
        __syncthreads();
        if (coal) {
            // end(j) = start(j+1) from the exclusive starts now in cnt (offs + 1
            // is 16-byte aligned, hg_capi pads it; vb + 4c is a multiple of 4)
            for (uint32_t c = tid; 4 * c < pv; c += kBuildBlock) {
                const uint4 st = lds128(cnt + 4 * c);
                const uint32_t nxt = 4 * c + 4 < pv ? cnt[4 * c + 4] : cntp;
                *reinterpret_cast<uint4*>(offs + vb + 4 * c + 1) =
                    make_uint4(uint32_t(so) + st.y, uint32_t(so) + st.z, uint32_t(so) + st.w,
                               uint32_t(so) + nxt);
            }
        }
        if (staged) {
            // staging aligned like the destination modulo 16 bytes (the table
            // arrays of a vertex-range slice start at any entry)
            K* skp = sk + ((reinterpret_cast<uintptr_t>(okeys + s) / sizeof(K)) & (KA - 1));
            VT* svp = sv + ((reinterpret_cast<uintptr_t>(ovals + s) / sizeof(VT)) & (VA - 1));
            for_items([&](int k, auto chk) {
                const uint32_t i = tid + k * kBuildBlock;
                if (!decltype(chk)::value || i < cntp) {
                    const uint32_t pos = cnt[lr[k] >> 16] + (lr[k] & 0xFFFFu);
                    skp[pos] = PE::key(ent[k]);
                    svp[pos] = PE::val(ent[k]);
                }
            });
            fence_proxy_async();
            __syncthreads();
            const bool a = bulk_store_span(okeys + s, skp, cntp, tid, kBuildBlock);
            const bool b = bulk_store_span(ovals + s, svp, cntp, tid, kBuildBlock);
            if (a || b) bulk_commit();
            zero_cnt();  // counters of the next partition (cnt is no longer read)
        }
        __syncthreads();
    }
    if (tid == 0) bulk_wait_all();
}

template <typename OffT>
__global__ void k_fill_offs(OffT* __restrict__ offs, uint64_t n, OffT v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        offs[i] = v;
}

// ---------------------------------------------------------------- K7b
// Partitions holding more entries than K7 can stage (heavy keys under skew,
// e.g. C3's Zipf ranks) are built by the whole grid instead of one CTA, with
// the partition's slice of `offs` as counter / cursor array (the V1 scheme):
//   k7b_prefix  one thread: prefix of the queued partitions' entry counts
//   k7b_count   grid-stride over all queued entries; warp-aggregated global
//               atomics on offs[v+1] (a hot vertex costs one atomic per warp)
//   k7b_scan    one CTA per queued partition: offs[v+1] := s + exclusive
//               prefix (the placement cursor)
//   k7b_place   grid-stride again; aggregated tickets on the cursors leave
//               offs[v+1] = end(v) and give each entry its slot
constexpr uint32_t kBigChunk = 4096;  // entries of a queued partition per K7b CTA task

// Queued entry g -> (partition index in the list, entry position).
__device__ __forceinline__ uint32_t big_owner(const uint64_t* pref, uint32_t nb, uint64_t g) {
    uint32_t lo = 0, hi = nb;  // pref[lo] <= g < pref[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pref[mid] <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// Exclusive prefixes of the queued partitions' entry counts (pref) and K7b
// chunk counts (cpref), one CTA: each thread sums a run of consecutive list
// entries, a block scan of the run totals, then the runs are written
// (round 1 walked the list with one thread: 65536 dependent loads for C3).
constexpr int kBigPrefixBlock = 1024;

template <typename OffT>
__global__ void __launch_bounds__(kBigPrefixBlock)
k7b_prefix(const OffT* __restrict__ part_start, const uint32_t* __restrict__ list,
           const uint32_t* __restrict__ big_n, uint64_t* __restrict__ pref,
           uint64_t* __restrict__ cpref) {
    __shared__ uint64_t s_a[kBigPrefixBlock / 32], s_c[kBigPrefixBlock / 32];
    const uint32_t nb = *big_n;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (nb + kBigPrefixBlock - 1) / kBigPrefixBlock;
    const uint32_t i0 = min(nb, tid * per), i1 = min(nb, i0 + per);
    auto size_of = [&](uint32_t i) {
        return uint64_t(part_start[list[i] + 1]) - uint64_t(part_start[list[i]]);
    };
    uint64_t a = 0, c = 0;
    for (uint32_t i = i0; i < i1; ++i) {
        const uint64_t sz = size_of(i);
        a += sz;
        c += (sz + kBigChunk - 1) / kBigChunk;
    }
    uint64_t ia = a, ic = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t ya = __shfl_up_sync(0xffffffffu, ia, d);
        const uint64_t yc = __shfl_up_sync(0xffffffffu, ic, d);
        if (int(lane) >= d) {
            ia += ya;
            ic += yc;
        }
    }
    if (lane == 31) {
        s_a[warp] = ia;
        s_c[warp] = ic;
    }
    __syncthreads();
    uint64_t ba = 0, bc = 0;
    for (uint32_t w = 0; w < warp; ++w) {
        ba += s_a[w];
        bc += s_c[w];
    }
    uint64_t acc = ba + ia - a, cacc = bc + ic - c;
    for (uint32_t i = i0; i < i1; ++i) {
        pref[i] = acc;
        cpref[i] = cacc;
        const uint64_t sz = size_of(i);
        acc += sz;
        cacc += (sz + kBigChunk - 1) / kBigChunk;
    }
    if (tid == kBigPrefixBlock - 1) {
        pref[nb] = ba + ia;
        cpref[nb] = bc + ic;
    }
}

// Block-aggregated variant for partitions of <= 2^14 vertices: a CTA takes a
// 4096-entry chunk of one queued partition, counts it per vertex in shared
// memory, and touches the global counters / cursors once per (chunk, vertex)
// instead of once per entry or warp -- a hot key costs one global atomic per
// chunk. PLACE: the chunk reserves each vertex's run with one global atomic,
// then hands out slots from shared memory.
// A thread loads its kBigPer entries of the chunk up front (all loads in
// flight at once; they are issued before the counters are zeroed) and keeps
// them, their vertices and their peer masks in registers, so PLACE reads and
// hashes each entry once. Peer groups: a warp whose lanes all hold one vertex
// (the common case inside a partition queued for a heavy key) skips
// match.any.
constexpr int kBigBlock = 512;
constexpr int kBigPer = int(kBigChunk) / kBigBlock;

__device__ __forceinline__ uint32_t big_peers(uint32_t active, uint32_t v) {
    const uint32_t v0 = __shfl_sync(active, v, __ffs(active) - 1);
    if (__all_sync(active, v == v0)) return active;
    return __match_any_sync(active, v);
}

// One K7b chunk task: partition p, cn entries starting at input index c0
// (slack region or dense range of the partition; written once
// per launch by k7b_map, so a chunk's CTA does one broadcast load instead of a
// binary search over the queue: the search was K7b's top stall).
struct __align__(16) BigChunk {
    uint32_t p, cn;
    uint64_t c0;
};

template <typename OffT>
__global__ void __launch_bounds__(256)
k7b_map(const OffT* __restrict__ part_start, const uint32_t* __restrict__ list,
        const uint32_t* __restrict__ big_n, const uint64_t* __restrict__ cpref,
        BigChunk* __restrict__ map, uint64_t in_cap, const uint32_t* __restrict__ slack_flag) {
    const bool slack_in = in_cap && !*slack_flag;
    const uint32_t nb = *big_n;
    if (nb == 0) return;
    const uint64_t nchunks = cpref[nb];
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < nchunks;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t li = big_owner(cpref, nb, c);
        const uint32_t p = list[li];
        const uint64_t s = part_start[p], e = part_start[p + 1];
        const uint64_t c0 = s + (c - cpref[li]) * kBigChunk;
        BigChunk b;
        b.p = p;
        b.cn = uint32_t((e < c0 + kBigChunk ? e : c0 + kBigChunk) - c0);
        b.c0 = (slack_in ? uint64_t(p) * in_cap : s) + (c0 - s);  // index into the input
        map[c] = b;
    }
}

template <typename K, typename VT, typename OffT, int POW2, bool PLACE>
__global__ void __launch_bounds__(kBigBlock, 2)
k7b_chunk(const typename EntryT<K, VT>::T* __restrict__ reorg, const BigChunk* __restrict__ map,
          const uint32_t* __restrict__ big_n,
          const uint64_t* __restrict__ cpref, uint64_t nv_total, uint64_t seed, Divisor nv,
          uint32_t pshift, OffT* __restrict__ offs, K* __restrict__ okeys, VT* __restrict__ ovals,
          uint64_t in_cap, const uint32_t* __restrict__ slack_flag) {
    using PE = EntryT<K, VT>;
    extern __shared__ __align__(128) unsigned char smem[];
    OffT* const hist = reinterpret_cast<OffT*>(smem);
    const uint32_t nb = *big_n;
    if (nb == 0) return;
    const uint64_t nchunks = cpref[nb];
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint64_t P = uint64_t(1) << pshift;
    // counters start at zero; the count pass re-zeroes the ones it used
    // while reserving, the place pass zeroes all at the start of a chunk
    if constexpr (!PLACE) {
        for (uint32_t v = tid; v < P; v += kBigBlock) hist[v] = 0;
    }
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const BigChunk bc = map[c];
        const uint64_t p = bc.p;
        const uint32_t cn = bc.cn;
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : P);
        const typename PE::T* rin = reorg + bc.c0;
        typename PE::T en[kBigPer];
#pragma unroll
        for (int k = 0; k < kBigPer; ++k) {
            const uint32_t j = tid + k * kBigBlock;
            if (j < cn) en[k] = rin[j];
        }
        if constexpr (PLACE) {
            for (uint32_t v = tid; v < pv; v += kBigBlock) hist[v] = 0;
        }
        __syncthreads();
        uint32_t lv[kBigPer], peers[kBigPer];
#pragma unroll
        for (int k = 0; k < kBigPer; ++k) {
            const uint32_t j = tid + k * kBigBlock;
            const bool act = j < cn;
            const uint32_t active = __ballot_sync(0xffffffffu, act);
            if (act) {
                lv[k] = uint32_t(vhash<POW2>(PE::key(en[k]), seed, nv) - vb);
                peers[k] = big_peers(active, lv[k]);
                if (lane == uint32_t(__ffs(peers[k]) - 1)) atom_add(hist + lv[k], OffT(__popc(peers[k])));
            }
        }
        __syncthreads();
        for (uint32_t v = tid; v < pv; v += kBigBlock) {
            const OffT h = hist[v];
            if (h) {
                const OffT base = atom_add(offs + vb + v + 1, h);
                hist[v] = PLACE ? base : OffT(0);
            }
        }
        if constexpr (PLACE) {
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kBigPer; ++k) {
                const uint32_t j = tid + k * kBigBlock;
                if (j < cn) {
                    const uint32_t pk = peers[k];
                    const uint32_t leader = __ffs(pk) - 1;
                    OffT base = 0;
                    if (lane == leader) base = atom_add(hist + lv[k], OffT(__popc(pk)));
                    base = __shfl_sync(pk, base, leader);
                    const uint64_t slot = uint64_t(base) + __popc(pk & lanemask_lt());
                    okeys[slot] = PE::key(en[k]);
                    ovals[slot] = PE::val(en[k]);
                }
            }
        }
        __syncthreads();
    }
}


template <typename K, typename VT, typename OffT, int POW2, bool PLACE>
__global__ void __launch_bounds__(256)
k7b_pass(const typename EntryT<K, VT>::T* __restrict__ reorg, const OffT* __restrict__ part_start,
         const uint32_t* __restrict__ list, const uint32_t* __restrict__ big_n,
         const uint64_t* __restrict__ pref, uint64_t seed, Divisor nv, uint32_t pshift,
         OffT* __restrict__ offs, K* __restrict__ okeys, VT* __restrict__ ovals, uint64_t in_cap,
         const uint32_t* __restrict__ slack_flag) {
    using PE = EntryT<K, VT>;
    const bool slack_in = in_cap && !*slack_flag;
    constexpr bool V32 = sizeof(OffT) == 4;
    const uint32_t nb = *big_n;
    if (nb == 0) return;
    const uint64_t total = pref[nb];
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t g0 = uint64_t(blockIdx.x) * blockDim.x; g0 < total; g0 += stride) {
        const uint64_t g = g0 + threadIdx.x;
        const bool act = g < total;
        const uint32_t active = __ballot_sync(0xffffffffu, act);
        if (!act) continue;
        const uint32_t li = big_owner(pref, nb, g);
        const uint64_t p = list[li];
        const uint64_t pos = (slack_in ? p * in_cap : uint64_t(part_start[p])) + (g - pref[li]);
        const auto en = reorg[pos];
        const uint64_t v = vhash<POW2>(PE::key(en), seed, nv);  // local vertex id
        if constexpr (!PLACE) {
            aggregated_count<V32>(offs + v + 1, active, v);
        } else {
            const uint64_t slot = aggregated_ticket<V32>(offs + v + 1, active, v);
            okeys[slot] = PE::key(en);
            ovals[slot] = PE::val(en);
        }
    }
    (void)pshift;
}

template <typename OffT>
__global__ void __launch_bounds__(1024)
k7b_scan(const OffT* __restrict__ part_start, const uint32_t* __restrict__ list,
         const uint32_t* __restrict__ big_n, uint64_t nv_total, uint32_t pshift, uint64_t obase,
         OffT* __restrict__ offs) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint64_t s_carry, s_tot;
    const uint32_t nb = *big_n;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t li = blockIdx.x; li < nb; li += gridDim.x) {
        const uint64_t p = list[li];
        const uint64_t vb = p << pshift;
        const uint64_t P = uint64_t(1) << pshift;
        const uint64_t pv = nv_total - vb < P ? nv_total - vb : P;
        if (threadIdx.x == 0) s_carry = part_start[p] + obase;
        __syncthreads();
        for (uint64_t j0 = 0; j0 < pv; j0 += blockDim.x) {
            const uint64_t j = j0 + threadIdx.x;
            const uint64_t c = j < pv ? uint64_t(offs[vb + j + 1]) : 0;
            uint64_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (int(lane) >= d) inc += y;
            }
            if (lane == 31) s_warp[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                const uint64_t w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
                uint64_t wi = w;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint64_t y = __shfl_up_sync(0xffffffffu, wi, d);
                    if (int(lane) >= d) wi += y;
                }
                if (lane < (blockDim.x >> 5)) s_warp[lane] = wi - w;
                if (lane == 31) s_tot = wi;  // chunk total
            }
            __syncthreads();
            const uint64_t carry = s_carry;
            if (j < pv) offs[vb + j + 1] = OffT(carry + s_warp[warp] + inc - c);
            __syncthreads();
            if (threadIdx.x == 0) s_carry = carry + s_tot;
            __syncthreads();
        }
    }
}

template <typename K, typename VT, typename OffT, int POW2>
cudaError_t build_v2_impl(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    using E = typename EntryT<K, VT>::T;
    const Divisor nv = make_divisor(global_nv(t), t.vbase);
    OffT* offs = static_cast<OffT*>(t.offs);
    cudaError_t e;
    if (t.n == 0) {
        if (t.obase == 0) return cudaMemsetAsync(offs, 0, (t.nv + 1) * sizeof(OffT), s);
        k_fill_offs<OffT><<<unsigned(std::min<uint64_t>((t.nv + 256) / 256, 4096)), 256, 0, s>>>(
            offs, t.nv + 1, OffT(t.obase));
        return cudaGetLastError();
    }

    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    (void)smem_optin;
    // ~4096 entries per partition (2048 for 16-byte entries); K7 stages up
    // to BuildLayout::kCap entries of a partition in shared memory
    const PartGeom g = make_geom(t.nv, t.n, a.partition_vertices, sizeof(E) >= 16 ? 2048.0 : 4096.0);
    const size_t smem = BuildLayout<K, VT>::bytes(1u << g.pshift);

    // slack (histogram-free) partition layout when it fits; the flag word
    // lives in the scratch tail (ticket + 2)
    const Slack sl_caps = make_slack<OffT>(g, t.n, t.nv, nullptr);
    const uint64_t nb1 = (g.nparts + (uint64_t(1) << g.b2) - 1) >> g.b2;
    const size_t ps_bytes = ((g.nparts + 1) * sizeof(OffT) + 255) & ~size_t(255);
    const size_t pscr = PartitionScratch<K, VT, OffT>::bytes(g, t.n, nb1 * sl_caps.cap1);
    const uint64_t reorg_n = std::max<uint64_t>(t.n, g.nparts * sl_caps.cap2);
    const size_t reorg_bytes = (reorg_n * sizeof(E) + 255) & ~size_t(255);
    // K7b queue: at most nparts oversized partitions
    const size_t list_bytes = ((g.nparts + 1) * 4 + 255) & ~size_t(255);
    const size_t pref_bytes = (2 * (g.nparts + 1) * 8 + 255) & ~size_t(255);  // pref | cpref
    // K7b chunk table: at most n / kBigChunk + nparts chunks
    const size_t map_bytes = ((t.n / kBigChunk + g.nparts + 1) * sizeof(BigChunk) + 255) & ~size_t(255);
    char* scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                             ps_bytes + pscr + reorg_bytes + list_bytes + pref_bytes + map_bytes + 2048,
                             s)) !=
        cudaSuccess)
        return e;
    OffT* part_start = reinterpret_cast<OffT*>(scratch);
    void* pscratch = scratch + ps_bytes;
    E* reorg = reinterpret_cast<E*>(scratch + ps_bytes + pscr);
    uint32_t* big_list = reinterpret_cast<uint32_t*>(scratch + ps_bytes + pscr + reorg_bytes);
    uint64_t* big_pref = reinterpret_cast<uint64_t*>(scratch + ps_bytes + pscr + reorg_bytes + list_bytes);
    BigChunk* big_map = reinterpret_cast<BigChunk*>(scratch + ps_bytes + pscr + reorg_bytes + list_bytes +
                                                    pref_bytes);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch + ps_bytes + pscr + reorg_bytes + list_bytes +
                                                   pref_bytes + map_bytes);  // ticket, big_n, slack flag
    Slack sl = sl_caps;
    sl.flag = ticket + 2;
    do {
        if ((e = cudaMemsetAsync(ticket, 0, 16, s)) != cudaSuccess) break;  // ticket, big_n, flag
        e = partition<K, VT, OffT, POW2>(static_cast<const K*>(a.keys),
                                         static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind,
                                         nv, g, part_start, pscratch, reorg, s, kBuildPassNames,
                                         static_cast<const E*>(a.records), 0, &sl);
        const uint64_t in_cap = sl.cap1 && sl.cap2 && g.b2 > 0 ? sl.cap2 : 0;
        if (e != cudaSuccess) break;
        auto kb = k_part_build<K, VT, OffT, POW2>;
        if ((e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem))) != cudaSuccess)
            break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb, kBuildBlock, smem);
        const unsigned gk = unsigned(
            std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * num_sms(), g.nparts));
        HG_LAUNCH("k7_part_build", s,
                  kb<<<gk, kBuildBlock, smem, s>>>(reorg, part_start, g.nparts, t.nv, t.seed,
                                                   t.hash_kind, nv, g.pshift, t.obase, offs,
                                                   static_cast<K*>(t.keys),
                                                   static_cast<VT*>(t.vals), big_list,
                                                   ticket + 1, in_cap, sl.flag));
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        // oversized partitions (device-side count; the kernels exit at once
        // when there are none)
        uint32_t* big_n = ticket + 1;
        uint64_t* big_cpref = big_pref + g.nparts + 1;
        HG_LAUNCH("k7b_big_prefix", s,
                  (k7b_prefix<OffT><<<1, kBigPrefixBlock, 0, s>>>(part_start, big_list, big_n,
                                                                  big_pref, big_cpref)));
        const unsigned gb = unsigned(num_sms() * 8);
        // block-aggregated K7b when a partition's counters fit shared memory
        const size_t hsm = (size_t(1) << g.pshift) * sizeof(OffT);
        const bool chunked = hsm <= (size_t(64) << 10);
        if (chunked) {
            auto kc0 = k7b_chunk<K, VT, OffT, POW2, false>;
            auto kc1 = k7b_chunk<K, VT, OffT, POW2, true>;
            if (hsm > (size_t(48) << 10) &&
                ((e = cudaFuncSetAttribute(kc0, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hsm))) !=
                     cudaSuccess ||
                 (e = cudaFuncSetAttribute(kc1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hsm))) !=
                     cudaSuccess))
                break;
            const unsigned gc = unsigned(num_sms() * 2);
            HG_LAUNCH("k7b_big_map", s,
                      (k7b_map<OffT><<<unsigned(num_sms() * 2), 256, 0, s>>>(part_start, big_list, big_n,
                                                                         big_cpref, big_map, in_cap, sl.flag)));
            HG_LAUNCH("k7b_big_count", s,
                      (kc0<<<gc, kBigBlock, hsm, s>>>(reorg, big_map, big_n, big_cpref, t.nv,
                                               t.seed, nv, g.pshift, offs, nullptr, nullptr, in_cap,
                                               sl.flag)));
            HG_LAUNCH("k7b_big_scan", s,
                      (k7b_scan<OffT><<<unsigned(num_sms() * 2), 1024, 0, s>>>(part_start, big_list,
                                                                           big_n, t.nv, g.pshift,
                                                                           t.obase, offs)));
            HG_LAUNCH("k7b_big_place", s,
                      (kc1<<<gc, kBigBlock, hsm, s>>>(reorg, big_map, big_n, big_cpref, t.nv,
                                               t.seed, nv, g.pshift, offs, static_cast<K*>(t.keys) - t.obase,
                                               static_cast<VT*>(t.vals) - t.obase, in_cap, sl.flag)));
            e = cudaGetLastError();
            break;
        }
        HG_LAUNCH("k7b_big_count", s,
                  (k7b_pass<K, VT, OffT, POW2, false><<<gb, 256, 0, s>>>(
                      reorg, part_start, big_list, big_n, big_pref, t.seed, nv, g.pshift, offs,
                      nullptr, nullptr, in_cap, sl.flag)));
        HG_LAUNCH("k7b_big_scan", s,
                  (k7b_scan<OffT><<<unsigned(num_sms() * 2), 1024, 0, s>>>(part_start, big_list,
                                                                       big_n, t.nv, g.pshift,
                                                                       t.obase, offs)));
        HG_LAUNCH("k7b_big_place", s,
                  (k7b_pass<K, VT, OffT, POW2, true><<<gb, 256, 0, s>>>(
                      reorg, part_start, big_list, big_n, big_pref, t.seed, nv, g.pshift, offs,
                      static_cast<K*>(t.keys) - t.obase, static_cast<VT*>(t.vals) - t.obase, in_cap,
                      sl.flag)));
        e = cudaGetLastError();
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

#define HG_INST1(K, VT, OffT, HM) \
    template cudaError_t build_v2_impl<K, VT, OffT, HM>(const TableDesc&, const BuildArgs&, cudaStream_t);
#define HG_INST(K, VT, OffT) \
    HG_INST1(K, VT, OffT, 0) HG_INST1(K, VT, OffT, 1) HG_INST1(K, VT, OffT, 2) HG_INST1(K, VT, OffT, 3)
HG_INST(uint32_t, uint32_t, uint32_t)
HG_INST(uint32_t, uint32_t, uint64_t)
HG_INST(uint32_t, uint64_t, uint32_t)
HG_INST(uint32_t, uint64_t, uint64_t)
HG_INST(uint64_t, uint32_t, uint32_t)
HG_INST(uint64_t, uint32_t, uint64_t)
HG_INST(uint64_t, uint64_t, uint32_t)
HG_INST(uint64_t, uint64_t, uint64_t)
#undef HG_INST1
#undef HG_INST

}  // namespace hg
