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

template <typename K, typename VT>
struct BuildLayout {
    using E = typename EntryT<K, VT>::T;
    static constexpr int kItems = sizeof(E) >= 16 ? 6 : 9;
    static constexpr uint32_t kCap = kBuildBlock * kItems;  // staged entries per partition
    __host__ __device__ static size_t in_bytes() { return align16(size_t(kCap) * sizeof(E) + 32); }
    __host__ __device__ static size_t k_bytes() { return align16(size_t(kCap + 4) * sizeof(K)); }
    __host__ __device__ static size_t v_bytes() { return align16(size_t(kCap + 4) * sizeof(VT)); }
    static size_t bytes(uint32_t P) { return align16(size_t(P) * 4) + in_bytes() + k_bytes() + v_bytes(); }
};

template <typename K, typename VT, typename OffT, int POW2>
__global__ void __launch_bounds__(kBuildBlock)
k_part_build(const typename EntryT<K, VT>::T* __restrict__ reorg,
             const OffT* __restrict__ part_start /* nparts + 1 partition offsets */,
             uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
             uint32_t pshift, OffT* __restrict__ offs, K* __restrict__ okeys,
             VT* __restrict__ ovals, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_n) {
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
    auto issue = [&](uint64_t s, uint64_t e) {  // thread 0
        if (e - s <= cap) {
            fence_proxy_async();
            s_ofs = tma_load_span(inb, reorg + s, uint32_t((e - s) * sizeof(E)), &s_bar);
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const uint64_t p0 = blockIdx.x;
        if (p0 < nparts) {
            s_s = part_start[p0];
            s_e = part_start[p0 + 1];
            issue(s_s, s_e);
        }
        if (p0 + step < nparts) {
            n_s = part_start[p0 + step];
            n_e = part_start[p0 + step + 1];
        }
    }
    __syncthreads();
    uint32_t phase = 0;
    for (uint64_t p = blockIdx.x; p < nparts; p += step) {
        const uint64_t s = s_s, e = s_e;
        const uint32_t cntp = uint32_t(e - s);
        const bool staged = cntp <= cap;
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
        if ((pv & 3) == 0) {
            for (uint32_t j = 4 * tid; j < pv; j += 4 * kBuildBlock) sts128(cnt + j, make_uint4(0, 0, 0, 0));
        } else {
            for (uint32_t j = tid; j < pv; j += kBuildBlock) cnt[j] = 0;
        }
        E ent[kItems];
        if (staged) {
            mbar_wait(&s_bar, phase);
            phase ^= 1;
            const E* src = reinterpret_cast<const E*>(inb + s_ofs);
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kBuildBlock;
                if (i < cntp) ent[k] = src[i];
            }
        }
        __syncthreads();  // cnt zeroed, input buffer consumed
        if (tid == 0) {
            // next partition's entries stream in while this one is built
            const uint64_t pn = p + step;
            if (pn < nparts) issue(n_s, n_e);
            s_s = n_s;
            s_e = n_e;
            if (pn + step < nparts) {
                n_s = part_start[pn + step];
                n_e = part_start[pn + step + 1];
            }
        }
        // count: the second hash evaluation of V2's create_table pass
        // (core.hpp:126-133); the returned count is the entry's rank
        uint32_t lr[kItems];
        if (staged) {
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kBuildBlock;
                if (i < cntp) {
                    const uint32_t lv = uint32_t(hv<POW2>(PE::key(ent[k]), seed, hk, nv) - vb);
                    lr[k] = (lv << 16) | atomicAdd(cnt + lv, 1u);
                }
            }
        } else {
            // oversized (skewed) partition: built by the grid-wide K7b
            // kernels; here only its counters (offs[vb+1 .. vb+pv]) are zeroed
            for (uint32_t j = tid; j < pv; j += kBuildBlock) offs[vb + j + 1] = OffT(0);
            if (p == 0 && tid == 0) offs[0] = 0;
            if (tid == 0) big_list[atomicAdd(big_n, 1u)] = uint32_t(p);
            __syncthreads();
            continue;
        }
        __syncthreads();
        // exclusive scan of cnt[0..pv): thread owns `per` consecutive counters
        // (vectorised 16-byte shared loads/stores when per is a multiple of 4)
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
        if (warp == 0) {
            const uint32_t w = lane < kBuildBlock / 32 ? s_warp[lane] : 0;
            uint32_t wi = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
                if (int(lane) >= d) wi += y;
            }
            if (lane < kBuildBlock / 32) s_warp[lane] = wi - w;
        }
        __syncthreads();
        uint32_t acc = s_warp[warp] + inc - run;
        if (vec) {
            for (uint32_t q = 0; q < per; q += 4) {
                const uint4 c4 = lds128(cnt + j0 + q);
                const uint4 st = make_uint4(acc, acc + c4.x, acc + c4.x + c4.y,
                                            acc + c4.x + c4.y + c4.z);
                sts128(cnt + j0 + q, st);
                const uint32_t nxt = st.w + c4.w;
                if (!coal) {
                    offs[vb + j0 + q + 1] = OffT(s + st.y);
                    offs[vb + j0 + q + 2] = OffT(s + st.z);
                    offs[vb + j0 + q + 3] = OffT(s + st.w);
                    offs[vb + j0 + q + 4] = OffT(s + nxt);
                }
                acc = nxt;
            }
        } else {
            for (uint32_t j = j0; j < j1; ++j) {
                const uint32_t c = cnt[j];
                cnt[j] = acc;  // exclusive start
                acc += c;
                if (!coal) offs[vb + j + 1] = OffT(s + acc);  // end(j)
            }
        }
        if (p == 0 && tid == 0) offs[0] = 0;
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
                    make_uint4(uint32_t(s) + st.y, uint32_t(s) + st.z, uint32_t(s) + st.w,
                               uint32_t(s) + nxt);
            }
        }
        if (staged) {
            K* skp = sk + (s & (KA - 1));
            VT* svp = sv + (s & (VA - 1));
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kBuildBlock;
                if (i < cntp) {
                    const uint32_t pos = cnt[lr[k] >> 16] + (lr[k] & 0xFFFFu);
                    skp[pos] = PE::key(ent[k]);
                    svp[pos] = PE::val(ent[k]);
                }
            }
            fence_proxy_async();
            __syncthreads();
            const bool a = bulk_store_span(okeys + s, skp, cntp, tid, kBuildBlock);
            const bool b = bulk_store_span(ovals + s, svp, cntp, tid, kBuildBlock);
            if (a || b) bulk_commit();
        }
        __syncthreads();
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------- K67 (fused)
// Pass 2 of the partitioning (K6b) and the per-partition build (K7) in one
// persistent kernel, so the partition-ordered entries travel through L2
// instead of HBM. Tasks come from one atomic ticket in the order
//   [pass-2 tiles of bucket 0][partitions of bucket 0][tiles of bucket 1]...
// (bucket = one pass-1 digit = 2^b2 partitions, ~8 MB of entries at C2), so
// at any time the grid works on about one bucket: its tiles scatter the
// bucket's entries into `reorg`, and its partition tasks -- which wait for
// the bucket's tile counter -- read them back while they are still in L2 and
// then discard the lines (discard.global.L2: no write-back of dead data).
// Thread 0 schedules: while the CTA processes task i, the TMA load of task
// i+1 is already in flight into the other of two stage buffers (a partition
// task whose bucket is not finished yet is loaded at the top of the next
// iteration instead). A stage buffer holds a tile or a partition's entries;
// after a partition's entries are in registers it is reused as the key /
// value staging for that partition's TMA bulk stores.
constexpr int kFuseBlock = 512;
constexpr uint32_t kFuseLag = 1;  // buckets between a bucket's tiles and its partitions

template <typename K, typename VT>
struct FuseLayout {
    using E = typename EntryT<K, VT>::T;
    static constexpr int kTileItems = split_items<E>();
    static constexpr uint32_t kTile = kFuseBlock * kTileItems;
    static constexpr int kItems = 9;                        // partition entries per thread
    // staged entries per partition: 1/16 above the 4096-entry partitions the
    // geometry aims for (larger ones take the K7b path), so two CTAs fit an SM
    static constexpr uint32_t kCap = 4096 + 256;
    static_assert(kCap <= uint32_t(kFuseBlock) * kItems, "items per thread");
    static constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
    // stage: a tile, or a partition's entries and later its key staging
    static constexpr size_t kStage =
        align16(cmax(cmax(size_t(kTile) * sizeof(E), size_t(kCap) * sizeof(E)),
                     size_t(kCap + 4) * sizeof(K)) + 32);
    // region B: a tile's digit-sorted entries + digits, or a partition's
    // vertex counters followed by its value staging
    static size_t region_b(uint32_t P) {
        return cmax(align16(size_t(kTile) * sizeof(E)) + align16(kTile),
                    align16(size_t(P) * 4) + align16(size_t(kCap + 4) * sizeof(VT)));
    }
    static size_t bytes(uint32_t P) { return 2 * kStage + region_b(P); }
};

struct FuseTask {
    uint64_t s, e;      // tile: entry range in mid; partition: entry range in reorg
    uint64_t p;         // partition id (partition task)
    uint32_t b;         // bucket
    uint32_t kind;      // 0 none (past the end), 1 tile, 2 partition, 3 oversized partition
    uint32_t ofs;       // byte offset of the data inside the stage buffer
    uint32_t loaded;    // a TMA load was issued (the stage barrier will complete)
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void discard_l2(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <typename K, typename VT, typename OffT, int POW2>
__global__ void __launch_bounds__(kFuseBlock, 2)
k_split_build(const typename EntryT<K, VT>::T* __restrict__ mid, OffT* __restrict__ cur2,
              const OffT* __restrict__ part_start, const uint64_t* __restrict__ tile_prefix,
              uint32_t nb1, uint32_t b2, uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk,
              Divisor nv, uint32_t pshift, typename EntryT<K, VT>::T* __restrict__ reorg,
              OffT* __restrict__ offs, K* __restrict__ okeys, VT* __restrict__ ovals,
              uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_n,
              uint32_t* __restrict__ ticket, uint32_t* __restrict__ done) {
    using PE = EntryT<K, VT>;
    using E = typename PE::T;
    using L = FuseLayout<K, VT>;
    constexpr int kItems = L::kItems;
    constexpr int kTileItems = L::kTileItems;
    constexpr uint32_t cap = L::kCap;
    constexpr uint32_t KA = 16 / sizeof(K), VA = 16 / sizeof(VT);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* const stage0 = smem;
    unsigned char* const regb = smem + 2 * L::kStage;
    E* const s_ent = reinterpret_cast<E*>(regb);
    uint8_t* const s_dig = regb + align16(size_t(L::kTile) * sizeof(E));
    uint32_t* const cnt = reinterpret_cast<uint32_t*>(regb);
    __shared__ uint64_t s_bar[2];
    __shared__ FuseTask s_task[2];
    __shared__ uint32_t s_ts[kMaxDigits + 1 + kFuseLag], s_tp[kMaxDigits + 1];
    __shared__ OffT s_bs[kMaxDigits + 1];
    __shared__ uint32_t s_cnt[kMaxDigits], s_off[kMaxDigits];
    __shared__ OffT s_gbo[kMaxDigits];
    __shared__ uint32_t s_wsum[kFuseBlock / 32];
    __shared__ uint32_t s_defer;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t P = 1u << pshift;
    const uint32_t ndig = 1u << b2;
    for (uint32_t b = tid; b <= nb1; b += kFuseBlock) {
        const uint64_t q = (uint64_t(b) << b2) < nparts ? (uint64_t(b) << b2) : nparts;
        s_tp[b] = tile_prefix[b];
        s_bs[b] = part_start[q];
    }
    __syncthreads();
    // Step k of the task sequence = [tiles of bucket k][partitions of bucket
    // k - kLag]: a bucket's partitions are handed out one bucket after its
    // tiles, so they rarely wait, while ~kLag + 1 buckets (~16 MB at C2) are
    // live in L2. s_ts[k] = first task of step k.
    const uint32_t nsteps = nb1 + kFuseLag;
    if (tid == 0) {
        uint64_t acc = 0;
        for (uint32_t k = 0; k < nsteps; ++k) {
            s_ts[k] = acc;
            if (k < nb1) acc += s_tp[k + 1] - s_tp[k];
            if (k >= kFuseLag) {
                const uint64_t b = k - kFuseLag;
                const uint64_t hi = ((b + 1) << b2) < nparts ? ((b + 1) << b2) : nparts;
                acc += hi - (b << b2);
            }
        }
        s_ts[nsteps] = acc;
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // ---- scheduler helpers (thread 0)
    auto decode = [&](uint64_t t, FuseTask& k) {
        k.kind = 0;
        k.loaded = 0;
        if (t >= s_ts[nsteps]) return;
        uint32_t lo = 0, hi = nsteps;
        while (hi - lo > 1) {
            const uint32_t m = (lo + hi) >> 1;
            if (s_ts[m] <= t) lo = m; else hi = m;
        }
        const uint64_t r = t - s_ts[lo];
        const uint64_t ntiles = lo < nb1 ? s_tp[lo + 1] - s_tp[lo] : 0;
        if (r < ntiles) {
            k.b = lo;
            k.kind = 1;
            k.s = s_bs[lo] + r * L::kTile;
            k.e = s_bs[lo + 1] < k.s + L::kTile ? s_bs[lo + 1] : k.s + L::kTile;
        } else {
            k.b = lo - kFuseLag;
            k.p = (uint64_t(k.b) << b2) + (r - ntiles);
            k.s = part_start[k.p];
            k.e = part_start[k.p + 1];
            k.kind = k.e - k.s <= cap ? 2 : 3;
        }
    };
    auto bucket_ready = [&](uint32_t b) { return ld_acquire_u32(done + b) >= uint32_t(s_tp[b + 1] - s_tp[b]); };
    auto issue = [&](FuseTask& k, int st) {  // data load of a decoded task
        if (k.kind == 1 || k.kind == 2) {
            const E* src = k.kind == 1 ? mid + k.s : reorg + k.s;
            fence_proxy_async();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            k.ofs = tma_load_span(stage0 + st * L::kStage, src, uint32_t((k.e - k.s) * sizeof(E)),
                                  &s_bar[st]);
            k.loaded = 1;
        }
    };

    if (tid == 0) {
        FuseTask k;
        decode(atomicAdd(ticket, 1u), k);
        if (k.kind == 2)
            while (!bucket_ready(k.b)) __nanosleep(200);
        issue(k, 0);
        s_task[0] = k;
        s_defer = 0;
    }
    uint32_t ph[2] = {0, 0};
    for (uint32_t it = 0;; ++it) {
        const int st = int(it & 1);
        __syncthreads();  // s_task[st] published; previous task fully done
        FuseTask cur = s_task[st];
        if (cur.kind == 0) break;
        if (tid == 0 && s_defer) {
            // deferred load of this partition task: its bucket is finishing
            while (!bucket_ready(cur.b)) __nanosleep(100);
            issue(cur, st);
            s_task[st] = cur;
            s_defer = 0;
        }
        if (tid == 0) {
            // next task: load it now into the other stage unless it must wait
            bulk_wait_read();  // earlier bulk stores no longer read that buffer
            FuseTask nk;
            decode(atomicAdd(ticket, 1u), nk);
            if (nk.kind == 2 && !bucket_ready(nk.b)) {
                s_defer = 1;
            } else {
                issue(nk, st ^ 1);
            }
            s_task[st ^ 1] = nk;
        }
        __syncthreads();
        cur = s_task[st];
        const unsigned char* const sbuf = stage0 + st * L::kStage;
        if (cur.loaded) {
            mbar_wait(&s_bar[st], ph[st]);
            ph[st] ^= 1;
        }
        if (cur.kind == 1) {
            // ---------------- pass-2 tile: split by the low digit
            const E* src = reinterpret_cast<const E*>(sbuf + cur.ofs);
            const uint32_t n_t = uint32_t(cur.e - cur.s);
            const uint64_t cbase = uint64_t(cur.b) << b2;
            for (uint32_t d = tid; d < ndig; d += kFuseBlock) s_cnt[d] = 0;
            __syncthreads();
            E ent[kTileItems];
            uint32_t dr[kTileItems];
#pragma unroll
            for (int k = 0; k < kTileItems; ++k) {
                const uint32_t j = tid + k * kFuseBlock;
                if (j < n_t) {
                    ent[k] = src[j];
                    const uint32_t pp = uint32_t(hv<POW2>(PE::key(ent[k]), seed, hk, nv) >> pshift);
                    const uint32_t d = pp & (ndig - 1);
                    dr[k] = (d << 16) | atomicAdd(s_cnt + d, 1u);
                }
            }
            __syncthreads();
            const uint32_t c = tid < ndig ? s_cnt[tid] : 0;
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (int(lane) >= d) inc += y;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            if (tid < ndig) {
                uint32_t base = 0;
                for (uint32_t w = 0; w < warp; ++w) base += s_wsum[w];
                const uint32_t off = base + inc - c;
                s_off[tid] = off;
                if (c) s_gbo[tid] = atom_add(cur2 + cbase + tid, OffT(c)) - OffT(off);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kTileItems; ++k) {
                const uint32_t j = tid + k * kFuseBlock;
                if (j < n_t) {
                    const uint32_t d = dr[k] >> 16;
                    const uint32_t slot = s_off[d] + (dr[k] & 0xFFFFu);
                    s_ent[slot] = ent[k];
                    s_dig[slot] = uint8_t(d);
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kTileItems; ++k) {
                const uint32_t j = tid + k * kFuseBlock;
                if (j < n_t) reorg[uint64_t(s_gbo[s_dig[j]]) + j] = s_ent[j];
            }
            // publish the tile: the barrier orders every thread's stores before
            // thread 0's (cumulative) fence and the counter increment
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(done + cur.b, 1u);
            }
        } else if (cur.kind == 3) {
            // ---------------- oversized partition: queued for the K7b kernels
            const uint64_t vb = cur.p << pshift;
            const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
            for (uint32_t j = tid; j < pv; j += kFuseBlock) offs[vb + j + 1] = OffT(0);
            if (cur.p == 0 && tid == 0) offs[0] = 0;
            if (tid == 0) big_list[atomicAdd(big_n, 1u)] = uint32_t(cur.p);
        } else {
            // ---------------- partition build (K7 logic)
            const uint64_t s = cur.s;
            const uint32_t cntp = uint32_t(cur.e - cur.s);
            const uint64_t vb = cur.p << pshift;
            const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
            for (uint32_t j = tid; j < pv; j += kFuseBlock) cnt[j] = 0;
            const E* src = reinterpret_cast<const E*>(sbuf + cur.ofs);
            E ent[kItems];
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kFuseBlock;
                if (i < cntp) ent[k] = src[i];
            }
            __syncthreads();  // counters zeroed; stage data in registers
            // the partition's reorg lines are dead now: drop them from L2
            {
                const uintptr_t a0 = reinterpret_cast<uintptr_t>(reorg + s);
                const uintptr_t a1 = reinterpret_cast<uintptr_t>(reorg + cur.e);
                const uintptr_t l0 = (a0 + 127) & ~uintptr_t(127), l1 = a1 & ~uintptr_t(127);
                for (uintptr_t a = l0 + uintptr_t(tid) * 128; a + 128 <= l1; a += uintptr_t(kFuseBlock) * 128)
                    discard_l2(reinterpret_cast<const void*>(a));
            }
            uint32_t lr[kItems];
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kFuseBlock;
                if (i < cntp) {
                    const uint32_t lv = uint32_t(hv<POW2>(PE::key(ent[k]), seed, hk, nv) - vb);
                    lr[k] = (lv << 16) | atomicAdd(cnt + lv, 1u);
                }
            }
            __syncthreads();
            const uint32_t per = (pv + kFuseBlock - 1) / kFuseBlock;
            const uint32_t j0 = min(pv, tid * per), j1 = min(pv, j0 + per);
            const bool vec = (per & 3) == 0 && j1 - j0 == per && per <= 16;
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
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                const uint32_t w = lane < kFuseBlock / 32 ? s_wsum[lane] : 0;
                uint32_t wi = w;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
                    if (int(lane) >= d) wi += y;
                }
                if (lane < kFuseBlock / 32) s_wsum[lane] = wi - w;
            }
            __syncthreads();
            uint32_t acc = s_wsum[warp] + inc - run;
            if (vec) {
                for (uint32_t q = 0; q < per; q += 4) {
                    const uint4 c4 = lds128(cnt + j0 + q);
                    const uint4 stv = make_uint4(acc, acc + c4.x, acc + c4.x + c4.y,
                                                 acc + c4.x + c4.y + c4.z);
                    sts128(cnt + j0 + q, stv);
                    const uint32_t nxt = stv.w + c4.w;
                    if constexpr (sizeof(OffT) == 4) {
                        *reinterpret_cast<uint4*>(offs + vb + j0 + q + 1) =
                            make_uint4(uint32_t(s) + stv.y, uint32_t(s) + stv.z, uint32_t(s) + stv.w,
                                       uint32_t(s) + nxt);
                    } else {
                        offs[vb + j0 + q + 1] = OffT(s + stv.y);
                        offs[vb + j0 + q + 2] = OffT(s + stv.z);
                        offs[vb + j0 + q + 3] = OffT(s + stv.w);
                        offs[vb + j0 + q + 4] = OffT(s + nxt);
                    }
                    acc = nxt;
                }
            } else {
                for (uint32_t j = j0; j < j1; ++j) {
                    const uint32_t c = cnt[j];
                    cnt[j] = acc;
                    acc += c;
                    offs[vb + j + 1] = OffT(s + acc);
                }
            }
            if (cur.p == 0 && tid == 0) offs[0] = 0;
            __syncthreads();
            // key / value staging in this stage buffer (its entries are in registers)
            unsigned char* const stg = stage0 + st * L::kStage;
            K* skp = reinterpret_cast<K*>(stg) + (s & (KA - 1));
            VT* svp = reinterpret_cast<VT*>(regb + align16(size_t(P) * 4)) + (s & (VA - 1));
#pragma unroll
            for (int k = 0; k < kItems; ++k) {
                const uint32_t i = tid + k * kFuseBlock;
                if (i < cntp) {
                    const uint32_t pos = cnt[lr[k] >> 16] + (lr[k] & 0xFFFFu);
                    skp[pos] = PE::key(ent[k]);
                    svp[pos] = PE::val(ent[k]);
                }
            }
            fence_proxy_async();
            __syncthreads();
            const bool x = bulk_store_span(okeys + s, skp, cntp, tid, kFuseBlock);
            const bool y = bulk_store_span(ovals + s, svp, cntp, tid, kFuseBlock);
            if (x || y) bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_all();
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

template <typename OffT>
__global__ void k7b_prefix(const OffT* __restrict__ part_start, const uint32_t* __restrict__ list,
                           const uint32_t* __restrict__ big_n, uint64_t* __restrict__ pref,
                           uint64_t* __restrict__ cpref) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t nb = *big_n;
    uint64_t acc = 0, cacc = 0;
    for (uint32_t i = 0; i < nb; ++i) {
        pref[i] = acc;
        cpref[i] = cacc;
        const uint64_t sz = uint64_t(part_start[list[i] + 1]) - uint64_t(part_start[list[i]]);
        acc += sz;
        cacc += (sz + kBigChunk - 1) / kBigChunk;
    }
    pref[nb] = acc;
    cpref[nb] = cacc;
}

// Block-aggregated variant for partitions of <= 2^14 vertices: a CTA takes a
// 4096-entry chunk of one queued partition, counts it per vertex in shared
// memory (warp-aggregated shared atomics), and touches the global counters /
// cursors once per (chunk, vertex) instead of once per entry or warp -- a
// hot key costs one global atomic per chunk. PLACE: the chunk reserves each
// vertex's run with one global atomic, then hands out slots from shared
// memory.
template <typename K, typename VT, typename OffT, int POW2, bool PLACE>
__global__ void __launch_bounds__(512)
k7b_chunk(const typename EntryT<K, VT>::T* __restrict__ reorg, const OffT* __restrict__ part_start,
          const uint32_t* __restrict__ list, const uint32_t* __restrict__ big_n,
          const uint64_t* __restrict__ cpref, uint64_t nv_total, uint64_t seed, Divisor nv,
          uint32_t pshift, OffT* __restrict__ offs, K* __restrict__ okeys, VT* __restrict__ ovals) {
    using PE = EntryT<K, VT>;
    extern __shared__ __align__(128) unsigned char smem[];
    OffT* const hist = reinterpret_cast<OffT*>(smem);
    const uint32_t nb = *big_n;
    if (nb == 0) return;
    const uint64_t nchunks = cpref[nb];
    const uint32_t tid = threadIdx.x;
    const uint64_t P = uint64_t(1) << pshift;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint32_t li = big_owner(cpref, nb, c);
        const uint64_t p = list[li];
        const uint64_t s = part_start[p], e = part_start[p + 1];
        const uint64_t c0 = s + (c - cpref[li]) * kBigChunk;
        const uint64_t c1 = e < c0 + kBigChunk ? e : c0 + kBigChunk;
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : P);
        for (uint32_t v = tid; v < pv; v += blockDim.x) hist[v] = 0;
        __syncthreads();
        for (uint64_t j0 = c0; j0 < c1; j0 += blockDim.x) {
            const uint64_t j = j0 + tid;
            const bool act = j < c1;
            const uint32_t active = __ballot_sync(0xffffffffu, act);
            if (act) {
                const uint32_t lv = uint32_t(vhash<POW2>(PE::key(reorg[j]), seed, nv) - vb);
                aggregated_count<true>(hist + lv, active, lv);
            }
        }
        __syncthreads();
        for (uint32_t v = tid; v < pv; v += blockDim.x) {
            const OffT h = hist[v];
            if (h) {
                const OffT base = atom_add(offs + vb + v + 1, h);
                if constexpr (PLACE) hist[v] = base;
            }
        }
        if constexpr (PLACE) {
            __syncthreads();
            for (uint64_t j0 = c0; j0 < c1; j0 += blockDim.x) {
                const uint64_t j = j0 + tid;
                const bool act = j < c1;
                const uint32_t active = __ballot_sync(0xffffffffu, act);
                if (act) {
                    const auto en = reorg[j];
                    const uint32_t lv = uint32_t(vhash<POW2>(PE::key(en), seed, nv) - vb);
                    const uint64_t slot = aggregated_ticket<true>(hist + lv, active, lv);
                    okeys[slot] = PE::key(en);
                    ovals[slot] = PE::val(en);
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
         OffT* __restrict__ offs, K* __restrict__ okeys, VT* __restrict__ ovals) {
    using PE = EntryT<K, VT>;
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
        const uint64_t pos = uint64_t(part_start[p]) + (g - pref[li]);
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
         const uint32_t* __restrict__ big_n, uint64_t nv_total, uint32_t pshift,
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
        if (threadIdx.x == 0) s_carry = part_start[p];
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
    if (t.n == 0) return cudaMemsetAsync(offs, 0, (t.nv + 1) * sizeof(OffT), s);

    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    (void)smem_optin;
    // ~4096 entries per partition (2048 for 16-byte entries); K7 stages up
    // to BuildLayout::kCap entries of a partition in shared memory
    const PartGeom g = make_geom(t.nv, t.n, a.partition_vertices, sizeof(E) >= 16 ? 2048.0 : 4096.0);
    const size_t smem = BuildLayout<K, VT>::bytes(1u << g.pshift);

    const size_t ps_bytes = ((g.nparts + 1) * sizeof(OffT) + 255) & ~size_t(255);
    const size_t pscr = PartitionScratch<K, VT, OffT>::bytes(g, t.n);
    const size_t reorg_bytes = (t.n * sizeof(E) + 255) & ~size_t(255);
    // K7b queue: at most nparts oversized partitions
    const size_t list_bytes = ((g.nparts + 1) * 4 + 255) & ~size_t(255);
    const size_t pref_bytes = (2 * (g.nparts + 1) * 8 + 255) & ~size_t(255);  // pref | cpref
    char* scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                             ps_bytes + pscr + reorg_bytes + list_bytes + pref_bytes + 2048, s)) !=
        cudaSuccess)
        return e;
    OffT* part_start = reinterpret_cast<OffT*>(scratch);
    void* pscratch = scratch + ps_bytes;
    E* reorg = reinterpret_cast<E*>(scratch + ps_bytes + pscr);
    uint32_t* big_list = reinterpret_cast<uint32_t*>(scratch + ps_bytes + pscr + reorg_bytes);
    uint64_t* big_pref = reinterpret_cast<uint64_t*>(scratch + ps_bytes + pscr + reorg_bytes + list_bytes);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch + ps_bytes + pscr + reorg_bytes + list_bytes +
                                                   pref_bytes);  // ticket, big_n, done[kMaxDigits + 1]
    do {
        if ((e = cudaMemsetAsync(ticket, 0, 8 + 4 * (kMaxDigits + 1), s)) != cudaSuccess)
            break;  // ticket, big_n, per-bucket tile counters
        // Opt-in (HG_FUSE=1): pass 2 + K7 fused (K67) for 8-byte entries with two
        // radix passes. It moves 4 GB less DRAM traffic at C2 but, limited to
        // two CTAs per SM with a one-task prefetch, measured 3.78 ms against
        // 2.6 ms for K6b + K7, so it is not the default.
        const bool fuse = sizeof(E) == 8 && g.b2 > 0 && getenv("HG_FUSE") &&
                          getenv("HG_FUSE")[0] == '1';
        Pass2State<K, VT, OffT> p2;
        e = partition<K, VT, OffT, POW2>(static_cast<const K*>(a.keys),
                                         static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind,
                                         nv, g, part_start, pscratch, reorg, s, kBuildPassNames,
                                         fuse ? &p2 : nullptr);
        if (e != cudaSuccess) break;
        if (fuse) {
            using FL = FuseLayout<K, VT>;
            auto kf = k_split_build<K, VT, OffT, POW2>;
            const size_t fsm = FL::bytes(1u << g.pshift);
            if ((e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(fsm))) != cudaSuccess)
                break;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, kFuseBlock, fsm);
            const unsigned gf = unsigned(std::max(1, per_sm) * num_sms());
            uint32_t* done = ticket + 2;
            HG_LAUNCH("k67_split_build", s,
                      kf<<<gf, kFuseBlock, fsm, s>>>(p2.mid, p2.cur2, part_start, p2.tile_prefix,
                                                     p2.nb1, g.b2, g.nparts, t.nv, t.seed,
                                                     t.hash_kind, nv, g.pshift, reorg, offs,
                                                     static_cast<K*>(t.keys),
                                                     static_cast<VT*>(t.vals), big_list, ticket + 1,
                                                     ticket, done));
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        if (!fuse) {
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
                                                   t.hash_kind, nv, g.pshift, offs,
                                                   static_cast<K*>(t.keys),
                                                   static_cast<VT*>(t.vals), big_list,
                                                   ticket + 1));
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        // oversized partitions (device-side count; the kernels exit at once
        // when there are none)
        uint32_t* big_n = ticket + 1;
        uint64_t* big_cpref = big_pref + g.nparts + 1;
        k7b_prefix<OffT><<<1, 32, 0, s>>>(part_start, big_list, big_n, big_pref, big_cpref);
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
            const unsigned gc = unsigned(num_sms() * 3);
            HG_LAUNCH("k7b_big_count", s,
                      (kc0<<<gc, 512, hsm, s>>>(reorg, part_start, big_list, big_n, big_cpref, t.nv,
                                               t.seed, nv, g.pshift, offs, nullptr, nullptr)));
            HG_LAUNCH("k7b_big_scan", s,
                      (k7b_scan<OffT><<<unsigned(num_sms() * 2), 1024, 0, s>>>(part_start, big_list,
                                                                           big_n, t.nv, g.pshift,
                                                                           offs)));
            HG_LAUNCH("k7b_big_place", s,
                      (kc1<<<gc, 512, hsm, s>>>(reorg, part_start, big_list, big_n, big_cpref, t.nv,
                                               t.seed, nv, g.pshift, offs, static_cast<K*>(t.keys),
                                               static_cast<VT*>(t.vals))));
            e = cudaGetLastError();
            break;
        }
        HG_LAUNCH("k7b_big_count", s,
                  (k7b_pass<K, VT, OffT, POW2, false><<<gb, 256, 0, s>>>(
                      reorg, part_start, big_list, big_n, big_pref, t.seed, nv, g.pshift, offs,
                      nullptr, nullptr)));
        HG_LAUNCH("k7b_big_scan", s,
                  (k7b_scan<OffT><<<unsigned(num_sms() * 2), 1024, 0, s>>>(part_start, big_list,
                                                                       big_n, t.nv, g.pshift,
                                                                       offs)));
        HG_LAUNCH("k7b_big_place", s,
                  (k7b_pass<K, VT, OffT, POW2, true><<<gb, 256, 0, s>>>(
                      reorg, part_start, big_list, big_n, big_pref, t.seed, nv, g.pshift, offs,
                      static_cast<K*>(t.keys), static_cast<VT*>(t.vals))));
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
