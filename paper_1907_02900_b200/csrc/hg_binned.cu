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
    static constexpr int kItems = sizeof(E) >= 16 ? 6 : 10;
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
             VT* __restrict__ ovals) {
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
        for (uint32_t j = tid; j < pv; j += kBuildBlock) cnt[j] = 0;
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
            for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
                const uint32_t lv = uint32_t(hv<POW2>(PE::key(reorg[s + i]), seed, hk, nv) - vb);
                atomicAdd(cnt + lv, 1u);
            }
        }
        __syncthreads();
        // exclusive scan of cnt[0..pv): thread owns `per` consecutive counters
        // (vectorised 16-byte shared loads/stores when per is a multiple of 4)
        const uint32_t per = (pv + kBuildBlock - 1) / kBuildBlock;
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
                if constexpr (sizeof(OffT) == 4) {
                    // offs + 1 is 16-byte aligned (hg_capi pads it); vb + j0 + q is a multiple of 4
                    *reinterpret_cast<uint4*>(offs + vb + j0 + q + 1) =
                        make_uint4(uint32_t(s) + st.y, uint32_t(s) + st.z, uint32_t(s) + st.w,
                                   uint32_t(s) + nxt);
                } else {
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
                offs[vb + j + 1] = OffT(s + acc);  // end(j)
            }
        }
        if (p == 0 && tid == 0) offs[0] = 0;
        // the previous partition's bulk stores must have read the staging arrays
        if (tid == 0) bulk_wait_read();
        __syncthreads();
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
        } else {
            for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
                const E en = reorg[s + i];
                const uint32_t lv = uint32_t(hv<POW2>(PE::key(en), seed, hk, nv) - vb);
                const uint64_t pos = s + atomicAdd(cnt + lv, 1u);
                okeys[pos] = PE::key(en);
                ovals[pos] = PE::val(en);
            }
        }
        __syncthreads();
    }
    if (tid == 0) bulk_wait_all();
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
    char* scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                             ps_bytes + pscr + reorg_bytes + 256, s)) != cudaSuccess)
        return e;
    OffT* part_start = reinterpret_cast<OffT*>(scratch);
    void* pscratch = scratch + ps_bytes;
    E* reorg = reinterpret_cast<E*>(scratch + ps_bytes + pscr);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch + ps_bytes + pscr + reorg_bytes);
    do {
        if ((e = cudaMemsetAsync(ticket, 0, 4, s)) != cudaSuccess) break;
        e = partition<K, VT, OffT, POW2>(static_cast<const K*>(a.keys),
                                         static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind,
                                         nv, g, part_start, pscratch, reorg, s, kBuildPassNames);
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
                                                   t.hash_kind, nv, g.pshift, offs,
                                                   static_cast<K*>(t.keys),
                                                   static_cast<VT*>(t.vals)));
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
