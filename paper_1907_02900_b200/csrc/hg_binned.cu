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

// K7 shared-memory layout (1 CTA of 1024 threads per SM):
//   cnt[P] u32 | lv[cap] u16 | in[2][cap] entries (TMA double buffer) | keys[cap] | vals[cap]
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename K, typename VT>
struct BuildLayout {
    using E = typename EntryT<K, VT>::T;
    __host__ __device__ static size_t in_bytes(uint32_t cap) { return align16(size_t(cap) * sizeof(E) + 32); }
    static size_t bytes(uint32_t P, uint32_t cap) {
        return align16(size_t(P) * 4) + align16(size_t(cap) * 2) + 2 * in_bytes(cap) +
               align16(size_t(cap) * sizeof(K)) + align16(size_t(cap) * sizeof(VT));
    }
    static uint32_t cap_for(uint32_t P, size_t budget) {
        const size_t fixed = align16(size_t(P) * 4) + 5 * 16 + 64;
        if (budget <= fixed) return 0;
        return uint32_t((budget - fixed) / (2 + 2 * sizeof(E) + sizeof(K) + sizeof(VT))) & ~7u;
    }
};

constexpr int kBuildBlock = 1024;

template <typename K, typename VT, typename OffT, bool POW2>
__global__ void __launch_bounds__(kBuildBlock, 1)
k_part_build(const typename EntryT<K, VT>::T* __restrict__ reorg,
             const OffT* __restrict__ part_start /* nparts + 1 partition offsets */,
             uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
             uint32_t pshift, uint32_t cap, OffT* __restrict__ offs, K* __restrict__ okeys,
             VT* __restrict__ ovals) {
    using PE = EntryT<K, VT>;
    using E = typename PE::T;
    using L = BuildLayout<K, VT>;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t P = 1u << pshift;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    uint16_t* lvs = reinterpret_cast<uint16_t*>(smem + align16(size_t(P) * 4));
    unsigned char* inb0 = reinterpret_cast<unsigned char*>(lvs) + align16(size_t(cap) * 2);
    unsigned char* inb1 = inb0 + L::in_bytes(cap);
    K* sk = reinterpret_cast<K*>(inb1 + L::in_bytes(cap));
    VT* sv = reinterpret_cast<VT*>(reinterpret_cast<unsigned char*>(sk) + align16(size_t(cap) * sizeof(K)));
    __shared__ uint64_t s_bar[2];
    __shared__ uint64_t s_s[2], s_e[2];
    __shared__ uint32_t s_ofs[2];
    __shared__ uint32_t s_warp[kBuildBlock / 32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t nwarps = kBuildBlock / 32;

    auto issue = [&](uint64_t p, int buf) {  // thread 0
        if (p >= nparts) return;
        const uint64_t s = part_start[p], e = part_start[p + 1];
        s_s[buf] = s;
        s_e[buf] = e;
        if (e - s <= cap) {
            fence_proxy_async();
            s_ofs[buf] = tma_load_span(buf ? inb1 : inb0, reorg + s, uint32_t((e - s) * sizeof(E)),
                                       &s_bar[buf]);
        }
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        issue(blockIdx.x, 0);
    }
    __syncthreads();
    uint32_t use[2] = {0, 0};
    for (uint64_t p = blockIdx.x, it = 0; p < nparts; p += gridDim.x, ++it) {
        const int buf = int(it & 1);
        const uint64_t s = s_s[buf], e = s_e[buf];
        const uint32_t cntp = uint32_t(e - s);
        const bool staged = uint64_t(cntp) <= cap;
        if (tid == 0) issue(p + gridDim.x, buf ^ 1);
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
        for (uint32_t j = tid; j < pv; j += kBuildBlock) cnt[j] = 0;
        if (staged) {
            mbar_wait(&s_bar[buf], use[buf] & 1);
            ++use[buf];
        }
        const E* src = staged ? reinterpret_cast<const E*>((buf ? inb1 : inb0) + s_ofs[buf])
                              : reorg + s;
        __syncthreads();
        // count: the second hash evaluation of V2's create_table pass (core.hpp:126-133)
        for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
            const uint32_t lv = uint32_t(hv<POW2>(PE::key(src[i]), seed, hk, nv) - vb);
            if (staged) lvs[i] = uint16_t(lv);
            atomicAdd(cnt + lv, 1u);
        }
        __syncthreads();
        // exclusive scan of cnt[0..pv): each thread owns a contiguous run
        const uint32_t per = (pv + kBuildBlock - 1) / kBuildBlock;
        const uint32_t j0 = min(pv, tid * per), j1 = min(pv, j0 + per);
        uint32_t run = 0;
        for (uint32_t j = j0; j < j1; ++j) run += cnt[j];
        uint32_t inc = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (int(lane) >= d) inc += y;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = s_warp[lane];
            uint32_t wi = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
                if (int(lane) >= d) wi += y;
            }
            s_warp[lane] = wi - w;
        }
        __syncthreads();
        uint32_t acc = s_warp[warp] + inc - run;
        for (uint32_t j = j0; j < j1; ++j) {
            const uint32_t c = cnt[j];
            cnt[j] = acc;  // exclusive start = placement cursor
            acc += c;
            offs[vb + j + 1] = OffT(s + acc);  // end(j) (contiguous per thread)
        }
        if (p == 0 && tid == 0) offs[0] = 0;
        __syncthreads();
        if (staged) {
            for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
                const E ent = src[i];
                const uint32_t pos = atomicAdd(cnt + lvs[i], 1u);
                sk[pos] = PE::key(ent);
                sv[pos] = PE::val(ent);
            }
            __syncthreads();
            for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
                okeys[s + i] = sk[i];
                ovals[s + i] = sv[i];
            }
        } else {
            for (uint32_t i = tid; i < cntp; i += kBuildBlock) {
                const E ent = src[i];
                const uint32_t lv = uint32_t(hv<POW2>(PE::key(ent), seed, hk, nv) - vb);
                const uint64_t pos = s + atomicAdd(cnt + lv, 1u);
                okeys[pos] = PE::key(ent);
                ovals[pos] = PE::val(ent);
            }
        }
        __syncthreads();
    }
    (void)nwarps;
}

template <typename K, typename VT, typename OffT, bool POW2>
cudaError_t build_v2_impl(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    using E = typename EntryT<K, VT>::T;
    const Divisor nv = make_divisor(t.nv);
    OffT* offs = static_cast<OffT*>(t.offs);
    cudaError_t e;
    if (t.n == 0) return cudaMemsetAsync(offs, 0, (t.nv + 1) * sizeof(OffT), s);

    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t budget = size_t(smem_optin) - 2048;
    // ~4096 entries per partition; K7 stages up to `cap` entries per partition
    const PartGeom g = make_geom(t.nv, t.n, a.partition_vertices, 4096.0);
    const uint32_t cap = std::min<uint32_t>(BuildLayout<K, VT>::cap_for(1u << g.pshift, budget),
                                            65535u);
    const size_t smem = BuildLayout<K, VT>::bytes(1u << g.pshift, cap);

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
    do {
        e = partition<K, VT, OffT, POW2>(static_cast<const K*>(a.keys),
                                         static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind,
                                         nv, g, part_start, pscratch, reorg, s, "k4_part_hist");
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
                                                   t.hash_kind, nv, g.pshift, cap, offs,
                                                   static_cast<K*>(t.keys),
                                                   static_cast<VT*>(t.vals)));
        e = cudaGetLastError();
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

#define HG_INST(K, VT, OffT)                                                                   \
    template cudaError_t build_v2_impl<K, VT, OffT, true>(const TableDesc&, const BuildArgs&, \
                                                          cudaStream_t);                       \
    template cudaError_t build_v2_impl<K, VT, OffT, false>(const TableDesc&, const BuildArgs&, \
                                                           cudaStream_t);
HG_INST(uint32_t, uint32_t, uint32_t)
HG_INST(uint32_t, uint32_t, uint64_t)
HG_INST(uint32_t, uint64_t, uint32_t)
HG_INST(uint32_t, uint64_t, uint64_t)
HG_INST(uint64_t, uint32_t, uint32_t)
HG_INST(uint64_t, uint32_t, uint64_t)
HG_INST(uint64_t, uint64_t, uint32_t)
HG_INST(uint64_t, uint64_t, uint64_t)
#undef HG_INST

}  // namespace hg
