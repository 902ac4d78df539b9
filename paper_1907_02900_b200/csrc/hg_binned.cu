// hg_binned.cu -- binned ("advanced", V2) HashGraph build on sm_100a.
//
// Replaces proj/include/hashgraph/core.hpp:183-230 (build_v2): keys are first
// scattered into contiguous vertex-range partitions ("bins",
// bin = v / bin_size, core.hpp:192-197), then every partition is built on
// chip. B200 mapping:
//   K4 k_part_hist    partition histogram            (core.hpp:195-203)
//   K5 scan           exclusive scan, in place       (core.hpp:205)
//   K6 k_part_scatter multisplit (key,val) -> reorg  (core.hpp:207-219)
//   K7 k_part_build   per partition, in shared memory: count, scan, place,
//                     then coalesced stores of offsets / keys / vals
//                     (core.hpp:221-223: create_table over the reorg array)
// The partition width P is a power of two sized so one partition's vertex
// counters plus its staged entries fit one CTA's shared memory; this is the
// B200 analogue of the reference's "bins sized to the LLC".
// The reference's bin_count only tunes CPU cache locality and never changes
// the output (hashgraph_bench.cpp:471), so P is chosen for the hardware.
#include <algorithm>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_scan.cuh"

namespace hg {

int num_sms();

template <typename K, typename VT>
struct PackedEntry;
template <>
struct PackedEntry<uint32_t, uint32_t> {
    using T = uint2;
    __device__ static T pack(uint32_t k, uint32_t v) { return make_uint2(k, v); }
    __device__ static uint32_t key(const T& e) { return e.x; }
    __device__ static uint32_t val(const T& e) { return e.y; }
};
template <typename K, typename VT>
struct PackedEntry {
    using T = ulonglong2;
    __device__ static T pack(K k, VT v) { return make_ulonglong2(k, v); }
    __device__ static K key(const T& e) { return K(e.x); }
    __device__ static VT val(const T& e) { return VT(e.y); }
};

template <typename K, typename F>
__device__ __forceinline__ void for_each_key2(const K* __restrict__ keys, uint64_t n, F&& f) {
    constexpr int VEC = 16 / sizeof(K);
    using V = typename std::conditional<sizeof(K) == 4, uint4, ulonglong2>::type;
    const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t head = ((16 - (reinterpret_cast<uintptr_t>(keys) & 15)) & 15) / sizeof(K);
    if (head > n) head = n;
    if (gtid < head) f(gtid, keys[gtid]);
    const uint64_t nvec = (n - head) / VEC;
    const V* body = reinterpret_cast<const V*>(keys + head);
    uint64_t q = gtid;
    for (; q + stride < nvec; q += 2 * stride) {
        const V a = __ldcs(body + q);
        const V b = __ldcs(body + q + stride);
        const K* ka = reinterpret_cast<const K*>(&a);
        const K* kb = reinterpret_cast<const K*>(&b);
#pragma unroll
        for (int k = 0; k < VEC; ++k) f(head + q * VEC + k, ka[k]);
#pragma unroll
        for (int k = 0; k < VEC; ++k) f(head + (q + stride) * VEC + k, kb[k]);
    }
    if (q < nvec) {
        const V a = __ldcs(body + q);
        const K* ka = reinterpret_cast<const K*>(&a);
#pragma unroll
        for (int k = 0; k < VEC; ++k) f(head + q * VEC + k, ka[k]);
    }
    const uint64_t done = head + nvec * VEC;
    if (gtid < n - done) f(done + gtid, keys[done + gtid]);
}

template <bool POW2>
__device__ __forceinline__ uint64_t vtx(uint64_t key, uint64_t seed, int hk, const Divisor& nv) {
    return hk == kHashIdentity ? vertex_of<kHashIdentity, POW2>(key, seed, nv)
                               : vertex_of<kHashMix64, POW2>(key, seed, nv);
}

// ---------------------------------------------------------------- K4

constexpr int kSmemHistMax = 8192;  // partitions histogrammed in shared memory

template <typename K, typename OffT, bool POW2>
__global__ void __launch_bounds__(256)
k_part_hist(const K* __restrict__ keys, uint64_t n, uint64_t seed, int hk, Divisor nv,
            uint32_t pshift, uint64_t nparts, OffT* __restrict__ hist) {
    __shared__ uint32_t sh[kSmemHistMax];
    const bool priv = nparts <= kSmemHistMax;
    if (priv) {
        for (uint32_t i = threadIdx.x; i < nparts; i += blockDim.x) sh[i] = 0;
        __syncthreads();
    }
    for_each_key2(keys, n, [&](uint64_t, K key) {
        const uint64_t p = vtx<POW2>(key, seed, hk, nv) >> pshift;
        if (priv) {
            atomicAdd(sh + p, 1u);
        } else {
            aggregated_count<true>(hist + p, __activemask(), p);
        }
    });
    if (priv) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nparts; i += blockDim.x)
            if (sh[i]) red_add(hist + i, OffT(sh[i]));
    }
}

// ---------------------------------------------------------------- K6

template <typename K, typename VT, typename OffT, bool POW2>
__global__ void __launch_bounds__(256)
k_part_scatter(const K* __restrict__ keys, const VT* __restrict__ vals, uint64_t n,
               uint64_t seed, int hk, Divisor nv, uint32_t pshift, OffT* __restrict__ cursor,
               typename PackedEntry<K, VT>::T* __restrict__ reorg) {
    using PE = PackedEntry<K, VT>;
    for_each_key2(keys, n, [&](uint64_t i, K key) {
        const uint64_t p = vtx<POW2>(key, seed, hk, nv) >> pshift;
        const OffT pos = aggregated_ticket<true>(cursor + p, __activemask(), p);
        reorg[pos] = PE::pack(key, vals ? vals[i] : VT(i));
    });
}

// ---------------------------------------------------------------- K7

// Shared-memory layout per CTA (each region 16-byte aligned):
//   cnt[P] u32 | lv[cap] u16 | skeys[cap] K | svals[cap] VT
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename K, typename VT>
__host__ __device__ constexpr size_t part_smem_bytes(uint32_t P, uint32_t cap) {
    return align16(size_t(P) * 4) + align16(size_t(cap) * 2) + align16(size_t(cap) * sizeof(K)) +
           align16(size_t(cap) * sizeof(VT));
}

template <typename K, typename VT, typename OffT, bool POW2>
__global__ void __launch_bounds__(512)
k_part_build(const typename PackedEntry<K, VT>::T* __restrict__ reorg,
             const OffT* __restrict__ part_end /* part_end[p] = end of partition p */,
             uint64_t nparts, uint64_t nv_total, uint64_t seed, int hk, Divisor nv,
             uint32_t pshift, uint32_t cap, OffT* __restrict__ offs, K* __restrict__ okeys,
             VT* __restrict__ ovals, uint32_t* ticket) {
    using PE = PackedEntry<K, VT>;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = 1u << pshift;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
    uint16_t* lvs = reinterpret_cast<uint16_t*>(smem + align16(size_t(P) * 4));
    K* sk = reinterpret_cast<K*>(smem + align16(size_t(P) * 4) + align16(size_t(cap) * 2));
    VT* sv = reinterpret_cast<VT*>(reinterpret_cast<unsigned char*>(sk) + align16(size_t(cap) * sizeof(K)));
    __shared__ uint32_t s_part;
    __shared__ uint32_t s_warp[16];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

    while (true) {
        if (tid == 0) s_part = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t p = s_part;
        if (p >= nparts) break;
        const uint64_t s = p == 0 ? 0 : uint64_t(part_end[p - 1]);
        const uint64_t e = part_end[p];
        const uint64_t cntp = e - s;
        const uint64_t vb = p << pshift;
        const uint32_t pv = uint32_t(nv_total - vb < P ? nv_total - vb : uint64_t(P));
        const bool staged = cntp <= cap;

        for (uint32_t j = tid; j < pv; j += blockDim.x) cnt[j] = 0;
        __syncthreads();
        // count (second hash evaluation of V2's create_table pass, core.hpp:126-133)
        for (uint64_t i = tid; i < cntp; i += blockDim.x) {
            const auto ent = reorg[s + i];
            const uint32_t lv = uint32_t(vtx<POW2>(PE::key(ent), seed, hk, nv) - vb);
            if (staged) lvs[i] = uint16_t(lv);
            atomicAdd(cnt + lv, 1u);
        }
        __syncthreads();
        // exclusive scan of cnt[0..pv) in shared memory; offs[vb+j+1] = s + inclusive(j)
        const uint32_t per = (pv + blockDim.x - 1) / blockDim.x;
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
            const uint32_t w = lane < nwarps ? s_warp[lane] : 0;
            uint32_t wi = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
                if (int(lane) >= d) wi += y;
            }
            if (lane < nwarps) s_warp[lane] = wi - w;
        }
        __syncthreads();
        uint32_t acc = s_warp[warp] + inc - run;
        for (uint32_t j = j0; j < j1; ++j) {
            const uint32_t c = cnt[j];
            cnt[j] = acc;  // exclusive start = placement cursor
            acc += c;
        }
        __syncthreads();
        // offsets: offs[vb + j + 1] = s + end(j), coalesced
        for (uint32_t j = tid; j < pv; j += blockDim.x) {
            const uint32_t endj = (j + 1 < pv) ? cnt[j + 1] : uint32_t(cntp);
            offs[vb + j + 1] = OffT(s + endj);
        }
        if (p == 0 && tid == 0) offs[0] = 0;
        __syncthreads();
        // place
        if (staged) {
            for (uint64_t i = tid; i < cntp; i += blockDim.x) {
                const auto ent = reorg[s + i];
                const uint32_t pos = atomicAdd(cnt + lvs[i], 1u);
                sk[pos] = PE::key(ent);
                sv[pos] = PE::val(ent);
            }
            __syncthreads();
            for (uint64_t i = tid; i < cntp; i += blockDim.x) {
                okeys[s + i] = sk[i];
                ovals[s + i] = sv[i];
            }
        } else {
            for (uint64_t i = tid; i < cntp; i += blockDim.x) {
                const auto ent = reorg[s + i];
                const uint32_t lv = uint32_t(vtx<POW2>(PE::key(ent), seed, hk, nv) - vb);
                const uint64_t pos = s + atomicAdd(cnt + lv, 1u);
                okeys[pos] = PE::key(ent);
                ovals[pos] = PE::val(ent);
            }
        }
        __syncthreads();
    }
}

template <typename K, typename VT, typename OffT, bool POW2>
cudaError_t build_v2_impl(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    using E = typename PackedEntry<K, VT>::T;
    const Divisor nv = make_divisor(t.nv);
    OffT* offs = static_cast<OffT*>(t.offs);
    cudaError_t e;
    if (t.n == 0) return cudaMemsetAsync(offs, 0, (t.nv + 1) * sizeof(OffT), s);

    // Partition width P = 2^pshift <= 2^16 (u16 local vertex ids). Auto: the
    // widest P whose expected entry count (N*P/V) stays within ~60% of the
    // shared-memory staging capacity, so almost every partition is staged.
    int dev = 0;
    cudaGetDevice(&dev);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t budget = std::min<size_t>(size_t(smem_optin) - 1024, 112 * 1024);
    auto cap_for = [&](uint32_t ps) -> uint32_t {
        const size_t fixed = align16((size_t(1) << ps) * 4) + 64;
        if (budget <= fixed) return 0;
        return uint32_t((budget - fixed) / (2 + sizeof(K) + sizeof(VT))) & ~7u;
    };
    uint32_t pshift = 12;
    if (a.partition_vertices) {
        pshift = 0;
        while ((uint64_t(1) << (pshift + 1)) <= a.partition_vertices && pshift < 16) ++pshift;
    } else {
        const double per_vertex = double(t.n) / double(t.nv);
        while (pshift > 5 && per_vertex * double(1u << pshift) > 0.6 * cap_for(pshift)) --pshift;
        while (pshift < 14 && per_vertex * double(2u << pshift) <= 0.6 * cap_for(pshift + 1))
            ++pshift;
    }
    while (pshift > 0 && (uint64_t(1) << (pshift - 1)) >= t.nv) --pshift;
    const uint32_t P = 1u << pshift;
    const uint64_t nparts = (t.nv + P - 1) >> pshift;
    const uint32_t cap = cap_for(pshift);
    const size_t smem = part_smem_bytes<K, VT>(P, cap);

    // scratch: part[nparts+1] | scan scratch | reorg[n] | ticket
    const size_t part_bytes = ((nparts + 1) * sizeof(OffT) + 255) & ~size_t(255);
    const size_t scan_bytes = (scan_scratch_bytes(nparts) + 255) & ~size_t(255);
    const size_t reorg_bytes = (t.n * sizeof(E) + 255) & ~size_t(255);
    char* scratch = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                             part_bytes + scan_bytes + reorg_bytes + 256, s)) != cudaSuccess)
        return e;
    OffT* part = reinterpret_cast<OffT*>(scratch);
    void* scan_scr = scratch + part_bytes;
    E* reorg = reinterpret_cast<E*>(scratch + part_bytes + scan_bytes);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch + part_bytes + scan_bytes + reorg_bytes);
    const K* keys = static_cast<const K*>(a.keys);

    do {
        if ((e = cudaMemsetAsync(part, 0, (nparts + 1) * sizeof(OffT), s)) != cudaSuccess) break;
        if ((e = cudaMemsetAsync(ticket, 0, 4, s)) != cudaSuccess) break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_part_hist<K, OffT, POW2>, 256, 0);
        unsigned g = unsigned(std::max(1, per_sm) * num_sms());
        g = unsigned(std::min<uint64_t>(g, (t.n + 255) / 256));
        HG_LAUNCH("k4_part_hist", s, k_part_hist<K, OffT, POW2><<<g, 256, 0, s>>>(keys, t.n, t.seed, t.hash_kind, nv, pshift,
                                                     nparts, part + 1));
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        if ((e = launch_scan<OffT, OffT>(part + 1, part + 1, nparts, scan_scr, nullptr, s, "k5_part_scan")) !=
            cudaSuccess)
            break;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_part_scatter<K, VT, OffT, POW2>,
                                                      256, 0);
        g = unsigned(std::max(1, per_sm) * num_sms());
        g = unsigned(std::min<uint64_t>(g, (t.n + 255) / 256));
        HG_LAUNCH("k6_part_scatter", s, k_part_scatter<K, VT, OffT, POW2><<<g, 256, 0, s>>>(
            keys, static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind, nv, pshift, part + 1,
            reorg));
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        // after K6, part[p+1] == end(p)
        auto kb = k_part_build<K, VT, OffT, POW2>;
        if ((e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem))) != cudaSuccess)
            break;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb, 512, smem);
        g = unsigned(std::min<uint64_t>(uint64_t(std::max(1, per_sm)) * num_sms(), nparts));
        HG_LAUNCH("k7_part_build", s, kb<<<g, 512, smem, s>>>(reorg, part + 1, nparts, t.nv, t.seed, t.hash_kind, nv, pshift,
                                cap, offs, static_cast<K*>(t.keys), static_cast<VT*>(t.vals),
                                ticket));
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
