// hg_shard.cu -- hash-range routing for the multi-GPU (sharded) table.
//
// The reference partitions its vertex range only for cache locality
// (core.hpp:192-197, bin = v / ceil(V / bins)); with G GPUs the same formula
// at bins = G picks the owner GPU: owner(v) = v / ceil(V/G).
// K11 (this file) groups a GPU's keys by owner so that one NCCL all-to-all
// (torch.distributed over NVLink) moves every key to the GPU that builds /
// probes its vertex range:
//   k_route_hist     per-owner counts (shared-memory histogram, G <= 256)
//   scan             owner starts
//   k_route_scatter  per 4096-key tile: shared-memory rank by owner, one
//                    global atomic per (tile, owner) reserving a run, then
//                    the tile is staged owner-sorted and written as coalesced
//                    runs into SoA keys[] / vals[] send buffers.
#include <algorithm>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_radix.cuh"
#include "hg_scan.cuh"

namespace hg {

constexpr int kRouteBlock = 512;
constexpr int kRouteItems = 4;
constexpr int kRouteTile = kRouteBlock * kRouteItems;

// Owner of an item: its key's hash range (build / probe routing: owner =
// ((h(key) mod V) - vertex_base) / span) or its value's range (match pairs
// returned to the rank holding the probe: owner = value / span).
template <int POW2>
struct OwnHash {
    uint64_t seed;
    Divisor gv, span;
    __device__ __forceinline__ uint32_t operator()(uint64_t key, uint64_t) const {
        return uint32_t(div_of<false>(vhash<POW2>(key, seed, gv), span));
    }
};
struct OwnVal {
    Divisor span;
    __device__ __forceinline__ uint32_t operator()(uint64_t, uint64_t val) const {
        return uint32_t(div_of<false>(val, span));
    }
};

template <typename K, typename VT, typename Own>
__global__ void __launch_bounds__(kRouteBlock)
k_route_hist(const K* __restrict__ keys, const VT* __restrict__ vals, uint64_t n, uint64_t val_base,
             Own own, uint32_t shards, unsigned long long* __restrict__ counts) {
    __shared__ uint32_t sh[256];
    for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(sh + own(uint64_t(keys[i]), vals ? uint64_t(vals[i]) : val_base + i), 1u);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < shards; i += blockDim.x)
        if (sh[i]) atomicAdd(counts + i, (unsigned long long)sh[i]);
}

// REC: owner-grouped AoS records {key, value} (EntryT<K, VT>::T, the binned
// build's entry type: one buffer, one all-to-all) instead of SoA keys / values.
template <typename K, typename VT, typename Own, bool REC>
__global__ void __launch_bounds__(kRouteBlock)
k_route_scatter(const K* __restrict__ keys, const VT* __restrict__ vals, uint64_t n,
                uint64_t val_base, Own own, uint32_t shards, unsigned long long* __restrict__ cursor,
                K* __restrict__ okeys, VT* __restrict__ ovals,
                typename EntryT<K, VT>::T* __restrict__ orec) {
    __shared__ K s_k[kRouteTile];
    __shared__ VT s_v[kRouteTile];
    __shared__ uint8_t s_o[kRouteTile];
    __shared__ uint32_t s_cnt[256], s_off[256];
    __shared__ unsigned long long s_gbo[256];
    const uint32_t tid = threadIdx.x;
    const uint64_t ntiles = (n + kRouteTile - 1) / kRouteTile;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tile * kRouteTile;
        const uint32_t cnt = uint32_t(n - t0 < kRouteTile ? n - t0 : kRouteTile);
        for (uint32_t d = tid; d < shards; d += kRouteBlock) s_cnt[d] = 0;
        __syncthreads();
        K kk[kRouteItems];
        VT vv[kRouteItems];
        uint32_t orank[kRouteItems];
#pragma unroll
        for (int k = 0; k < kRouteItems; ++k) {
            const uint32_t j = tid + k * kRouteBlock;
            if (j < cnt) {
                kk[k] = keys[t0 + j];
                vv[k] = vals ? vals[t0 + j] : VT(val_base + t0 + j);
                const uint32_t o = own(uint64_t(kk[k]), uint64_t(vv[k]));
                orank[k] = (o << 16) | atomicAdd(s_cnt + o, 1u);
            }
        }
        __syncthreads();
        if (tid < 32) {
            // exclusive scan of <= 256 shard counts by one warp
            uint32_t c[8], run = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t d = tid * 8 + q;
                c[q] = d < shards ? s_cnt[d] : 0;
                run += c[q];
            }
            uint32_t inc = run;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (int(tid) >= d) inc += y;
            }
            uint32_t acc = inc - run;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t d = tid * 8 + q;
                if (d < shards) {
                    s_off[d] = acc;
                    if (c[q]) s_gbo[d] = atomicAdd(cursor + d, (unsigned long long)c[q]) - acc;
                }
                acc += c[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kRouteItems; ++k) {
            const uint32_t j = tid + k * kRouteBlock;
            if (j < cnt) {
                const uint32_t o = orank[k] >> 16;
                const uint32_t slot = s_off[o] + (orank[k] & 0xFFFFu);
                s_k[slot] = kk[k];
                s_v[slot] = vv[k];
                s_o[slot] = uint8_t(o);
            }
        }
        __syncthreads();
        for (uint32_t j = tid; j < cnt; j += kRouteBlock) {
            const uint64_t dst = s_gbo[s_o[j]] + j;
            if constexpr (REC) {
                orec[dst] = EntryT<K, VT>::make(s_k[j], s_v[j]);
            } else {
                okeys[dst] = s_k[j];
                if (ovals) ovals[dst] = s_v[j];  // keys-only routing (count-only probes)
            }
        }
        __syncthreads();
    }
}

template <typename K, typename VT, typename Own, bool REC>
static cudaError_t route_impl(const void* keys, const void* vals, uint64_t n, uint64_t val_base,
                              const Own& own, uint32_t G, void* out_keys, void* out_vals,
                              void* out_rec, uint64_t* shard_counts, cudaStream_t s) {
    auto* counts = reinterpret_cast<unsigned long long*>(shard_counts);
    cudaError_t e = cudaMemsetAsync(counts, 0, G * 8, s);
    if (e != cudaSuccess || n == 0) return e;
    const int sms = num_sms();
    const unsigned gh = unsigned(std::min<uint64_t>((n + kRouteBlock - 1) / kRouteBlock, uint64_t(sms) * 4));
    HG_LAUNCH("k11_route_hist", s,
              (k_route_hist<K, VT, Own><<<gh, kRouteBlock, 0, s>>>(
                  static_cast<const K*>(keys), static_cast<const VT*>(vals), n, val_base, own, G,
                  counts)));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // cursor[d] = exclusive prefix of counts
    unsigned long long* cursor = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&cursor), (G + 1) * 8 + 256 +
                                                                  scan_scratch_bytes(G), s)) != cudaSuccess)
        return e;
    void* scr = reinterpret_cast<char*>(cursor) + ((G + 1) * 8 + 255) / 256 * 256;
    e = launch_scan<unsigned long long, unsigned long long>(counts, cursor, G, scr, nullptr, s,
                                                            "route_scan");
    if (e == cudaSuccess) {
        const uint64_t tiles = (n + kRouteTile - 1) / kRouteTile;
        const unsigned gs = unsigned(std::min<uint64_t>(tiles, uint64_t(sms) * 2));
        HG_LAUNCH("k11_route_scatter", s,
                  (k_route_scatter<K, VT, Own, REC><<<gs, kRouteBlock, 0, s>>>(
                      static_cast<const K*>(keys), static_cast<const VT*>(vals), n, val_base, own, G,
                      cursor, static_cast<K*>(out_keys), static_cast<VT*>(out_vals),
                      static_cast<typename EntryT<K, VT>::T*>(out_rec))));
        e = cudaGetLastError();
    }
    cudaFreeAsync(cursor, s);
    return e;
}

template <typename OffT>
__global__ void k_split_counts(const OffT* __restrict__ start, uint32_t G,
                               unsigned long long* __restrict__ counts) {
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) counts[g] = start[g + 1] - start[g];
}

// Power-of-two spans (owner = local vertex >> log2(span): V and G powers of
// two, e.g. the weak-scaling C2 and strong-scaling C5 configs) route with one
// pass of the partition machinery (hg_radix.cuh: TMA-staged tiles, shared-
// memory ranking, coalesced runs) instead of K11: records {key, val_base + i}
// or bare keys grouped by owner, counts from the owner starts.
template <typename K, typename VT, int HM>
static cudaError_t route_split(const void* keys, uint64_t n, uint64_t val_base, uint64_t seed,
                               int hash_kind, const Divisor& gv, uint32_t sshift, uint32_t G,
                               void* out, uint64_t* shard_counts, cudaStream_t s) {
    PartGeom g;
    g.pshift = sshift;
    g.nparts = G;
    g.bits = g.b1 = ceil_log2(G);
    g.b2 = 0;
    const size_t sbytes = ((G + 1) * 8 + 255) & ~size_t(255);
    const size_t pbytes = PartitionScratch<K, VT, uint64_t>::bytes(g, n);
    char* scr = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scr), sbytes + pbytes, s);
    if (e != cudaSuccess) return e;
    static const char* const kNames[3] = {"k11_route_hist", "k11_route_split", "-"};
    uint64_t* start = reinterpret_cast<uint64_t*>(scr);
    e = partition<K, VT, uint64_t, HM>(static_cast<const K*>(keys), static_cast<const VT*>(nullptr),
                                       n, seed, hash_kind, gv, g, start, scr + sbytes,
                                       static_cast<typename EntryT<K, VT>::T*>(out), s, kNames,
                                       nullptr, val_base);
    if (e == cudaSuccess) {
        k_split_counts<uint64_t><<<1, 256, 0, s>>>(start, G,
                                                   reinterpret_cast<unsigned long long*>(shard_counts));
        e = cudaGetLastError();
    }
    cudaFreeAsync(scr, s);
    return e;
}

template <typename K, typename VT>
static cudaError_t route_hash_typed(const void* keys, const void* vals, uint64_t n, uint64_t val_base,
                                    uint64_t seed, int hash_kind, uint64_t V, uint64_t vbase,
                                    uint64_t nloc, uint64_t span, uint32_t G, void* out_keys,
                                    void* out_vals, void* out_rec, uint64_t* shard_counts,
                                    cudaStream_t s) {
    const Divisor gv = make_divisor(V, vbase);  // (h mod V) - vbase
    const uint64_t spv = span ? span : (nloc + G - 1) / G;
    const Divisor sp = make_divisor(spv);
    const bool split = sp.pow2 && vals == nullptr && (out_rec || out_vals == nullptr) && n &&
                       G <= 256 && (uint64_t(G) << sp.shift) >= nloc;
    return dispatch_hash_mode(hash_mode(V, hash_kind), [&](auto m) {
        constexpr int HM = decltype(m)::value;
        if (split) {
            if (out_rec)
                return route_split<K, VT, HM>(keys, n, val_base, seed, hash_kind, gv, sp.shift, G,
                                              out_rec, shard_counts, s);
            return route_split<K, void, HM>(keys, n, 0, seed, hash_kind, gv, sp.shift, G, out_keys,
                                            shard_counts, s);
        }
        const OwnHash<HM> own{seed, gv, sp};
        return out_rec ? route_impl<K, VT, OwnHash<HM>, true>(keys, vals, n, val_base, own, G, nullptr,
                                                             nullptr, out_rec, shard_counts, s)
                       : route_impl<K, VT, OwnHash<HM>, false>(keys, vals, n, val_base, own, G,
                                                              out_keys, out_vals, nullptr,
                                                              shard_counts, s);
    });
}

cudaError_t route_keys(const void* keys, int key_bytes, const void* vals, int val_bytes,
                       uint64_t n, uint64_t val_base, uint64_t seed, int hash_kind,
                       uint64_t global_vertices, uint64_t vertex_base, uint64_t local_vertices,
                       uint64_t span, uint32_t shards, void* out_keys, void* out_vals,
                       uint64_t* shard_counts, cudaStream_t s, void* out_records) {
#define HG_ROUTE(K, VT)                                                                          \
    return route_hash_typed<K, VT>(keys, vals, n, val_base, seed, hash_kind, global_vertices,     \
                                   vertex_base, local_vertices, span, shards, out_keys, out_vals, \
                                   out_records, shard_counts, s)
    if (key_bytes == 4) {
        if (val_bytes == 4) HG_ROUTE(uint32_t, uint32_t);
        HG_ROUTE(uint32_t, uint64_t);
    }
    if (val_bytes == 4) HG_ROUTE(uint64_t, uint32_t);
    HG_ROUTE(uint64_t, uint64_t);
#undef HG_ROUTE
}

cudaError_t route_pairs(const void* left, const void* right, int pair_bytes, uint64_t n,
                        uint64_t span, uint32_t shards, void* out_records, uint64_t* shard_counts,
                        cudaStream_t s) {
    const OwnVal own{make_divisor(span)};
    if (pair_bytes == 4)
        return route_impl<uint32_t, uint32_t, OwnVal, true>(left, right, n, 0, own, shards, nullptr,
                                                           nullptr, out_records, shard_counts, s);
    return route_impl<uint64_t, uint64_t, OwnVal, true>(left, right, n, 0, own, shards, nullptr,
                                                       nullptr, out_records, shard_counts, s);
}

}  // namespace hg
