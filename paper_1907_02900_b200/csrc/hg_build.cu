// hg_build.cu -- HashGraph table construction on sm_100a.
//
// Simple build (V1), replacing proj/include/hashgraph/core.hpp:120-177
// (detail::create_table + build_v1):
//   K1 k_hash_count  counts[h(k)]++            (core.hpp:126-133)
//   K2 scan          exclusive scan, in place  (core.hpp:135 -> parallel.hpp:141-192)
//   K3 k_scatter     pos = cursor[h(k)]++      (core.hpp:137-150)
// One (V+1)-entry array serves as counter, offsets and placement cursor:
// K1 counts vertex v into offs[v+1]; the in-place exclusive scan turns
// offs[v+1] into start(v); K3's fetch-add on offs[v+1] hands out slots
// start(v)..end(v)-1 and leaves offs[v+1] == end(v) == start(v+1), i.e. the
// finished CSR offsets (offs[0] stays 0). This drops the reference's separate
// counter zeroing (core.hpp:137) and offsets gather from the placement pass.
//
// Binned build (V2, core.hpp:183-230) lives in hg_binned.cu. The optional
// "stable" post-pass (k_seg_sort_*) orders every segment by input index,
// which is exactly the reference's ExecMode::sequential layout
// (core.hpp:115-119: sequential placement keeps source order).
#include <algorithm>
#include <cstdio>

#include "hg_common.cuh"
#include "hg_internal.h"
#include "hg_radix.cuh"
#include "hg_scan.cuh"

namespace hg {

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// A table (or scratch) of more than 1/8 of device memory: the stream is
// drained first, so that the pool serves it from the blocks freed by earlier
// work on the stream (e.g. the previous table of a build / probe loop)
// instead of growing while those frees are still pending -- near the memory
// limit that growth stalls for hundreds of ms (measured at C5, 2^32 keys on
// one GPU: 1.2 s steps instead of 207 ms).
bool huge_allocation(uint64_t bytes) {
    static uint64_t total = 0;
    if (!total) {
        size_t f = 0, t = 0;
        cudaMemGetInfo(&f, &t);
        total = t ? t : (uint64_t(180) << 30);
    }
    return bytes > total / 8;
}

size_t smem_optin() {
    static int bytes = 0;
    if (!bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (bytes <= 0) bytes = 227 * 1024;
    }
    return size_t(bytes);
}

template <typename Kern>
static unsigned persistent_grid(Kern k, int block, size_t smem, uint64_t work_items) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t cap = uint64_t(per_sm) * num_sms();
    const uint64_t need = (work_items + block - 1) / block;
    return unsigned(std::max<uint64_t>(1, std::min(cap, need)));
}

// Grid-stride loop over keys with 16-byte vector loads (two in flight per
// thread), calling f(i, key) for every key. Lanes of a warp stay converged
// inside f except in the unaligned head / ragged tail.
template <typename K, typename F>
__device__ __forceinline__ void for_each_key(const K* __restrict__ keys, uint64_t n, F&& f) {
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

// ---------------------------------------------------------------- K1 / K3

template <typename K, typename OffT, int POW2>
__global__ void __launch_bounds__(256)
k_hash_count(const K* __restrict__ keys, uint64_t n, uint64_t seed, int hk, Divisor nv,
             OffT* __restrict__ cnt, int aggregate) {
    constexpr bool V32 = sizeof(OffT) == 4;
    for_each_key(keys, n, [&](uint64_t, K key) {
        const uint64_t v = vhash<POW2>(key, seed, nv);
        if (aggregate) {
            aggregated_count<V32>(cnt + v, __activemask(), v);
        } else {
            red_add(cnt + v, OffT(1));
        }
    });
}

template <typename K, typename VT, typename OffT, int POW2>
__global__ void __launch_bounds__(256)
k_scatter(const K* __restrict__ keys, const VT* __restrict__ vals, uint64_t n, uint64_t seed,
          int hk, Divisor nv, OffT* __restrict__ cursor, K* __restrict__ okeys,
          VT* __restrict__ ovals, int aggregate) {
    constexpr bool V32 = sizeof(OffT) == 4;
    for_each_key(keys, n, [&](uint64_t i, K key) {
        const uint64_t v = vhash<POW2>(key, seed, nv);
        OffT pos;
        if (aggregate) {
            pos = aggregated_ticket<V32>(cursor + v, __activemask(), v);
        } else {
            pos = atom_add(cursor + v, OffT(1));
        }
        okeys[pos] = key;
        ovals[pos] = vals ? vals[i] : VT(i);
    });
}

// --------------------------------------------------- stable segment order
// Sequential-mode layout (core.hpp:115-119): every segment in ascending input
// index. Short segments: one thread, insertion sort. Long segments: one CTA,
// an ascending-only bitonic network (valid for any length: the implicit +inf
// padding never moves, so comparators touching it are skipped).

constexpr int kSmallSeg = 16;
constexpr int kSmemSeg = 2048;

template <typename K, typename VT, typename OffT>
__global__ void __launch_bounds__(256)
k_seg_sort_small(const OffT* __restrict__ offs, uint64_t nv, K* keys, VT* vals,
                 uint64_t* big_list, unsigned long long* big_n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv; v += stride) {
        const uint64_t b = offs[v], e = offs[v + 1];
        const uint64_t len = e - b;
        if (len <= 1) continue;
        if (len > kSmallSeg) {
            big_list[atomicAdd(big_n, 1ull)] = v;
            continue;
        }
        K kk[kSmallSeg];
        VT vv[kSmallSeg];
        for (uint32_t t = 0; t < len; ++t) {
            kk[t] = keys[b + t];
            vv[t] = vals[b + t];
        }
        for (uint32_t t = 1; t < len; ++t) {
            const K ck = kk[t];
            const VT cv = vv[t];
            int u = int(t) - 1;
            while (u >= 0 && vv[u] > cv) {
                kk[u + 1] = kk[u];
                vv[u + 1] = vv[u];
                --u;
            }
            kk[u + 1] = ck;
            vv[u + 1] = cv;
        }
        for (uint32_t t = 0; t < len; ++t) {
            keys[b + t] = kk[t];
            vals[b + t] = vv[t];
        }
    }
}

template <typename K, typename VT>
__device__ __forceinline__ void cmp_swap(K* k, VT* v, uint64_t i, uint64_t j) {
    if (v[j] < v[i]) {
        const VT tv = v[i];
        v[i] = v[j];
        v[j] = tv;
        const K tk = k[i];
        k[i] = k[j];
        k[j] = tk;
    }
}

template <typename K, typename VT>
__device__ void block_bitonic_by_val(K* k, VT* v, uint64_t len) {
    uint64_t p2 = 1;
    while (p2 < len) p2 <<= 1;
    const uint64_t pairs = p2 / 2;
    for (uint64_t size = 2; size <= p2; size <<= 1) {
        const uint64_t h = size / 2;
        for (uint64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
            const uint64_t blk = t / h, off = t % h;
            const uint64_t i = blk * size + off, j = blk * size + size - 1 - off;
            if (j < len) cmp_swap(k, v, i, j);
        }
        __syncthreads();
        for (uint64_t half = h / 2; half >= 1; half >>= 1) {
            for (uint64_t t = threadIdx.x; t < pairs; t += blockDim.x) {
                const uint64_t blk = t / half, off = t % half;
                const uint64_t i = blk * 2 * half + off, j = i + half;
                if (j < len) cmp_swap(k, v, i, j);
            }
            __syncthreads();
        }
    }
}

template <typename K, typename VT, typename OffT>
__global__ void __launch_bounds__(512)
k_seg_sort_big(const OffT* __restrict__ offs, K* keys, VT* vals, const uint64_t* list,
               const unsigned long long* list_n) {
    __shared__ K sk[kSmemSeg];
    __shared__ VT sv[kSmemSeg];
    const uint64_t cnt = *list_n;
    for (uint64_t it = blockIdx.x; it < cnt; it += gridDim.x) {
        const uint64_t v = list[it];
        const uint64_t b = offs[v], len = uint64_t(offs[v + 1]) - b;
        if (len <= kSmemSeg) {
            for (uint64_t t = threadIdx.x; t < len; t += blockDim.x) {
                sk[t] = keys[b + t];
                sv[t] = vals[b + t];
            }
            __syncthreads();
            block_bitonic_by_val(sk, sv, len);
            for (uint64_t t = threadIdx.x; t < len; t += blockDim.x) {
                keys[b + t] = sk[t];
                vals[b + t] = sv[t];
            }
            __syncthreads();
        } else {
            block_bitonic_by_val(keys + b, vals + b, len);
            __threadfence_block();
            __syncthreads();
        }
    }
}

template <typename K, typename VT, typename OffT>
static cudaError_t stable_order(const TableDesc& t, cudaStream_t s) {
    if (t.n < 2) return cudaSuccess;
    const uint64_t cap = t.n / (kSmallSeg + 1) + 1;
    void* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, (cap + 1) * sizeof(uint64_t), s);
    if (e != cudaSuccess) return e;
    uint64_t* list = static_cast<uint64_t*>(scratch);
    auto* list_n = reinterpret_cast<unsigned long long*>(list + cap);
    cudaMemsetAsync(list_n, 0, 8, s);
    const unsigned g1 = persistent_grid(k_seg_sort_small<K, VT, OffT>, 256, 0, t.nv);
    HG_LAUNCH("seg_sort_small", s, k_seg_sort_small<K, VT, OffT><<<g1, 256, 0, s>>>(static_cast<const OffT*>(t.offs), t.nv,
                                                    static_cast<K*>(t.keys),
                                                    static_cast<VT*>(t.vals), list, list_n));
    HG_LAUNCH("seg_sort_big", s, k_seg_sort_big<K, VT, OffT><<<num_sms() * 2, 512, 0, s>>>(
        static_cast<const OffT*>(t.offs), static_cast<K*>(t.keys), static_cast<VT*>(t.vals), list,
        list_n));
    e = cudaGetLastError();
    cudaFreeAsync(scratch, s);
    return e;
}

// ------------------------------------------------------------------ V1

template <typename K, typename VT, typename OffT, int POW2>
static cudaError_t build_v1_impl(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    const Divisor nv = make_divisor(global_nv(t), t.vbase);
    OffT* offs = static_cast<OffT*>(t.offs);
    cudaError_t e = cudaMemsetAsync(offs, 0, (t.nv + 1) * sizeof(OffT), s);
    if (e != cudaSuccess || t.n == 0) return e;
    const K* keys = static_cast<const K*>(a.keys);
    const unsigned g1 = persistent_grid(k_hash_count<K, OffT, POW2>, 256, 0, t.n);
    HG_LAUNCH("k1_hash_count", s, k_hash_count<K, OffT, POW2><<<g1, 256, 0, s>>>(keys, t.n, t.seed, t.hash_kind, nv, offs + 1,
                                                   a.aggregate));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    void* scratch = nullptr;
    if ((e = cudaMallocAsync(&scratch, scan_scratch_bytes(t.nv), s)) != cudaSuccess) return e;
    e = launch_scan<OffT, OffT>(offs + 1, offs + 1, t.nv, scratch, nullptr, s, "k2_scan");
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return e;
    const unsigned g3 = persistent_grid(k_scatter<K, VT, OffT, POW2>, 256, 0, t.n);
    HG_LAUNCH("k3_scatter", s, k_scatter<K, VT, OffT, POW2><<<g3, 256, 0, s>>>(
        keys, static_cast<const VT*>(a.vals), t.n, t.seed, t.hash_kind, nv, offs + 1,
        static_cast<K*>(t.keys), static_cast<VT*>(t.vals), a.aggregate));
    return cudaGetLastError();
}

// Binned build, hg_binned.cu.
template <typename K, typename VT, typename OffT, int POW2>
cudaError_t build_v2_impl(const TableDesc& t, const BuildArgs& a, cudaStream_t s);

static const char* const kSliceNames[3] = {"slice_hist", "slice_split", "slice_split2"};

// Geometry of the one-digit split into G vertex-range slices of 2^sshift
// vertices: "partition" = slice.
inline PartGeom slice_geom(uint32_t sshift, uint64_t G) {
    PartGeom g;
    g.pshift = sshift;
    g.nparts = G;
    g.bits = ceil_log2(G);
    g.b1 = g.bits;
    g.b2 = 0;
    return g;
}

// Width (log2 vertices) of the slices a binned build is split into, 0 when
// the whole vertex range fits 2^16 partitions of the tuned width (~4096
// entries, 2048 for 16-byte entries; make_geom in hg_radix.cuh).
static uint32_t v2_slice_shift(const TableDesc& t, const BuildArgs& a, size_t entry_bytes) {
    if (t.n == 0) return 0;
    const double target = entry_bytes >= 16 ? 2048.0 : 4096.0;
    uint32_t ps = 0;
    if (a.partition_vertices) {
        ps = ceil_log2(a.partition_vertices);
        if (ps > kMaxPartShift) ps = kMaxPartShift;
    } else {
        const double per_vertex = double(t.n) / double(t.nv);
        while (ps < kMaxPartShift && per_vertex * double(uint64_t(2) << ps) <= target) ++ps;
    }
    // Slice when 2^16 partitions would be wider than kMaxPartShift, or hold
    // more than 4x the tuned entry count (oversized partitions go through
    // the grid-wide K7b path, which beats an extra split pass up to ~4x:
    // C3 u64 at load 1 runs 2x-oversized partitions).
    // A requested partition width (partition_vertices) is kept exactly.
    const uint32_t vbits = ceil_log2(t.nv);
    const uint32_t slack = a.partition_vertices ? 0 : 2;
    if (vbits > 16 + kMaxPartShift || vbits > 16 + ps + slack) return 16 + ps;
    return 0;
}

// Binned build over a vertex range wider than 2^16 partitions of the tuned
// width (V > 2^28 at load 1, e.g. 2^31 keys or C5's 2^31-vertex shards). The
// reference's bin split (core.hpp:192-197) is applied once more on top: K11
// splits the keys into G slices of 2^sshift consecutive vertices as AoS
// records {key, input position} (one pass of the partition machinery,
// hg_radix.cuh), then each slice is built by the binned build (whose first
// pass reads the records) into its range of the one table -- offsets written with the slice's entry
// base (TableDesc::obase), keys / values at the slice's entry range -- so
// every slice keeps the tuned partition geometry (two 8-bit digits, K7 at two
// CTAs per SM). Extra traffic: one histogram + one split pass over the keys.
template <typename K, typename VT, typename OffT, int HM>
static cudaError_t build_v2_sliced(const TableDesc& t, const BuildArgs& a, uint32_t sshift,
                                   cudaStream_t s) {
    const uint64_t S = uint64_t(1) << sshift;
    const uint64_t G = (t.nv + S - 1) / S;
    if (G > 256) return cudaErrorInvalidValue;
    using E = typename EntryT<K, VT>::T;
    // one multisplit pass with digit = local vertex >> sshift (hg_radix.cuh:
    // histogram, scan, TMA-staged split) -> records grouped by slice
    const PartGeom sg = slice_geom(sshift, G);
    const size_t rbytes = (t.n * sizeof(E) + 255) & ~size_t(255);
    const size_t sbytes = ((G + 1) * 8 + 255) & ~size_t(255);
    const size_t pbytes = PartitionScratch<K, VT, uint64_t>::bytes(sg, t.n);
    char* scratch = nullptr;
    cudaError_t e = cudaSuccess;
    if (huge_allocation(rbytes + sbytes + pbytes)) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), rbytes + sbytes + pbytes, s);
    if (e != cudaSuccess) return e;
    E* rec = reinterpret_cast<E*>(scratch);
    uint64_t* dstart = reinterpret_cast<uint64_t*>(scratch + rbytes);
    uint64_t cnt[257];
    do {
        const Divisor nv = make_divisor(global_nv(t), t.vbase);
        if ((e = partition<K, VT, uint64_t, HM>(static_cast<const K*>(a.keys),
                                                static_cast<const VT*>(a.vals), t.n, t.seed,
                                                t.hash_kind, nv, sg, dstart, scratch + rbytes + sbytes,
                                                rec, s, kSliceNames,
                                                static_cast<const E*>(a.records))) != cudaSuccess)
            break;
        if ((e = cudaMemcpyAsync(cnt, dstart, (G + 1) * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess)
            break;
        for (uint64_t g = 0; g < G; ++g) cnt[g] = cnt[g + 1] - cnt[g];  // slice sizes
        uint64_t start = 0;
        for (uint64_t g = 0; g < G && e == cudaSuccess; ++g) {
            TableDesc sub = t;
            sub.nv = t.nv - g * S < S ? t.nv - g * S : S;
            sub.n = cnt[g];
            sub.gnv = global_nv(t);
            sub.vbase = t.vbase + g * S;
            sub.obase = t.obase + start;
            sub.offs = static_cast<OffT*>(t.offs) + g * S;
            sub.keys = static_cast<K*>(t.keys) + start;
            sub.vals = static_cast<VT*>(t.vals) + start;
            BuildArgs sa = a;
            sa.keys = nullptr;
            sa.vals = nullptr;
            sa.records = rec + start;
            sa.n = cnt[g];
            sa.stable = 0;
            e = build_v2_impl<K, VT, OffT, HM>(sub, sa, s);
            start += cnt[g];
        }
    } while (false);
    cudaFreeAsync(scratch, s);
    return e;
}

// AoS records -> SoA keys / values (the simple build takes SoA input; the
// binned build's first pass, sliced or not, reads records directly).
template <typename K, typename VT>
__global__ void k_unpack_records(const typename EntryT<K, VT>::T* __restrict__ rec, uint64_t n,
                                 K* __restrict__ keys, VT* __restrict__ vals) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const auto r = rec[i];
        keys[i] = EntryT<K, VT>::key(r);
        vals[i] = EntryT<K, VT>::val(r);
    }
}

template <typename K, typename VT, typename OffT>
static cudaError_t build_typed(const TableDesc& t, const BuildArgs& a, cudaStream_t s);

template <typename K, typename VT, typename OffT>
static cudaError_t build_from_records_soa(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    const size_t kb = (t.n * sizeof(K) + 255) & ~size_t(255);
    char* scr = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scr), kb + t.n * sizeof(VT) + 256, s);
    if (e != cudaSuccess) return e;
    K* keys = reinterpret_cast<K*>(scr);
    VT* vals = reinterpret_cast<VT*>(scr + kb);
    k_unpack_records<K, VT><<<unsigned(std::min<uint64_t>((t.n + 255) / 256, uint64_t(num_sms()) * 16)),
                              256, 0, s>>>(static_cast<const typename EntryT<K, VT>::T*>(a.records),
                                           t.n, keys, vals);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        BuildArgs b = a;
        b.records = nullptr;
        b.keys = keys;
        b.vals = vals;
        e = build_typed<K, VT, OffT>(t, b, s);
    }
    cudaFreeAsync(scr, s);
    return e;
}

template <typename K, typename VT, typename OffT>
static cudaError_t build_typed(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    const uint32_t sshift = a.variant == 2 ? v2_slice_shift(t, a, sizeof(typename EntryT<K, VT>::T)) : 0;
    if (a.records && t.n && a.variant != 2) return build_from_records_soa<K, VT, OffT>(t, a, s);
    cudaError_t e = dispatch_hash_mode(hash_mode(global_nv(t), t.hash_kind), [&](auto hm) {
        constexpr int HM = decltype(hm)::value;
        if (sshift) return build_v2_sliced<K, VT, OffT, HM>(t, a, sshift, s);
        return a.variant == 2 ? build_v2_impl<K, VT, OffT, HM>(t, a, s)
                              : build_v1_impl<K, VT, OffT, HM>(t, a, s);
    });
    if (e == cudaSuccess && a.stable) e = stable_order<K, VT, OffT>(t, s);
    return e;
}

template <typename K, typename VT>
static cudaError_t build_off(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    return t.off_bytes == 4 ? build_typed<K, VT, uint32_t>(t, a, s)
                            : build_typed<K, VT, uint64_t>(t, a, s);
}

template <typename K>
static cudaError_t build_val(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    return t.val_bytes == 4 ? build_off<K, uint32_t>(t, a, s) : build_off<K, uint64_t>(t, a, s);
}

cudaError_t build_table(const TableDesc& t, const BuildArgs& a, cudaStream_t s) {
    return t.key_bytes == 4 ? build_val<uint32_t>(t, a, s) : build_val<uint64_t>(t, a, s);
}

}  // namespace hg
