// hg_common.cuh -- device primitives shared by every HashGraph kernel (sm_100a).
//
// Bit-exact device restatement of the reference vertex hash
// (reference: proj/include/hashgraph/hash.hpp:12-19 mix64, :30-33
// VertexHasher = mix64(key ^ seed) % V) with an exact, division-free
// reduction, plus the tiny PTX helpers the kernels use.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace hg {

enum HashKind : int { kHashMix64 = 0, kHashIdentity = 1 };

// Exact "h mod d" / "h div d" for a runtime divisor d >= 1 without the ~60
// instruction emulated 64-bit division. magic = floor((2^64-1)/d); the
// estimate q = umulhi(h, magic) satisfies q_true-1 <= q <= q_true for every
// h < 2^64 (error h*(1/d - magic/2^64) <= h/2^64 < 1), so one correction
// step is exact. Power-of-two divisors use shift/mask (template POW2).
// For the vertex space, `base` is subtracted after the reduction: a
// hash-range shard owning global vertices [base, base + local V) numbers its
// vertices locally; base = 0 for an unsharded table.
struct Divisor {
    uint64_t d;
    uint64_t magic;
    uint32_t shift;  // log2(d) when d is a power of two
    uint32_t pow2;
    uint64_t base;
};

inline Divisor make_divisor(uint64_t d, uint64_t base = 0) {
    Divisor r;
    r.d = d;
    r.magic = ~uint64_t(0) / d;
    r.pow2 = (d & (d - 1)) == 0;
    r.shift = 0;
    while (r.pow2 && (uint64_t(1) << r.shift) < d) ++r.shift;
    r.base = base;
    return r;
}

template <int POW2>
__device__ __forceinline__ uint64_t mod_of(uint64_t h, const Divisor& m) {
    if constexpr (POW2) {
        return h & (m.d - 1);
    } else {
        const uint64_t q = __umul64hi(h, m.magic);
        uint64_t r = h - q * m.d;
        return r >= m.d ? r - m.d : r;
    }
}

template <int POW2>
__device__ __forceinline__ uint64_t div_of(uint64_t h, const Divisor& m) {
    if constexpr (POW2) {
        return h >> m.shift;
    } else {
        uint64_t q = __umul64hi(h, m.magic);
        const uint64_t r = h - q * m.d;
        return r >= m.d ? q + 1 : q;
    }
}

// hash.hpp:12-19 (murmur3 fmix64).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// hash.hpp:30-33; keys narrower than 64 bits are zero-extended first (the
// reference API is u64-only, core.hpp:161). kHashIdentity restates the
// fixture hasher of tests/support.hpp:42-46 (key % V).
template <int HK, int POW2>
__device__ __forceinline__ uint64_t vertex_of(uint64_t key, uint64_t seed, const Divisor& nv) {
    if constexpr (HK == kHashIdentity) {
        return mod_of<POW2>(key, nv) - nv.base;
    } else {
        return mod_of<POW2>(mix64(key ^ seed), nv) - nv.base;
    }
}

// Hash mode HM (a template parameter of every kernel): bit 0 = V is a power
// of two (mask instead of magic reduction), bit 1 = identity hasher.
template <int HM>
__device__ __forceinline__ uint64_t vhash(uint64_t key, uint64_t seed, const Divisor& nv) {
    return vertex_of<(HM & 2) ? kHashIdentity : kHashMix64, (HM & 1) != 0>(key, seed, nv);
}

inline int hash_mode(uint64_t global_vertices, int hash_kind) {
    return ((global_vertices & (global_vertices - 1)) == 0 ? 1 : 0) |
           (hash_kind == kHashIdentity ? 2 : 0);
}

// Calls f(std::integral_constant<int, HM>{}) for the runtime hash mode.
template <typename F>
inline auto dispatch_hash_mode(int hm, F&& f) {
    switch (hm) {
        case 0: return f(std::integral_constant<int, 0>{});
        case 1: return f(std::integral_constant<int, 1>{});
        case 2: return f(std::integral_constant<int, 2>{});
        default: return f(std::integral_constant<int, 3>{});
    }
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Streaming (evict-first) loads for read-once inputs so they do not displace
// the L2-resident working set (counters, partitions).
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
    return __ldcs(p);
}

// ---- TMA 1-D bulk copies + mbarriers (sm_90+ async proxy; SASS UBLKCP / SYNCS)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Orders this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (TMA) accesses to the same buffer.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// dst (shared) <- src (global), bytes % 16 == 0, both 16-byte aligned.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// global <- shared bulk store (async proxy), bytes % 16 == 0, both 16-byte aligned.
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_addr(src)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Waits until all committed bulk stores of this thread have finished reading
// shared memory (the staging buffer may be overwritten afterwards).
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Waits until all committed bulk stores of this thread are complete.
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Stores elements [0, n) of a shared staging array `src` to global `dst`
// where src[0] corresponds to dst[0] and (dst - src) is a multiple of 16
// bytes in address alignment terms (i.e. both have the same address & 15).
// The 16-byte-aligned middle goes out as one bulk copy issued by `lane0`
// (returns true when it issued one); the unaligned head and tail elements
// are stored by the calling threads (tid/nthreads). Caller must have fenced
// (fence_proxy_async) + synchronised the staging writes beforehand.
template <typename T>
__device__ __forceinline__ bool bulk_store_span(T* dst, const T* src, uint32_t n, uint32_t tid,
                                                uint32_t nthreads) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    const uint32_t head = uint32_t(((16 - (a & 15)) & 15) / sizeof(T));
    const uint32_t h = head < n ? head : n;
    const uint32_t body = ((n - h) * sizeof(T)) & ~uint32_t(15);
    const uint32_t body_n = body / sizeof(T);
    for (uint32_t i = tid; i < h; i += nthreads) dst[i] = src[i];
    for (uint32_t i = h + body_n + tid; i < n; i += nthreads) dst[i] = src[i];
    if (tid == 0 && body) {
        tma_store_1d(dst + h, src + h, body);
        return true;
    }
    return false;
}

// Issues the 16-byte-aligned superset of global bytes [src, src + bytes) into
// dst; returns the byte offset of src inside dst. Caller's buffer must hold
// bytes + 32.
__device__ __forceinline__ uint32_t tma_load_span(void* dst, const void* src, uint32_t bytes,
                                                  uint64_t* bar) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t lo = a & ~uintptr_t(15);
    const uintptr_t hi = (a + bytes + 15) & ~uintptr_t(15);
    const uint32_t len = uint32_t(hi - lo);
    mbar_arrive_expect_tx(bar, len);
    if (len) tma_load_1d(dst, reinterpret_cast<const void*>(lo), len, bar);
    return uint32_t(a - lo);
}

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_addr(p)));
    return v;
}

__device__ __forceinline__ void sts128(void* p, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_addr(p)), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint32_t atom_add(uint32_t* p, uint32_t v) { return atomicAdd(p, v); }
__device__ __forceinline__ uint64_t atom_add(uint64_t* p, uint64_t v) {
    return atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}
__device__ __forceinline__ void red_add(uint32_t* p, uint32_t v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_add(uint64_t* p, uint64_t v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// Peer mask of lanes holding the same vertex id: 32-bit match when every
// vertex id fits 32 bits (V <= 2^32), else the 64-bit form.
template <bool V32>
__device__ __forceinline__ uint32_t match_peers(uint32_t active, uint64_t v) {
    if constexpr (V32) {
        return __match_any_sync(active, static_cast<uint32_t>(v));
    } else {
        return __match_any_sync(active, static_cast<unsigned long long>(v));
    }
}

// Warp-aggregated atomicAdd of 1 on counter (CounterArray
// ticket semantics, parallel.hpp:112-118). Lanes with equal v form a peer
// group; the lowest lane adds popc(group) once, every lane gets a distinct
// ticket base + rank, so k adds on one slot hand out {old..old+k-1} exactly
// once (test_parallel.cpp:79-125). Must be called by all lanes in `active`.
template <bool V32, typename C>
__device__ __forceinline__ C aggregated_ticket(C* counter, uint32_t active, uint64_t v) {
    const uint32_t peers = match_peers<V32>(active, v);
    const uint32_t leader = __ffs(peers) - 1;
    const uint32_t rank = __popc(peers & lanemask_lt());
    C base = 0;
    if (lane_id() == leader) base = atom_add(counter, C(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    return base + C(rank);
}

template <bool V32, typename C>
__device__ __forceinline__ void aggregated_count(C* counter, uint32_t active, uint64_t v) {
    const uint32_t peers = match_peers<V32>(active, v);
    if (lane_id() == uint32_t(__ffs(peers) - 1)) red_add(counter, C(__popc(peers)));
}

// -1 when x == y and `in` (0 otherwise): one ISETP + SEL, and the caller sums
// with IADD3 -- no dependency chain through a running count.
template <typename K>
__device__ __forceinline__ uint32_t eq_and(K x, K y, bool in) {
    uint32_t d;
    if constexpr (sizeof(K) == 4) {
        asm("{.reg .pred p; setp.ne.u32 p, %3, 0; set.eq.and.u32.u32 %0, %1, %2, p;}"
            : "=r"(d)
            : "r"(x), "r"(y), "r"(uint32_t(in)));
    } else {
        asm("{.reg .pred p; setp.ne.u32 p, %3, 0; set.eq.and.u32.u64 %0, %1, %2, p;}"
            : "=r"(d)
            : "l"(x), "l"(y), "r"(uint32_t(in)));
    }
    return d;
}

// seg_count that also reports, in `pos`, the index of a match inside the
// segment (the only one when the count is 1): the single-pass pairs kernel
// needs it for its one-match fast path and no longer walks the segment again.
template <typename K>
__device__ __forceinline__ uint32_t seg_count_pos(const K* __restrict__ sp, uint64_t len, K key,
                                                  uint32_t& pos) {
    if (len <= 4) {
        uint32_t neg = 0, at = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            const bool in = q < len;
            const K x = in ? sp[q] : K(0);
            const uint32_t eq = eq_and(x, key, in);
            neg += eq;
            at |= eq & q;
        }
        pos = at;
        return 0u - neg;
    }
    uint32_t c = 0, at = 0;
    for (uint32_t t = 0; t < uint32_t(len); ++t) {
        const bool eq = sp[t] == key;
        c += eq;
        at = eq ? t : at;
    }
    pos = at;
    return c;
}

// Matches of `key` in the segment sp[0, len) for a short segment (the caller
// walks long ones warp-cooperatively). Segments of <= 4 entries (~99% at load
// 1) use a fixed, predicated 4-wide compare: no loop, no divergence.
template <typename K>
__device__ __forceinline__ uint32_t seg_count(const K* __restrict__ sp, uint64_t len, K key) {
    if (len <= 4) {
        uint32_t neg = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            const bool in = q < len;
            const K x = in ? sp[q] : K(0);
            neg += eq_and(x, key, in);
        }
        return 0u - neg;
    }
    uint32_t c = 0;
    for (uint32_t t = 0; t < uint32_t(len); ++t) c += sp[t] == key;
    return c;
}

}  // namespace hg
