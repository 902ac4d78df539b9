// hg_util.cu -- synthetic key generators and the device CSR validator.
//
// Generators: SURVEY.md Appendix B counter-based definitions, so host and
// device produce identical keys independent of chunking. (The reference's
// own keygen.hpp:59-73 uses sequential mt19937_64; those inputs are handed
// over as arrays / HGKEYS01 files instead.)
//
// Validator: device restatement of validate_csr (core.hpp:251-282) plus the
// key-consistency check edges[j].key == input[edges[j].index] that turns
// the structural check into a full equality proof at 2^28..2^32 (SURVEY.md
// 8(c) "Oracle at scale").
#include <algorithm>

#include "hg_common.cuh"
#include "hg_internal.h"

namespace hg {

int num_sms();

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t scramble31(uint64_t i) {
    uint32_t x = (uint32_t(i) * 0x9E3779B1u) & 0x7FFFFFFFu;
    x ^= x >> 16;
    x = (x * 0x85EBCA6Bu) & 0x7FFFFFFFu;
    x ^= x >> 13;
    return x;
}

template <typename K>
__global__ void k_generate(K* out, uint64_t n, int kind, uint64_t seed, uint64_t start,
                           double hit, const void* ref_, uint64_t n_ref) {
    const K* ref = static_cast<const K*>(ref_);
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t g = start + i;
        uint64_t k;
        if (kind == 0) {
            k = splitmix64(seed, g);
        } else if (kind == 1) {
            // C4 probes: hit with probability `hit` (double compare), else a
            // guaranteed miss (top bit set; C4 build keys are < 2^31).
            const uint64_t r = splitmix64(seed, 2 * g);
            const uint64_t u = splitmix64(seed, 2 * g + 1);
            const double x = double(u >> 11) * (1.0 / 9007199254740992.0);
            if (x < hit && n_ref) {
                k = uint64_t(ref[r % n_ref]);
            } else {
                k = sizeof(K) == 4 ? (r | 0x80000000ULL) : (r | 0x8000000000000000ULL);
            }
        } else if (kind == 2) {
            k = scramble31(g);  // kind 2: C4 unique build keys
        } else {
            // kind 3: C3 Zipf ranks over the host-built CDF (n_ref doubles):
            // r = lower_bound(CDF, u) + 1, key = mix64(r ^ 0x9E3779B97F4A7C15)
            const double* cdf = static_cast<const double*>(ref_);
            const double u = double(splitmix64(seed, g) >> 11) * (1.0 / 9007199254740992.0);
            uint64_t lo = 0, len = n_ref;
            while (len > 0) {
                const uint64_t h = len >> 1;
                if (cdf[lo + h] < u) {
                    lo += h + 1;
                    len -= h + 1;
                } else {
                    len = h;
                }
            }
            k = mix64((lo + 1) ^ 0x9E3779B97F4A7C15ULL);
        }
        out[i] = K(k);
    }
}

cudaError_t generate_keys(void* out, int key_bytes, uint64_t n, int kind, uint64_t seed,
                          uint64_t start, double hit, const void* ref, uint64_t n_ref,
                          cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    if (key_bytes == 4) {
        k_generate<uint32_t><<<grid, 256, 0, s>>>(static_cast<uint32_t*>(out), n, kind, seed, start,
                                                  hit, ref, n_ref);
    } else {
        k_generate<uint64_t><<<grid, 256, 0, s>>>(static_cast<uint64_t*>(out), n, kind, seed, start,
                                                  hit, ref, n_ref);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ validator
// Violation codes follow oracle/hg_oracle.c hgo_validate_csr:
// 3 offs[0] != 0, 4 offsets decrease, 5 offs[V] != N, 7 entry under a vertex
// its key does not hash to, 8 index out of range, 9 duplicate index,
// 10 key != input[index]. The smallest code found wins (atomicMin).

template <typename K, typename VT, typename OffT, int POW2>
__global__ void k_validate_vertices(const OffT* __restrict__ offs, uint64_t nv, uint64_t n,
                                    uint64_t seed, int hk, Divisor dv, const K* __restrict__ keys,
                                    uint32_t* code) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t tid0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid0 == 0) {
        if (offs[0] != 0) atomicMin(code, 3u);
        if (uint64_t(offs[nv]) != n) atomicMin(code, 5u);
    }
    for (uint64_t v = tid0; v < nv; v += stride) {
        const uint64_t b = offs[v], e = offs[v + 1];
        if (b > e) {
            atomicMin(code, 4u);
            continue;
        }
        if (e > n) continue;  // reported via code 4/5
        for (uint64_t j = b; j < e; ++j) {
            const uint64_t h = vhash<POW2>(keys[j], seed, dv);
            if (h != v) {
                atomicMin(code, 7u);
                break;
            }
        }
    }
}

template <typename K, typename VT>
__global__ void k_validate_entries(const K* __restrict__ keys, const VT* __restrict__ vals,
                                   uint64_t n, const K* __restrict__ input, uint32_t* seen,
                                   uint32_t* code) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
        const uint64_t idx = vals[j];
        if (idx >= n) {
            atomicMin(code, 8u);
            continue;
        }
        const uint32_t bit = 1u << (idx & 31);
        if (atomicOr(seen + (idx >> 5), bit) & bit) atomicMin(code, 9u);
        if (input && input[idx] != keys[j]) atomicMin(code, 10u);
    }
}

template <typename K, typename VT, typename OffT>
static cudaError_t validate_typed(const TableDesc& t, const void* input, uint32_t* d_code,
                                  cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(d_code, 0xff, 4, s);
    if (e != cudaSuccess) return e;
    const Divisor dv = make_divisor(global_nv(t), t.vbase);
    const unsigned grid = unsigned(num_sms()) * 8;
    dispatch_hash_mode(hash_mode(global_nv(t), t.hash_kind), [&](auto hm) {
        k_validate_vertices<K, VT, OffT, decltype(hm)::value><<<grid, 256, 0, s>>>(
            static_cast<const OffT*>(t.offs), t.nv, t.n, t.seed, t.hash_kind, dv,
            static_cast<const K*>(t.keys), d_code);
        return 0;
    });
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (t.n) {
        void* seen = nullptr;
        const size_t bytes = ((t.n + 31) / 32) * 4;
        if ((e = cudaMallocAsync(&seen, bytes, s)) != cudaSuccess) return e;
        cudaMemsetAsync(seen, 0, bytes, s);
        k_validate_entries<K, VT><<<grid, 256, 0, s>>>(
            static_cast<const K*>(t.keys), static_cast<const VT*>(t.vals), t.n,
            static_cast<const K*>(input), static_cast<uint32_t*>(seen), d_code);
        e = cudaGetLastError();
        cudaFreeAsync(seen, s);
    }
    return e;
}

template <typename K, typename VT>
static cudaError_t validate_off(const TableDesc& t, const void* in, uint32_t* c, cudaStream_t s) {
    return t.off_bytes == 4 ? validate_typed<K, VT, uint32_t>(t, in, c, s)
                            : validate_typed<K, VT, uint64_t>(t, in, c, s);
}
template <typename K>
static cudaError_t validate_val(const TableDesc& t, const void* in, uint32_t* c, cudaStream_t s) {
    return t.val_bytes == 4 ? validate_off<K, uint32_t>(t, in, c, s)
                            : validate_off<K, uint64_t>(t, in, c, s);
}
cudaError_t validate_table(const TableDesc& t, const void* input, uint32_t* d_code, cudaStream_t s) {
    return t.key_bytes == 4 ? validate_val<uint32_t>(t, input, d_code, s)
                            : validate_val<uint64_t>(t, input, d_code, s);
}

}  // namespace hg
