// hg_internal.h -- host-side launcher interface between the C-ABI layer
// (hg_capi.cu) and the kernel translation units. Plain types only.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hg {

// Device table storage (SoA CSR): offs[V+1] (u32 when the
// table holds < 2^32 entries and V <= 2^32, else u64), keys[N] (u32/u64),
// vals[N] (u32/u64; the reference's Entry::index, core.hpp:21-26).
struct TableDesc {
    uint64_t nv = 1;        // V (local vertex count)
    uint64_t n = 0;         // N
    uint64_t gnv = 0;       // global vertex count of a hash-range shard (0 = nv)
    uint64_t vbase = 0;     // first global vertex owned by this shard
    uint64_t obase = 0;     // entry base added to every offset written (a vertex-range
                            // slice of a larger table, build_v2_sliced)
    uint64_t seed = 0;
    int hash_kind = 0;      // 0 mix64, 1 identity
    int key_bytes = 4;      // 4 | 8
    int val_bytes = 4;      // 4 | 8
    int off_bytes = 4;      // 4 | 8
    void* offs = nullptr;   // V+1 entries (offs[0] == 0)
    void* keys = nullptr;
    void* vals = nullptr;
};

struct BuildArgs {
    const void* keys = nullptr;  // device, n entries of key_bytes
    const void* vals = nullptr;  // device or nullptr (then val = input position)
    uint64_t n = 0;
    int variant = 1;             // 1 simple (V1), 2 binned (V2)
    int aggregate = 1;           // warp-aggregated atomics
    int stable = 0;              // reproduce ExecMode::sequential segment order
    uint64_t partition_vertices = 0;  // V2 partition width (0 = auto)
    // non-null: the input is n AoS records {key, value} (EntryT<K, VT>::T,
    // routed by route_keys with out_records) instead of keys / vals
    const void* records = nullptr;
};

// Builds into t (offs/keys/vals already allocated). Scratch is allocated
// stream-ordered from the device pool.
cudaError_t build_table(const TableDesc& t, const BuildArgs& a, cudaStream_t s);

struct ProbeArgs {
    const void* probes = nullptr;  // device, m entries of key_bytes (same as table)
    uint64_t m = 0;
    uint32_t* counts = nullptr;    // nullable: per-probe match counts (u32); scratch for the
                                   // direct pairs path when the caller did not ask for counts
    bool counts_requested = true;  // the caller wants `counts` filled (in probe order)
    uint64_t* totals = nullptr;    // device [2]: match_count, key_comparisons (accumulated)
    // pairs (K9/K10): when pairs != nullptr, pair_offsets must hold m+1 u64.
    void* pairs = nullptr;         // device, cap pairs of pair_bytes*2
    int pair_bytes = 8;            // 4 (u32 pairs) | 8 (MatchPair u64 layout)
    uint64_t cap = 0;
    uint64_t* pair_offsets = nullptr;
    int method = 0;                // 0 auto, 1 direct gathers, 2 partitioned
    // partitioned probe only: m AoS records {key, original probe position}
    // (EntryT<K, u32 | u64>::T, route_keys with out_records) instead of
    // `probes`; per-probe counts land at the original positions
    const void* records = nullptr;
};

cudaError_t probe_table(const TableDesc& t, const ProbeArgs& a, cudaStream_t s);

// probe_new_prepared (join.hpp:143-166): intersects two tables over one
// vertex range (A.nv == B.nv, equal key widths). totals[2] (device) are
// accumulated; pairs (device, nullable) receive (A value, B value) in
// sequential order (vertex, A position, B position), the first `cap` kept.
struct IntersectArgs {
    uint64_t* totals = nullptr;
    void* pairs = nullptr;
    int pair_bytes = 8;
    uint64_t cap = 0;
};

cudaError_t intersect_tables(const TableDesc& A, const TableDesc& B, const IntersectArgs& a,
                             cudaStream_t s);

// Counter-based synthetic generators.
// kind 0: key[i] = splitmix64(seed, start+i) (truncated to key_bytes).
// kind 1: C4 probes with hit ratio `hit` against build keys `ref` (n_ref).
cudaError_t generate_keys(void* out, int key_bytes, uint64_t n, int kind, uint64_t seed,
                          uint64_t start, double hit, const void* ref, uint64_t n_ref,
                          cudaStream_t s);

// Device-side CSR validation (core.hpp:251-282 plus
// key == input[index]). Returns violation code in *d_code (0 valid).
cudaError_t validate_table(const TableDesc& t, const void* input_keys, uint32_t* d_code,
                           cudaStream_t s);

int num_sms();
size_t smem_optin();  // opt-in shared memory per CTA (227 KB on B200)
bool huge_allocation(uint64_t bytes);  // > 1/8 of device memory: drain the stream first

// Vertex-space divisor of a table: global V (sharded) or V, with the shard base.
inline uint64_t global_nv(const TableDesc& t) { return t.gnv ? t.gnv : t.nv; }

// Hash-range routing: groups n keys (+ values, or
// implicit values val_base + i) by owner shard = ((h(key) mod V) - vertex_base)
// / span (span 0: ceil(local_vertices / G)) into SoA out_keys/out_vals;
// shard_counts[G] (device, u64) receives the number of keys per shard.
// G <= 256. Multi-GPU routing uses vertex_base = 0, local_vertices = V, span 0;
// the sliced binned build routes a table's own vertex range
// [vertex_base, vertex_base + local_vertices) into power-of-two spans.
cudaError_t route_keys(const void* keys, int key_bytes, const void* vals, int val_bytes,
                       uint64_t n, uint64_t val_base, uint64_t seed, int hash_kind,
                       uint64_t global_vertices, uint64_t vertex_base, uint64_t local_vertices,
                       uint64_t span, uint32_t shards, void* out_keys, void* out_vals,
                       uint64_t* shard_counts, cudaStream_t s, void* out_records = nullptr);

// As route_keys with out_records != nullptr: owner-grouped AoS records
// {key, value} (EntryT<K, VT>::T: 8 bytes for u32/u32, else 16) instead of SoA.
// route_pairs: groups match pairs (left[i], right[i]) by owner = right / span
// into AoS records of 2 x pair_bytes (pairs returned to the probe's rank).
cudaError_t route_pairs(const void* left, const void* right, int pair_bytes, uint64_t n,
                        uint64_t span, uint32_t shards, void* out_records, uint64_t* shard_counts,
                        cudaStream_t s);

// Kernel timeline hooks (hg_prof.cu).
bool prof_enabled();
int prof_begin(const char* name, cudaStream_t s);
void prof_end(int token, cudaStream_t s);

// Launch `launch` (a statement launching one kernel on stream s) bracketed by
// profiler events named `name`.
#define HG_LAUNCH(name, s, ...)                     \
    do {                                            \
        const int tok_ = ::hg::prof_begin(name, s); \
        __VA_ARGS__;                                \
        ::hg::prof_end(tok_, s);                    \
    } while (0)

}  // namespace hg
