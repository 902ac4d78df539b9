/*
 * hg_b200.h -- C-ABI of the B200-native HashGraph engine (libhg_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/hashgraph, header-only C++20). The reference
 * has no FFI of its own; each entry point below names the reference
 * interface it replaces (file:line), and include/hashgraph/ headers re-export
 * the reference's C++ names on top of these calls.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross this boundary.
 *  - Every array argument may live in host memory (pageable or pinned) or in
 *    device memory of the current CUDA device; the library detects which and
 *    stages host data through the device in stream order.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Calls are stream-ordered. A call that returns host-visible scalars
 *    (hg_probe without device_result, hg_count_instances, hg_validate,
 *    hg_table_export into host memory) synchronises `stream` first.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    call fails with HG_ECUDA.
 */
#ifndef HG_B200_H
#define HG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 1

/* Error model. Replaces the reference's exceptions:
 *   std::invalid_argument (core.hpp:106-109 check_config, join.hpp:145-147) -> HG_EINVAL
 *   std::out_of_range     (core.hpp:88-90 vertex_entries)                   -> HG_ERANGE
 *   std::overflow_error   (parallel.hpp:153,171,178)                        -> HG_EOVERFLOW */
typedef enum hg_status {
    HG_OK = 0,
    HG_EINVAL = 1,
    HG_ERANGE = 2,
    HG_EOVERFLOW = 3,
    HG_ENOMEM = 4,
    HG_ECUDA = 5,
    HG_ENCCL = 6,
    HG_EUNSUPPORTED = 7,
    HG_EIO = 8 /* KeyFileError (keygen.hpp:75-77): I/O or key-file format problem */
} hg_status;

typedef enum hg_hash_kind {
    HG_HASH_MIX64 = 0,    /* VertexHasher: mix64(key ^ seed) % V (hash.hpp:27-34) */
    HG_HASH_IDENTITY = 1  /* key % V; the fixture hasher of tests/support.hpp:42-46 */
} hg_hash_kind;

typedef enum hg_variant {
    HG_BUILD_SIMPLE = 1, /* build_v1 (core.hpp:160-177) */
    HG_BUILD_BINNED = 2  /* build_v2 (core.hpp:183-230) */
} hg_variant;

/* BuildConfig (core.hpp:30-35) + the optional vertex_count override of
 * build_v1/build_v2 (core.hpp:165-166) + device knobs. */
typedef struct hg_build_config {
    double load_factor;          /* V = max(1, floor(N / load_factor)) (core.hpp:59-63) */
    uint64_t bin_count;          /* validated (>= 1, core.hpp:108); CPU-cache tuning knob */
    uint64_t hash_seed;          /* core.hpp:33 */
    uint64_t vertex_count;       /* 0 = derive from load_factor */
    int32_t variant;             /* hg_variant */
    int32_t hash_kind;           /* hg_hash_kind */
    int32_t stable;              /* 1 = ExecMode::sequential layout: segments in input order */
    int32_t aggregate;           /* warp-aggregated atomics: -1 auto, 0 off, 1 on */
    uint64_t partition_vertices; /* binned build partition width (power of two); 0 = auto */
    /* Hash-range shard (multi-GPU): when global_vertices != 0
     * the table holds global vertices [vertex_base, vertex_base + vertex_count)
     * of a V = global_vertices table; vertex v is stored as local v - vertex_base.
     * Keys must have been routed to this shard (hg_route). */
    uint64_t global_vertices;
    uint64_t vertex_base;
} hg_build_config;

/* Defaults of BuildConfig{} (core.hpp:30-35): load 1.0, bins 2^15, seed 0,
 * parallel mode (stable = 0), variant HG_BUILD_SIMPLE. */
void hg_build_config_init(hg_build_config* cfg);

/* derived_vertex_count (core.hpp:59-63). HG_EINVAL when load_factor <= 0. */
hg_status hg_derived_vertex_count(uint64_t n, double load_factor, uint64_t* out);

/* hash_to_vertex (hash.hpp:36-39) for a single key, host-side convenience
 * (the table paths evaluate the same function on the device). */
uint64_t hg_hash_to_vertex(uint64_t key, uint64_t seed, uint64_t num_vertices);

typedef struct hg_table hg_table;

/* build_v1 / build_v2 (core.hpp:173-177, :226-230 and the hasher-templated
 * overloads :160-171, :183-224).
 *   keys       n keys of key_width bytes (4 = u32, 8 = u64; u32 keys are
 *              zero-extended before hashing, exactly as the reference's
 *              u64-only API would see them)
 *   vals       NULL: each entry's value is its input position (Entry::index,
 *              core.hpp:21-26); else n values of val_width (4|8) bytes
 * On success *out owns the device-resident CSR table. */
hg_status hg_build(const void* keys, int32_t key_width, const void* vals, int32_t val_width,
                   uint64_t n, const hg_build_config* cfg, void* stream, hg_table** out);

typedef struct hg_table_info {
    uint64_t num_vertices; /* HashGraph::num_vertices (core.hpp:79) */
    uint64_t num_edges;    /* HashGraph::num_edges (core.hpp:80) */
    uint64_t hash_seed;    /* core.hpp:83 */
    double load_factor;    /* core.hpp:84 */
    int32_t key_width;
    int32_t val_width;
    int32_t off_width;     /* device offsets width (4 when N < 2^32 and V <= 2^32) */
    int32_t hash_kind;
} hg_table_info;

hg_status hg_table_get_info(const hg_table* t, hg_table_info* info);

/* Zero-copy device views of the SoA CSR (offsets[V+1], keys[N], vals[N]). */
hg_status hg_table_device_arrays(const hg_table* t, const void** offsets, const void** keys,
                                 const void** vals);

/* HashGraph::offsets()/edges() (core.hpp:81-82) in the reference layout,
 * widened to u64: offsets[V+1], keys[N], vals[N] (any may be NULL). */
hg_status hg_table_export(const hg_table* t, uint64_t* offsets, uint64_t* keys, uint64_t* vals,
                          void* stream);

/* hg_build from n AoS records {key, value} (the layout hg_route_records
 * writes: 8-byte records for key_width = val_width = 4, else 16-byte records
 * of two u64 fields); the binned build's first pass reads them directly. */
hg_status hg_build_records(const void* records, int32_t key_width, int32_t val_width, uint64_t n,
                           const hg_build_config* cfg, void* stream, hg_table** out);

/* A device table from caller arrays in the reference layout (HashGraph's
 * constructor from offsets/edges, core.hpp:71-77): offsets[V+1], keys[N],
 * vals[N] as u64 (host or device). No validation is done here; hg_validate
 * checks the invariants. */
hg_status hg_table_import(const uint64_t* offsets, const uint64_t* keys, const uint64_t* vals,
                          uint64_t num_vertices, uint64_t num_edges, uint64_t hash_seed,
                          double load_factor, int32_t hash_kind, void* stream, hg_table** out);

/* Frees the table's device buffers in stream order. */
hg_status hg_table_destroy(hg_table* t, void* stream);

/* ProbeOptions (join.hpp:25-28) + device output knobs. */
typedef struct hg_probe_options {
    int32_t materialize;     /* collect pairs (join.hpp:26) */
    int32_t pair_width;      /* 8: MatchPair{u64 left, u64 right} layout (join.hpp:18-23); 4: u32 pairs */
    uint64_t pair_cap;       /* join.hpp:27, default 2^24 */
    void* pairs;             /* >= pair_cap pairs; host or device */
    uint32_t* counts;        /* nullable: per-probe match counts (count_instances per key) */
    uint64_t* device_result; /* nullable device u64[2] {match_count, key_comparisons}; when set
                                the call is fully asynchronous (result is zeroed) */
    int32_t method;          /* 0 auto, 1 direct gathers, 2 vertex-range partitioned probes */
    int32_t flags;           /* HG_PROBE_* bits below */
    uint64_t hash_seed;      /* with HG_PROBE_HASHER: the probe-side hasher (join.hpp:110-131 */
    int32_t hash_kind;       /*   hashes every probe with the caller's hasher, not the table's) */
    int32_t reserved;
} hg_probe_options;

/* hg_probe_options.flags: the pinned host probe buffer already holds its final
 * contents when hg_probe is called (no earlier work on `stream` writes it), so
 * its chunked host->device copies may start before earlier work on `stream`
 * (e.g. the build of the probed table) has finished. Without it the copies
 * are ordered after all earlier work on `stream`. */
#define HG_PROBE_HOST_READY 1
/* hg_probe_options.flags: hash the probes with (hash_kind, hash_seed) instead
 * of the table's own hasher -- probe_standard(hg, keys, hasher, opts),
 * join.hpp:110-131: vertex = hasher(key, V), then that vertex's segment. */
#define HG_PROBE_HASHER 2

void hg_probe_options_init(hg_probe_options* opts);

/* JoinResult (join.hpp:30-35). */
typedef struct hg_probe_result {
    uint64_t match_count;     /* exact, independent of materialisation */
    uint64_t key_comparisons; /* full-key comparisons = sum of probed segment lengths */
    uint64_t pairs_written;   /* min(match_count, pair_cap) when materialising */
    int32_t truncated;        /* match_count > pair_cap */
} hg_probe_result;

/* probe_standard (join.hpp:110-136). Pairs are (left = build entry value,
 * right = probe position) (join.hpp:125), written to deterministic slots in
 * probe order; under a cap the first pair_cap slots are kept. probe_width
 * must equal the table's key width or be 4 for a u64-keyed table. */
hg_status hg_probe(const hg_table* t, const void* probes, int32_t probe_width, uint64_t m,
                   const hg_probe_options* opts, hg_probe_result* result, void* stream);

/* probe_new_prepared (join.hpp:143-166) over intersect_adjacency
 * (join.hpp:41-57): a and b must share the vertex range (num_vertices equal,
 * else HG_EINVAL as join.hpp:145-147 throws invalid_argument) and the key
 * width. Pairs are (left = a's entry value, right = b's entry value), written
 * in sequential order (vertex, then a position, then b position); under a
 * cap the first pair_cap of that order are kept. key_comparisons =
 * sum_v |A_v| * |B_v|. opts->counts must be NULL (there are no probes). */
hg_status hg_probe_new_prepared(const hg_table* a, const hg_table* b, const hg_probe_options* opts,
                                hg_probe_result* result, void* stream);

/* probe_new (join.hpp:170-182): builds keys_a and keys_b (key_width bytes
 * each) with the binned build over the shared V = derived_vertex_count(
 * max(na, nb), cfg->load_factor) (or cfg->vertex_count when non-zero), then
 * hg_probe_new_prepared. Entry values are input positions. */
hg_status hg_probe_new(const void* keys_a, uint64_t na, const void* keys_b, uint64_t nb,
                       int32_t key_width, const hg_build_config* cfg, const hg_probe_options* opts,
                       hg_probe_result* result, void* stream);

/* count_instances (core.hpp:235-246) with the table's own hasher. */
hg_status hg_count_instances(const hg_table* t, uint64_t key, uint64_t* out, void* stream);

/* count_instances(hg, key, hasher) (core.hpp:235-242): the key's vertex is
 * hasher(key, V) for the hasher (hash_kind, hash_seed) the caller passes. */
hg_status hg_count_instances_hasher(const hg_table* t, uint64_t key, int32_t hash_kind,
                                    uint64_t hash_seed, uint64_t* out, void* stream);

/* validate_csr (core.hpp:251-287) on the device, plus (input_keys != NULL)
 * the check keys[j] == input_keys[vals[j]]. *violation = 0 when valid, else
 * the code of the first violated invariant (see hg_util.cu). */
hg_status hg_validate(const hg_table* t, const void* input_keys, uint64_t expected_entries,
                      int32_t* violation, void* stream);

/* validate_csr(hg, expected, hasher) (core.hpp:251-282): as hg_validate, with
 * the hash-consistency check (entry under hasher(key, V)) made with the
 * caller's hasher (hash_kind, hash_seed). */
hg_status hg_validate_hasher(const hg_table* t, const void* input_keys, uint64_t expected_entries,
                             int32_t hash_kind, uint64_t hash_seed, int32_t* violation,
                             void* stream);

/* Multi-GPU routing (K11). Shard g of G owns global vertices
 * [g*S, min((g+1)*S, V)), S = ceil(V/G) (the reference's bin formula,
 * core.hpp:192-197, at bins = G). */
hg_status hg_shard_range(uint64_t global_vertices, uint32_t shards, uint32_t shard,
                         uint64_t* vertex_base, uint64_t* vertex_count);

/* Groups n device-resident keys by owner shard into SoA device buffers
 * out_keys/out_vals (n entries each, keys of shard 0 first) and writes the
 * per-shard counts to shard_counts (G entries; host or device). Values are
 * vals[i] or, when vals is NULL, val_base + i (global input positions) of
 * width val_width; out_vals may be NULL (keys only, e.g. count-only probes).
 * G <= 256. */
hg_status hg_route(const void* keys, int32_t key_width, const void* vals, int32_t val_width,
                   uint64_t n, uint64_t val_base, uint64_t hash_seed, int32_t hash_kind,
                   uint64_t global_vertices, uint32_t shards, void* out_keys, void* out_vals,
                   uint64_t* shard_counts, void* stream);

/* hg_route with owner-grouped AoS records {key, value} in ONE device buffer
 * (8-byte records for key_width = val_width = 4, else 16-byte records with
 * both fields widened to u64) -- the one buffer a single all-to-all moves and
 * hg_build_records consumes. shard_counts: device, G entries. */
hg_status hg_route_records(const void* keys, int32_t key_width, const void* vals,
                           int32_t val_width, uint64_t n, uint64_t val_base, uint64_t hash_seed,
                           int32_t hash_kind, uint64_t global_vertices, uint32_t shards,
                           void* out_records, uint64_t* shard_counts, void* stream);

/* Groups n match pairs (left[i], right[i]) (pair_width 4 or 8, device) by
 * owner = right[i] / span into AoS records {left, right} (device), G <= 256
 * -- the reverse routing that returns pairs to the rank holding each probe
 * (probes of rank r have global positions [r * span, (r + 1) * span)). */
hg_status hg_route_pairs(const void* left, const void* right, int32_t pair_width, uint64_t n,
                         uint64_t span, uint32_t shards, void* out_records, uint64_t* shard_counts,
                         void* stream);

/* Synthetic inputs: kind 0 = (u32|u64)splitmix64(seed, start+i);
 * kind 1 = C4 probes with hit ratio `hit` over ref[n_ref]; kind 2 = scramble31(start+i);
 * kind 3 = C3 Zipf keys mix64(r ^ 0x9E3779B97F4A7C15), r = lower_bound(cdf, u) + 1 with
 * u = (splitmix64(seed, start+i) >> 11) * 2^-53 and ref = the device CDF (n_ref doubles). */
hg_status hg_generate(void* out, int32_t key_width, uint64_t n, int32_t kind, uint64_t seed,
                      uint64_t start, double hit, const void* ref, uint64_t n_ref, void* stream);

/* Key files (keygen.hpp:97-132): 8-byte magic "HGKEYS01", little-endian u64
 * count, then count little-endian u64 keys -- the wire format shared with the
 * CPU reference. hg_keys_file_count validates the header and length.
 * hg_keys_read stores the keys into `out` (host or device, key_width 8, or 4
 * to narrow: HG_ERANGE if a key does not fit); device destinations are filled
 * in chunks through a pinned staging buffer. cap = capacity of `out` in keys
 * (HG_ERANGE when the file holds more). hg_keys_write writes n keys (host or
 * device, key_width 4 or 8; u32 keys are zero-extended). Errors: HG_EIO with
 * the reference's KeyFileError messages. */
hg_status hg_keys_file_count(const char* path, uint64_t* count);
hg_status hg_keys_read(const char* path, void* out, int32_t key_width, uint64_t cap, uint64_t* count,
                       void* stream);
hg_status hg_keys_write(const char* path, const void* keys, int32_t key_width, uint64_t n,
                        void* stream);

/* Kernel timeline (tracing): when enabled, every engine kernel launch is
 * bracketed by CUDA events on its stream. collect() waits for the recorded
 * events, aggregates per kernel name, clears the log and returns the number
 * of distinct kernels (entries beyond max_out are dropped). */
typedef struct hg_kernel_time {
    char name[48];
    uint64_t launches;
    double total_ms;
} hg_kernel_time;

void hg_profiler_enable(int32_t on);
int32_t hg_profiler_collect(hg_kernel_time* out, int32_t max_out);

/* Last error message of the calling thread. */
const char* hg_last_error(void);
int32_t hg_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HG_B200_H */
