// hashgraph/hashgraph.hpp -- C++ drop-in for the reference's hot-path API.
//
// Same namespace, names, types, defaults and exceptions as the reference
// headers (/root/reference/proj/include/hashgraph/{hash,core,join}.hpp), so a
// caller switches by pointing its include path here and linking
// libhg_b200.so. Every build / probe / validation runs on the B200 through
// the C-ABI in <hg_b200.h>; there is no CPU implementation behind these
// names. Replaced interfaces (reference file:line):
//   hash.hpp:12-19 detail::mix64, :27-34 VertexHasher, :36-39 hash_to_vertex
//   core.hpp:21-26 Entry, :28 ExecMode, :30-35 BuildConfig, :40-56 BuildStats,
//   :59-63 derived_vertex_count, :67-102 HashGraph, :160-177 build_v1,
//   :183-230 build_v2, :235-246 count_instances, :251-287 validate_csr
//   join.hpp:18-35 MatchPair / ProbeOptions / JoinResult, :110-136 probe_standard,
//   :41-57 intersect_adjacency, :143-166 probe_new_prepared, :170-182 probe_new
//
// Differences, by construction of a device engine:
//   * hashers: VertexHasher and hashgraph::IdentityHasher (key % V) run on
//     the device; any other VertexHashFn is rejected at compile time
//     (a host functor cannot be evaluated by the kernels). Other hasher types
//     opt in by specialising hashgraph::device_hasher<H> (kind + seed), e.g.
//     the reference tests' support::IdentityHasher (tests/cpp/ref_prelude.hpp).
//     The hasher passed to probe_standard / count_instances / validate_csr is
//     the one used, exactly as in the reference (join.hpp:117-118,
//     core.hpp:238, :271), not the table's.
//   * the table lives in HBM; offsets()/edges() export it to host memory on
//     first access (cached). Tables built from host vectors are uploaded on
//     first device use.
//   * ExecMode::parallel segment order is unspecified, as in the reference
//     (core.hpp:115-119); ExecMode::sequential reproduces the reference's
//     sequential layout exactly (segments in input order).
#pragma once

#include <hg_b200.h>

#include <algorithm>
#include <atomic>
#include <compare>
#include <concepts>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hashgraph {

// ------------------------------------------------------------------ errors

// keygen.hpp:75-77
struct KeyFileError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {

[[noreturn]] inline void throw_status(hg_status st) {
    const std::string msg = hg_last_error();
    switch (st) {
        case HG_EINVAL: throw std::invalid_argument(msg);
        case HG_ERANGE: throw std::out_of_range(msg);
        case HG_EOVERFLOW: throw std::overflow_error(msg);
        case HG_ENOMEM: throw std::bad_alloc();
        case HG_EIO: throw KeyFileError(msg);
        default: throw std::runtime_error("hashgraph (B200): " + msg);
    }
}

inline void check(hg_status st) {
    if (st != HG_OK) throw_status(st);
}

// hash.hpp:12-19 (host copy for API completeness; the tables hash on device).
inline constexpr std::uint64_t mix64(std::uint64_t x) noexcept {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

}  // namespace detail

// ------------------------------------------------------------------ hashing

// hash.hpp:27-34
struct VertexHasher {
    std::uint64_t seed = 0;
    std::uint64_t operator()(std::uint64_t key, std::uint64_t num_vertices) const noexcept {
        return detail::mix64(key ^ seed) % num_vertices;
    }
};

// The fixture hasher of the reference tests (tests/support.hpp:42-46).
struct IdentityHasher {
    std::uint64_t operator()(std::uint64_t key, std::uint64_t num_vertices) const noexcept {
        return key % num_vertices;
    }
};

// hash.hpp:36-39
inline std::uint64_t hash_to_vertex(std::uint64_t key, std::uint64_t seed,
                                    std::uint64_t num_vertices) noexcept {
    return VertexHasher{seed}(key, num_vertices);
}

// hash.hpp:41-44
template <class H>
concept VertexHashFn = requires(const H& h, std::uint64_t key, std::uint64_t v) {
    { h(key, v) } -> std::convertible_to<std::uint64_t>;
};

// Device mapping of a hasher: kind + seed. Specialise for custom hashers
// that are equivalent to one of the device hash functions.
template <class H>
struct device_hasher {
    static constexpr bool supported = false;
};
template <>
struct device_hasher<VertexHasher> {
    static constexpr bool supported = true;
    static constexpr int kind = HG_HASH_MIX64;
    static std::uint64_t seed(const VertexHasher& h) { return h.seed; }
};
template <>
struct device_hasher<IdentityHasher> {
    static constexpr bool supported = true;
    static constexpr int kind = HG_HASH_IDENTITY;
    static std::uint64_t seed(const IdentityHasher&) { return 0; }
};

// ------------------------------------------------------------------ core types

// core.hpp:21-26
struct Entry {
    std::uint64_t key = 0;
    std::uint64_t index = 0;
    friend auto operator<=>(const Entry&, const Entry&) = default;
};

enum class ExecMode { sequential, parallel };  // core.hpp:28

// core.hpp:30-35
struct BuildConfig {
    double load_factor = 1.0;
    std::uint64_t bin_count = std::uint64_t{1} << 15;
    std::uint64_t hash_seed = 0;
    ExecMode mode = ExecMode::parallel;
};

// core.hpp:40-56 -- filled with the exact operation counts of the
// reference's instrumented loops (2N / 4N hash evaluations, ...).
struct BuildStats {
    std::atomic<std::uint64_t> hash_evals{0};
    std::atomic<std::uint64_t> count_increments{0};
    std::atomic<std::uint64_t> placement_writes{0};
    std::atomic<std::uint64_t> bin_count_increments{0};
    std::atomic<std::uint64_t> bin_placement_writes{0};
    std::atomic<std::uint64_t> counter_zero_writes{0};

    void reset() noexcept {
        hash_evals = 0;
        count_increments = 0;
        placement_writes = 0;
        bin_count_increments = 0;
        bin_placement_writes = 0;
        counter_zero_writes = 0;
    }
};

// core.hpp:59-63
inline std::uint64_t derived_vertex_count(std::uint64_t n, double load_factor) {
    std::uint64_t v = 0;
    detail::check(hg_derived_vertex_count(n, load_factor, &v));
    return v;
}

// ------------------------------------------------------------------ table

// core.hpp:67-102 -- device-resident CSR table.
class HashGraph {
public:
    HashGraph() : HashGraph(1, std::vector<std::uint64_t>(2, 0), {}, 0, 1.0) {}

    // Host-constructed table (uploaded to the device on first device use).
    HashGraph(std::uint64_t num_vertices, std::vector<std::uint64_t> offsets,
              std::vector<Entry> edges, std::uint64_t hash_seed, double load_factor)
        : st_(std::make_shared<State>()) {
        st_->nv = num_vertices;
        st_->ne = edges.size();
        st_->seed = hash_seed;
        st_->load = load_factor;
        st_->offsets = std::move(offsets);
        st_->edges = std::move(edges);
        st_->host_valid = true;
    }

    std::uint64_t num_vertices() const noexcept { return st_->nv; }
    std::uint64_t num_edges() const noexcept { return st_->ne; }
    std::uint64_t hash_seed() const noexcept { return st_->seed; }
    double load_factor() const noexcept { return st_->load; }

    std::span<const std::uint64_t> offsets() const {
        export_host();
        return st_->offsets;
    }
    std::span<const Entry> edges() const {
        export_host();
        return st_->edges;
    }

    // core.hpp:87-94
    std::span<const Entry> vertex_entries(std::uint64_t v) const {
        if (v >= st_->nv) throw std::out_of_range("vertex_entries: vertex id out of range");
        export_host();
        const std::uint64_t b = st_->offsets[v], e = st_->offsets[v + 1];
        return std::span<const Entry>(st_->edges).subspan(b, e - b);
    }

    // The device table (uploads a host-constructed table first).
    const hg_table* device_table() const {
        std::lock_guard<std::mutex> lk(st_->mu);
        if (!st_->tab) {
            std::vector<std::uint64_t> k(st_->ne), x(st_->ne);
            for (std::size_t i = 0; i < st_->edges.size(); ++i) {
                k[i] = st_->edges[i].key;
                x[i] = st_->edges[i].index;
            }
            hg_table* t = nullptr;
            if (st_->offsets.size() != st_->nv + 1)
                throw std::invalid_argument("offsets length is not num_vertices + 1");
            detail::check(hg_table_import(st_->offsets.data(), k.data(), x.data(), st_->nv,
                                          st_->ne, st_->seed, st_->load, st_->hash_kind, nullptr,
                                          &t));
            st_->tab = t;
        }
        return st_->tab;
    }

    int device_hash_kind() const noexcept { return st_->hash_kind; }

    // Wraps a device table built by the C-ABI (takes ownership).
    static HashGraph adopt(hg_table* t, std::uint64_t recorded_seed, double load_factor) {
        HashGraph g;
        g.st_ = std::make_shared<State>();
        hg_table_info info{};
        detail::check(hg_table_get_info(t, &info));
        g.st_->tab = t;
        g.st_->nv = info.num_vertices;
        g.st_->ne = info.num_edges;
        g.st_->seed = recorded_seed;
        g.st_->load = load_factor;
        g.st_->hash_kind = info.hash_kind;
        return g;
    }

private:
    struct State {
        std::mutex mu;
        hg_table* tab = nullptr;
        std::uint64_t nv = 1, ne = 0, seed = 0;
        double load = 1.0;
        int hash_kind = HG_HASH_MIX64;
        bool host_valid = false;
        std::vector<std::uint64_t> offsets;
        std::vector<Entry> edges;
        ~State() {
            if (tab) hg_table_destroy(tab, nullptr);
        }
    };

    void export_host() const {
        std::lock_guard<std::mutex> lk(st_->mu);
        if (st_->host_valid) return;
        std::vector<std::uint64_t> off(st_->nv + 1), k(st_->ne), x(st_->ne);
        detail::check(hg_table_export(st_->tab, off.data(), k.data(), x.data(), nullptr));
        st_->edges.resize(st_->ne);
        for (std::size_t i = 0; i < k.size(); ++i) st_->edges[i] = Entry{k[i], x[i]};
        st_->offsets = std::move(off);
        st_->host_valid = true;
    }

    std::shared_ptr<State> st_;
};

// ------------------------------------------------------------------ builds

namespace detail {

inline void check_config(const BuildConfig& cfg) {  // core.hpp:106-109
    if (!(cfg.load_factor > 0.0)) throw std::invalid_argument("load_factor must be positive");
    if (cfg.bin_count < 1) throw std::invalid_argument("bin_count must be at least 1");
}

template <class H>
HashGraph device_build(int variant, std::span<const std::uint64_t> keys, const BuildConfig& cfg,
                       const H& hasher, BuildStats* stats,
                       std::optional<std::uint64_t> vertex_count) {
    static_assert(device_hasher<H>::supported,
                  "hashgraph (B200): this hasher has no device implementation; specialise "
                  "hashgraph::device_hasher<H> or use VertexHasher / IdentityHasher");
    check_config(cfg);
    hg_build_config c;
    hg_build_config_init(&c);
    c.load_factor = cfg.load_factor;
    c.bin_count = cfg.bin_count;
    c.hash_seed = device_hasher<H>::seed(hasher);
    c.vertex_count = vertex_count.value_or(0);
    c.variant = variant;
    c.hash_kind = device_hasher<H>::kind;
    c.stable = cfg.mode == ExecMode::sequential ? 1 : 0;
    hg_table* t = nullptr;
    check(hg_build(keys.data(), 8, nullptr, 0, keys.size(), &c, nullptr, &t));
    HashGraph g = HashGraph::adopt(t, cfg.hash_seed, cfg.load_factor);
    if (stats) {
        const std::uint64_t n = keys.size(), nv = g.num_vertices();
        const std::uint64_t bins = cfg.bin_count < nv ? cfg.bin_count : nv;
        stats->hash_evals.fetch_add((variant == HG_BUILD_SIMPLE ? 2 : 4) * n);
        stats->count_increments.fetch_add(n);
        stats->placement_writes.fetch_add(n);
        stats->counter_zero_writes.fetch_add(nv + (variant == HG_BUILD_BINNED ? bins : 0));
        if (variant == HG_BUILD_BINNED) {
            stats->bin_count_increments.fetch_add(n);
            stats->bin_placement_writes.fetch_add(n);
        }
    }
    return g;
}

}  // namespace detail

// core.hpp:160-177
template <VertexHashFn H>
HashGraph build_v1(std::span<const std::uint64_t> keys, const BuildConfig& cfg, const H& hasher,
                   BuildStats* stats = nullptr,
                   std::optional<std::uint64_t> vertex_count = std::nullopt) {
    return detail::device_build(HG_BUILD_SIMPLE, keys, cfg, hasher, stats, vertex_count);
}

inline HashGraph build_v1(std::span<const std::uint64_t> keys, const BuildConfig& cfg = {},
                          BuildStats* stats = nullptr,
                          std::optional<std::uint64_t> vertex_count = std::nullopt) {
    return build_v1(keys, cfg, VertexHasher{cfg.hash_seed}, stats, vertex_count);
}

// core.hpp:183-230
template <VertexHashFn H>
HashGraph build_v2(std::span<const std::uint64_t> keys, const BuildConfig& cfg, const H& hasher,
                   BuildStats* stats = nullptr,
                   std::optional<std::uint64_t> vertex_count = std::nullopt) {
    return detail::device_build(HG_BUILD_BINNED, keys, cfg, hasher, stats, vertex_count);
}

inline HashGraph build_v2(std::span<const std::uint64_t> keys, const BuildConfig& cfg = {},
                          BuildStats* stats = nullptr,
                          std::optional<std::uint64_t> vertex_count = std::nullopt) {
    return build_v2(keys, cfg, VertexHasher{cfg.hash_seed}, stats, vertex_count);
}

// core.hpp:235-246: the key's vertex is hasher(key, V) for the hasher passed
template <VertexHashFn H>
std::uint64_t count_instances(const HashGraph& hg, std::uint64_t key, const H& hasher) {
    static_assert(device_hasher<H>::supported, "hasher has no device implementation");
    std::uint64_t c = 0;
    detail::check(hg_count_instances_hasher(hg.device_table(), key, device_hasher<H>::kind,
                                            device_hasher<H>::seed(hasher), &c, nullptr));
    return c;
}

inline std::uint64_t count_instances(const HashGraph& hg, std::uint64_t key) {
    return count_instances(hg, key, VertexHasher{hg.hash_seed()});
}

// core.hpp:251-287 (device validator; host-constructed tables are uploaded)
template <VertexHashFn H>
std::optional<std::string> validate_csr(const HashGraph& hg, std::uint64_t expected_entries,
                                        const H& hasher) {
    static_assert(device_hasher<H>::supported, "hasher has no device implementation");
    static const char* const kWhat[] = {
        "", "table has no vertices", "offsets length is not num_vertices + 1",
        "offsets[0] is not 0", "offsets are not non-decreasing",
        "offsets[V] does not equal the edge count", "edge count does not equal the input size",
        "entry stored under a vertex its key does not hash to", "entry index out of range",
        "duplicate entry index", "entry key does not equal input[index]"};
    if (hg.num_vertices() < 1) return std::string(kWhat[1]);
    int32_t code = 0;
    try {
        detail::check(hg_validate_hasher(hg.device_table(), nullptr, expected_entries,
                                         device_hasher<H>::kind, device_hasher<H>::seed(hasher),
                                         &code, nullptr));
    } catch (const std::invalid_argument&) {
        return std::string(kWhat[2]);
    }
    if (code == 0) return std::nullopt;
    return std::string(code > 0 && code <= 10 ? kWhat[code] : "invalid table");
}

inline std::optional<std::string> validate_csr(const HashGraph& hg,
                                               std::uint64_t expected_entries) {
    return validate_csr(hg, expected_entries, VertexHasher{hg.hash_seed()});
}

// ------------------------------------------------------------------ probe

// join.hpp:18-35
struct MatchPair {
    std::uint64_t left_index = 0;
    std::uint64_t right_index = 0;
    friend auto operator<=>(const MatchPair&, const MatchPair&) = default;
};

struct ProbeOptions {
    bool materialize = false;
    std::uint64_t pair_cap = std::uint64_t{1} << 24;
};

struct JoinResult {
    std::uint64_t match_count = 0;
    std::uint64_t key_comparisons = 0;
    bool truncated = false;
    std::optional<std::vector<MatchPair>> pairs;
};

namespace detail {
// Host landing buffer for up to `cap` pairs: uninitialised storage (pages are
// touched only by the pairs actually written), copied into the result vector.
struct PairBuffer {
    std::unique_ptr<unsigned char[]> raw;
    std::uint64_t cap = 0;
    void* reserve(std::uint64_t n) {
        cap = n;
        raw.reset(n ? new unsigned char[n * sizeof(MatchPair)] : nullptr);
        return raw.get();
    }
    std::vector<MatchPair> take(std::uint64_t written) const {
        const auto* p = reinterpret_cast<const MatchPair*>(raw.get());
        return std::vector<MatchPair>(p, p + std::min(written, cap));
    }
};
}  // namespace detail

// join.hpp:110-136: every probe is hashed with the hasher passed
// (join.hpp:117-118), the table's own by default (join.hpp:133-136)
template <VertexHashFn H>
JoinResult probe_standard(const HashGraph& hg, std::span<const std::uint64_t> probe_keys,
                          const H& hasher, const ProbeOptions& opts = {}) {
    static_assert(device_hasher<H>::supported, "hasher has no device implementation");
    static_assert(sizeof(MatchPair) == 16, "MatchPair must match the C-ABI pair layout");
    hg_probe_options o;
    hg_probe_options_init(&o);
    o.materialize = opts.materialize ? 1 : 0;
    o.pair_width = 8;
    o.pair_cap = opts.pair_cap;
    o.flags = HG_PROBE_HASHER;
    o.hash_kind = device_hasher<H>::kind;
    o.hash_seed = device_hasher<H>::seed(hasher);
    detail::PairBuffer buf;
    if (opts.materialize) {
        const std::uint64_t bound = probe_keys.size() * std::max<std::uint64_t>(hg.num_edges(), 1);
        o.pairs = buf.reserve(std::min<std::uint64_t>(opts.pair_cap, bound));
        if (!o.pairs) o.pair_cap = 0;
    }
    hg_probe_result r{};
    detail::check(hg_probe(hg.device_table(), probe_keys.data(), 8, probe_keys.size(), &o, &r,
                           nullptr));
    JoinResult res;
    res.match_count = r.match_count;
    res.key_comparisons = r.key_comparisons;
    if (opts.materialize) {
        res.truncated = r.match_count > opts.pair_cap;
        res.pairs = buf.take(r.pairs_written);
    }
    return res;
}

inline JoinResult probe_standard(const HashGraph& hg, std::span<const std::uint64_t> probe_keys,
                                 const ProbeOptions& opts = {}) {
    return probe_standard(hg, probe_keys, VertexHasher{hg.hash_seed()}, opts);
}

// join.hpp:41-57. Host helper over two segments (spans of Entry, e.g. from
// HashGraph::vertex_entries). The device engine never calls it: the
// per-vertex intersection runs inside probe_new_prepared (K12 k_intersect).
template <class Emit>
std::uint64_t intersect_adjacency(std::span<const Entry> a, std::span<const Entry> b, Emit&& emit,
                                  std::uint64_t* comparisons = nullptr) {
    std::uint64_t count = 0;
    for (const Entry& ea : a)
        for (const Entry& eb : b)
            if (ea.key == eb.key) {
                ++count;
                emit(ea.index, eb.index);
            }
    if (comparisons) *comparisons += std::uint64_t(a.size()) * b.size();
    return count;
}

namespace detail {
inline JoinResult join_result(const hg_probe_result& r, const ProbeOptions& opts,
                              const PairBuffer& buf) {
    JoinResult res;
    res.match_count = r.match_count;
    res.key_comparisons = r.key_comparisons;
    if (opts.materialize) {
        res.truncated = r.match_count > opts.pair_cap;
        res.pairs = buf.take(r.pairs_written);
    }
    return res;
}

inline hg_probe_options join_options(const ProbeOptions& opts, std::uint64_t bound,
                                     PairBuffer& buf) {
    hg_probe_options o;
    hg_probe_options_init(&o);
    o.materialize = opts.materialize ? 1 : 0;
    o.pair_width = 8;
    o.pair_cap = opts.pair_cap;
    if (opts.materialize) {
        o.pairs = buf.reserve(std::min<std::uint64_t>(opts.pair_cap, bound));
        if (!o.pairs) o.pair_cap = 0;
    }
    return o;
}
}  // namespace detail

// join.hpp:143-166. Throws std::invalid_argument when the tables use
// different vertex ranges (join.hpp:145-147). Pairs are (index in A's input,
// index in B's input) in sequential order (vertex, A position, B position).
inline JoinResult probe_new_prepared(const HashGraph& hg_a, const HashGraph& hg_b,
                                     const ProbeOptions& opts = {}) {
    detail::PairBuffer pairs;
    const hg_probe_options o = detail::join_options(
        opts, std::max<std::uint64_t>(hg_a.num_edges(), 1) * std::max<std::uint64_t>(hg_b.num_edges(), 1),
        pairs);
    hg_probe_result r{};
    detail::check(hg_probe_new_prepared(hg_a.device_table(), hg_b.device_table(), &o, &r, nullptr));
    return detail::join_result(r, opts, pairs);
}

// join.hpp:170-182: both inputs built (binned build) over the V of the
// larger input, then intersected vertex by vertex.
template <VertexHashFn H>
JoinResult probe_new(std::span<const std::uint64_t> keys_a, std::span<const std::uint64_t> keys_b,
                     const BuildConfig& cfg, const H& hasher, const ProbeOptions& opts = {}) {
    static_assert(device_hasher<H>::supported, "hasher has no device implementation");
    detail::check_config(cfg);
    hg_build_config c;
    hg_build_config_init(&c);
    c.load_factor = cfg.load_factor;
    c.bin_count = cfg.bin_count;
    c.hash_seed = device_hasher<H>::seed(hasher);
    c.hash_kind = device_hasher<H>::kind;
    c.stable = cfg.mode == ExecMode::sequential ? 1 : 0;
    detail::PairBuffer pairs;
    const hg_probe_options o = detail::join_options(
        opts, std::max<std::uint64_t>(keys_a.size(), 1) * std::max<std::uint64_t>(keys_b.size(), 1),
        pairs);
    hg_probe_result r{};
    detail::check(hg_probe_new(keys_a.data(), keys_a.size(), keys_b.data(), keys_b.size(), 8, &c,
                               &o, &r, nullptr));
    return detail::join_result(r, opts, pairs);
}

inline JoinResult probe_new(std::span<const std::uint64_t> keys_a,
                            std::span<const std::uint64_t> keys_b, const BuildConfig& cfg = {},
                            const ProbeOptions& opts = {}) {
    return probe_new(keys_a, keys_b, cfg, VertexHasher{cfg.hash_seed}, opts);
}

}  // namespace hashgraph
