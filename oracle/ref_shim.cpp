// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim around the UNMODIFIED reference headers
// (/root/reference/proj/include/hashgraph/*.hpp), compiled where they lie by
// oracle/Makefile into oracle/_ref/libhgref.so. No reference source is copied
// into this repository: this file only includes the headers and forwards.
//
// Used (a) by tests/test_oracle.py to pin the plain-C restatement
// (oracle/hg_oracle.c) against the reference itself, and (b) by bench.py's
// cpu_baseline / --impl reference legs to time the reference's own parallel
// std::thread implementation on the host cores (HASHGRAPH_THREADS governs the
// thread count, parallel.hpp:25-34).
#include <hashgraph/hashgraph.hpp>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <vector>

using namespace hashgraph;

namespace {
struct IdentityHasher {  // tests/support.hpp:42-46 restated for fixtures
    std::uint64_t operator()(std::uint64_t key, std::uint64_t nv) const noexcept {
        return key % nv;
    }
};
}  // namespace

extern "C" {

std::uint64_t hgr_mix64(std::uint64_t x) { return detail::mix64(x); }

std::uint64_t hgr_hash_to_vertex(std::uint64_t key, std::uint64_t seed, std::uint64_t nv) {
    return hash_to_vertex(key, seed, nv);
}

int hgr_derived_vertex_count(std::uint64_t n, double load, std::uint64_t* out) {
    try {
        *out = derived_vertex_count(n, load);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// variant 1 = build_v1, 2 = build_v2; sequential != 0 -> ExecMode::sequential;
// vertex_count 0 -> derived; hash_kind 1 -> identity hasher.
// Returns an owned HashGraph* (or nullptr, *err set: 1 invalid_argument).
void* hgr_build(const std::uint64_t* keys, std::uint64_t n, int variant, double load,
                std::uint64_t bins, std::uint64_t seed, int sequential,
                std::uint64_t vertex_count, int hash_kind, int* err) {
    *err = 0;
    BuildConfig cfg;
    cfg.load_factor = load;
    cfg.bin_count = bins;
    cfg.hash_seed = seed;
    cfg.mode = sequential ? ExecMode::sequential : ExecMode::parallel;
    std::optional<std::uint64_t> vc;
    if (vertex_count) vc = vertex_count;
    std::span<const std::uint64_t> ks(keys, n);
    try {
        HashGraph hg;
        if (hash_kind == 1) {
            hg = variant == 2 ? build_v2(ks, cfg, IdentityHasher{}, nullptr, vc)
                              : build_v1(ks, cfg, IdentityHasher{}, nullptr, vc);
        } else {
            hg = variant == 2 ? build_v2(ks, cfg, nullptr, vc) : build_v1(ks, cfg, nullptr, vc);
        }
        return new HashGraph(std::move(hg));
    } catch (const std::invalid_argument&) {
        *err = 1;
    } catch (...) {
        *err = 99;
    }
    return nullptr;
}

void hgr_free(void* t) { delete static_cast<HashGraph*>(t); }

void hgr_info(const void* t, std::uint64_t* nv, std::uint64_t* ne) {
    const auto* hg = static_cast<const HashGraph*>(t);
    *nv = hg->num_vertices();
    *ne = hg->num_edges();
}

void hgr_export(const void* t, std::uint64_t* offsets, std::uint64_t* keys, std::uint64_t* idx) {
    const auto* hg = static_cast<const HashGraph*>(t);
    std::memcpy(offsets, hg->offsets().data(), hg->offsets().size() * 8);
    const auto e = hg->edges();
    for (std::size_t i = 0; i < e.size(); ++i) {
        keys[i] = e[i].key;
        idx[i] = e[i].index;
    }
}

// probe_standard (join.hpp:133-136). pairs_out (nullable, 2*cap u64) gets
// (left, right) pairs when materialize != 0; *npairs = pairs kept.
void hgr_probe(const void* t, const std::uint64_t* probes, std::uint64_t m, int materialize,
               std::uint64_t cap, std::uint64_t* match_count, std::uint64_t* comparisons,
               int* truncated, std::uint64_t* pairs_out, std::uint64_t* npairs) {
    const auto* hg = static_cast<const HashGraph*>(t);
    ProbeOptions opts;
    opts.materialize = materialize != 0;
    opts.pair_cap = cap;
    const JoinResult r = probe_standard(*hg, std::span<const std::uint64_t>(probes, m), opts);
    *match_count = r.match_count;
    *comparisons = r.key_comparisons;
    *truncated = r.truncated ? 1 : 0;
    *npairs = 0;
    if (r.pairs) {
        *npairs = r.pairs->size();
        if (pairs_out) {
            for (std::size_t i = 0; i < r.pairs->size(); ++i) {
                pairs_out[2 * i] = (*r.pairs)[i].left_index;
                pairs_out[2 * i + 1] = (*r.pairs)[i].right_index;
            }
        }
    }
}

namespace {
void copy_result(const JoinResult& r, std::uint64_t* match_count, std::uint64_t* comparisons,
                 int* truncated, std::uint64_t* pairs_out, std::uint64_t* npairs) {
    *match_count = r.match_count;
    *comparisons = r.key_comparisons;
    *truncated = r.truncated ? 1 : 0;
    *npairs = 0;
    if (r.pairs) {
        *npairs = r.pairs->size();
        if (pairs_out) {
            for (std::size_t i = 0; i < r.pairs->size(); ++i) {
                pairs_out[2 * i] = (*r.pairs)[i].left_index;
                pairs_out[2 * i + 1] = (*r.pairs)[i].right_index;
            }
        }
    }
}
}  // namespace

// probe_new_prepared (join.hpp:143-166). Returns 0, or 1 on invalid_argument
// (mismatched vertex ranges, join.hpp:145-147).
int hgr_probe_new_prepared(const void* a, const void* b, int materialize, std::uint64_t cap,
                           std::uint64_t* match_count, std::uint64_t* comparisons,
                           int* truncated, std::uint64_t* pairs_out, std::uint64_t* npairs) {
    ProbeOptions opts;
    opts.materialize = materialize != 0;
    opts.pair_cap = cap;
    try {
        copy_result(probe_new_prepared(*static_cast<const HashGraph*>(a),
                                       *static_cast<const HashGraph*>(b), opts),
                    match_count, comparisons, truncated, pairs_out, npairs);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// probe_new (join.hpp:170-182): both sides built with build_v2 over the
// shared V of the larger input. hash_kind 1 -> identity hasher.
int hgr_probe_new(const std::uint64_t* a, std::uint64_t na, const std::uint64_t* b,
                  std::uint64_t nb, double load, std::uint64_t bins, std::uint64_t seed,
                  int hash_kind, int materialize, std::uint64_t cap, std::uint64_t* match_count,
                  std::uint64_t* comparisons, int* truncated, std::uint64_t* pairs_out,
                  std::uint64_t* npairs) {
    BuildConfig cfg;
    cfg.load_factor = load;
    cfg.bin_count = bins;
    cfg.hash_seed = seed;
    ProbeOptions opts;
    opts.materialize = materialize != 0;
    opts.pair_cap = cap;
    std::span<const std::uint64_t> sa(a, na), sb(b, nb);
    try {
        const JoinResult r = hash_kind == 1 ? probe_new(sa, sb, cfg, IdentityHasher{}, opts)
                                            : probe_new(sa, sb, cfg, opts);
        copy_result(r, match_count, comparisons, truncated, pairs_out, npairs);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

std::uint64_t hgr_count_instances(const void* t, std::uint64_t key) {
    return count_instances(*static_cast<const HashGraph*>(t), key);
}

// validate_csr (core.hpp:284-287): 0 valid, 1 invalid.
int hgr_validate(const void* t, std::uint64_t expected) {
    return validate_csr(*static_cast<const HashGraph*>(t), expected).has_value() ? 1 : 0;
}

std::uint64_t hgr_sort_merge_join_count(const std::uint64_t* a, std::uint64_t na,
                                        const std::uint64_t* b, std::uint64_t nb) {
    return sort_merge_join_count(std::span<const std::uint64_t>(a, na),
                                 std::span<const std::uint64_t>(b, nb));
}

// exclusive_prefix_sum (parallel.hpp:199-203): 0 ok, 3 overflow_error.
int hgr_exclusive_prefix_sum(const std::uint64_t* counts, std::uint64_t n, unsigned threads,
                             std::uint64_t* out) {
    try {
        const auto r = exclusive_prefix_sum(std::span<const std::uint64_t>(counts, n), threads);
        std::memcpy(out, r.data(), r.size() * 8);
        return 0;
    } catch (const std::overflow_error&) {
        return 3;
    }
}

// keygen.hpp:59-73 generate().
int hgr_generate(int kind, std::uint64_t n, double mult, std::uint64_t seed, std::uint64_t* out) {
    KeySpec spec;
    spec.kind = kind == 1 ? KeyKind::uniform_multiplicity : KeyKind::sequence;
    spec.n = n;
    spec.multiplicity = mult;
    spec.seed = seed;
    try {
        const auto k = generate(spec);
        std::memcpy(out, k.data(), k.size() * 8);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

unsigned hgr_resolve_threads() { return resolve_threads(); }

// write_keys / read_keys (keygen.hpp:100-130): 0 ok, 1 KeyFileError.
int hgr_write_keys(const char* path, const std::uint64_t* keys, std::uint64_t n) {
    try {
        write_keys(path, std::span<const std::uint64_t>(keys, n));
        return 0;
    } catch (const KeyFileError&) {
        return 1;
    }
}

// *n = key count; keys (nullable, capacity cap) receives them.
int hgr_read_keys(const char* path, std::uint64_t* keys, std::uint64_t cap, std::uint64_t* n) {
    try {
        const auto k = read_keys(path);
        *n = k.size();
        if (keys && k.size() <= cap) std::memcpy(keys, k.data(), k.size() * 8);
        return 0;
    } catch (const KeyFileError&) {
        return 1;
    }
}

}  // extern "C"
