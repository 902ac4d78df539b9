/*
 * hg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the HashGraph reference hot path, used exclusively as
 * the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. Nothing in the product path (paper_1907_02900_b200/, the
 * C-ABI library, include/) may link or call this file.
 *
 * Every function follows the sequential (ExecMode::sequential, threads == 1)
 * semantics of the reference headers under /root/reference/proj/include:
 * with one thread the reference's parallel_for degenerates to a plain loop
 * (parallel.hpp:60-63, 90-96), so the outputs below are the reference's
 * byte-for-byte, including the intra-segment order (ascending input index).
 *
 * Parity of this restatement is pinned against (a) SURVEY.md Appendix A golden
 * vectors (computed with the reference headers) and (b) oracle/_ref, the
 * reference headers themselves compiled by oracle/Makefile -- see
 * tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HGO_OK 0
#define HGO_EINVAL 1
#define HGO_ENOMEM 4

enum { HGO_HASH_MIX64 = 0, HGO_HASH_IDENTITY = 1 };

/* hash.hpp:12-19 detail::mix64 (murmur3 fmix64 constants) */
uint64_t hgo_mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

/* hash.hpp:30-39 VertexHasher / hash_to_vertex: mix64(key ^ seed) % V.
 * hash_kind IDENTITY restates tests/support.hpp:42-46 (key % V). */
uint64_t hgo_vertex(uint64_t key, uint64_t seed, uint64_t nv, int hash_kind) {
    if (hash_kind == HGO_HASH_IDENTITY) return key % nv;
    return hgo_mix64(key ^ seed) % nv;
}

uint64_t hgo_hash_to_vertex(uint64_t key, uint64_t seed, uint64_t nv) {
    return hgo_vertex(key, seed, nv, HGO_HASH_MIX64);
}

/* Vectorised hash_to_vertex over an array (test convenience). */
void hgo_vertices(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t nv, int hash_kind,
                  uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = hgo_vertex(keys[i], seed, nv, hash_kind);
}

/* core.hpp:59-63 derived_vertex_count: max(1, floor(n / load)) in double. */
int hgo_derived_vertex_count(uint64_t n, double load, uint64_t* out) {
    if (!(load > 0.0)) return HGO_EINVAL;
    const double v = floor((double)n / load);
    *out = v < 1.0 ? 1 : (uint64_t)v;
    return HGO_OK;
}

/* core.hpp:120-153 detail::create_table, sequential: count (126-133), exclusive
 * scan (135 -> parallel.hpp:147-157), zero (137), place (140-150).
 * keys_at/idx_at are the entry sources (input array for V1, reorg for V2).
 * Output: offsets[V+1], ekeys[n], eidx[n]. */
static int create_table(const uint64_t* key_at, const uint64_t* idx_at, uint64_t n, uint64_t nv,
                        uint64_t seed, int hk, uint64_t* offsets, uint64_t* ekeys,
                        uint64_t* eidx) {
    uint64_t* counts = (uint64_t*)calloc(nv ? nv : 1, sizeof(uint64_t));
    if (!counts) return HGO_ENOMEM;
    for (uint64_t i = 0; i < n; ++i) counts[hgo_vertex(key_at[i], seed, nv, hk)]++;
    uint64_t run = 0;
    for (uint64_t v = 0; v < nv; ++v) {
        offsets[v] = run;
        run += counts[v];
    }
    offsets[nv] = run;
    memset(counts, 0, nv * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t k = key_at[i];
        const uint64_t v = hgo_vertex(k, seed, nv, hk);
        const uint64_t pos = offsets[v] + counts[v]++;
        ekeys[pos] = k;
        eidx[pos] = idx_at ? idx_at[i] : i;
    }
    free(counts);
    return HGO_OK;
}

/* core.hpp:160-177 build_v1 (sequential). nv must already be resolved by the
 * caller (vertex_count override or derived_vertex_count). */
int hgo_build_v1(const uint64_t* keys, uint64_t n, uint64_t nv, uint64_t seed, int hk,
                 uint64_t* offsets, uint64_t* ekeys, uint64_t* eidx) {
    if (nv < 1) return HGO_EINVAL;
    return create_table(keys, NULL, n, nv, seed, hk, offsets, ekeys, eidx);
}

/* core.hpp:183-230 build_v2 (sequential): bins = min(bin_count, V),
 * bin_size = ceil(V / bins) (192-193); bin count (195-203); scan (205);
 * bin scatter into reorg (210-219); create_table over reorg (221-223). */
int hgo_build_v2(const uint64_t* keys, uint64_t n, uint64_t nv, uint64_t bin_count,
                 uint64_t seed, int hk, uint64_t* offsets, uint64_t* ekeys, uint64_t* eidx) {
    if (nv < 1 || bin_count < 1) return HGO_EINVAL;
    const uint64_t bins = bin_count < nv ? bin_count : nv;
    const uint64_t bin_size = (nv + bins - 1) / bins;
    uint64_t* bc = (uint64_t*)calloc(bins, sizeof(uint64_t));
    uint64_t* bo = (uint64_t*)malloc(bins * sizeof(uint64_t));
    uint64_t* rk = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* ri = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    int rc = HGO_ENOMEM;
    if (!bc || !bo || !rk || !ri) goto out;
    for (uint64_t i = 0; i < n; ++i) bc[hgo_vertex(keys[i], seed, nv, hk) / bin_size]++;
    uint64_t run = 0;
    for (uint64_t b = 0; b < bins; ++b) {
        bo[b] = run;
        run += bc[b];
    }
    memset(bc, 0, bins * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t b = hgo_vertex(keys[i], seed, nv, hk) / bin_size;
        const uint64_t pos = bo[b] + bc[b]++;
        rk[pos] = keys[i];
        ri[pos] = i;
    }
    rc = create_table(rk, ri, n, nv, seed, hk, offsets, ekeys, eidx);
out:
    free(bc);
    free(bo);
    free(rk);
    free(ri);
    return rc;
}

/* core.hpp:235-246 count_instances. */
uint64_t hgo_count_instances(const uint64_t* offsets, const uint64_t* ekeys, uint64_t nv,
                             uint64_t seed, int hk, uint64_t key) {
    const uint64_t v = hgo_vertex(key, seed, nv, hk);
    uint64_t c = 0;
    for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) c += ekeys[j] == key;
    return c;
}

/* join.hpp:110-136 probe_standard + detail::ProbeAccumulator (63-103), one
 * chunk: match_count and key_comparisons are exact; pairs are emitted as
 * MatchPair{left = entry index, right = probe position} (join.hpp:125) in
 * probe order while slot < cap (join.hpp:71-74). pairs may be NULL (count
 * only). per_probe (nullable) receives each probe's match count
 * (= count_instances, core.hpp:235-246). */
void hgo_probe_standard(const uint64_t* offsets, const uint64_t* ekeys, const uint64_t* eidx,
                        uint64_t nv, uint64_t seed, int hk, const uint64_t* probes, uint64_t m,
                        uint64_t cap, uint64_t* pairs, uint64_t* per_probe, uint64_t* match_count,
                        uint64_t* comparisons, uint64_t* written) {
    uint64_t count = 0, cmp = 0, slot = 0;
    for (uint64_t j = 0; j < m; ++j) {
        const uint64_t key = probes[j];
        const uint64_t v = hgo_vertex(key, seed, nv, hk);
        uint64_t c = 0;
        for (uint64_t t = offsets[v]; t < offsets[v + 1]; ++t) {
            ++cmp;
            if (ekeys[t] == key) {
                ++c;
                if (pairs && slot < cap) {
                    pairs[2 * slot] = eidx[t];
                    pairs[2 * slot + 1] = j;
                }
                ++slot;
            }
        }
        if (per_probe) per_probe[j] = c;
        count += c;
    }
    *match_count = count;
    *comparisons = cmp;
    if (written) *written = pairs ? (slot < cap ? slot : cap) : 0;
}

/* join.hpp:41-57 intersect_adjacency driven by join.hpp:143-166
 * probe_new_prepared, one chunk: for each vertex v (ascending), every
 * (a, b) entry pair of the two segments is compared on the full key
 * (|A_v| * |B_v| comparisons); a match emits MatchPair{left = A entry index,
 * right = B entry index} while slot < cap. Order: vertex, then A position,
 * then B position -- the sequential emission order of the reference. */
void hgo_probe_new_prepared(const uint64_t* offs_a, const uint64_t* keys_a, const uint64_t* idx_a,
                            const uint64_t* offs_b, const uint64_t* keys_b, const uint64_t* idx_b,
                            uint64_t nv, uint64_t cap, uint64_t* pairs, uint64_t* match_count,
                            uint64_t* comparisons, uint64_t* written) {
    uint64_t count = 0, cmp = 0, slot = 0;
    for (uint64_t v = 0; v < nv; ++v) {
        for (uint64_t i = offs_a[v]; i < offs_a[v + 1]; ++i) {
            for (uint64_t j = offs_b[v]; j < offs_b[v + 1]; ++j) {
                ++cmp;
                if (keys_a[i] == keys_b[j]) {
                    ++count;
                    if (pairs && slot < cap) {
                        pairs[2 * slot] = idx_a[i];
                        pairs[2 * slot + 1] = idx_b[j];
                    }
                    ++slot;
                }
            }
        }
    }
    *match_count = count;
    *comparisons = cmp;
    if (written) *written = pairs ? (slot < cap ? slot : cap) : 0;
}

/* core.hpp:251-282 validate_csr, plus the key-consistency check SURVEY.md
 * 8(c) adds (edges[j].key == input[edges[j].index]) when input != NULL.
 * Returns 0 when valid, else the number of the first violated invariant. */
int hgo_validate_csr(const uint64_t* offsets, const uint64_t* ekeys, const uint64_t* eidx,
                     uint64_t nv, uint64_t num_edges, uint64_t expected, uint64_t seed, int hk,
                     const uint64_t* input) {
    if (nv < 1) return 1;
    if (offsets[0] != 0) return 3;
    for (uint64_t v = 0; v < nv; ++v)
        if (offsets[v] > offsets[v + 1]) return 4;
    if (offsets[nv] != num_edges) return 5;
    if (num_edges != expected) return 6;
    for (uint64_t v = 0; v < nv; ++v)
        for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j)
            if (hgo_vertex(ekeys[j], seed, nv, hk) != v) return 7;
    uint8_t* seen = (uint8_t*)calloc(num_edges ? num_edges : 1, 1);
    if (!seen) return 100;
    int rc = 0;
    for (uint64_t j = 0; j < num_edges; ++j) {
        if (eidx[j] >= num_edges) { rc = 8; break; }
        if (seen[eidx[j]]) { rc = 9; break; }
        seen[eidx[j]] = 1;
        if (input && input[eidx[j]] != ekeys[j]) { rc = 10; break; }
    }
    free(seen);
    return rc;
}

/* parallel.hpp:141-192 exclusive_scan_impl (sequential fold): out[n+1];
 * returns 3 (overflow) when the running sum wraps 64 bits (parallel.hpp:153). */
int hgo_exclusive_prefix_sum(const uint64_t* counts, uint64_t n, uint64_t* out) {
    uint64_t run = 0;
    for (uint64_t i = 0; i < n; ++i) {
        out[i] = run;
        run += counts[i];
        if (run < counts[i]) return 3;
    }
    out[n] = run;
    return HGO_OK;
}

/* baselines.hpp:138-163 sort_merge_join_count (hash-free join cardinality). */
static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}
uint64_t hgo_sort_merge_join_count(const uint64_t* a, uint64_t na, const uint64_t* b,
                                   uint64_t nb) {
    uint64_t* sa = (uint64_t*)malloc((na ? na : 1) * 8);
    uint64_t* sb = (uint64_t*)malloc((nb ? nb : 1) * 8);
    memcpy(sa, a, na * 8);
    memcpy(sb, b, nb * 8);
    qsort(sa, na, 8, cmp_u64);
    qsort(sb, nb, 8, cmp_u64);
    uint64_t count = 0, i = 0, j = 0;
    while (i < na && j < nb) {
        if (sa[i] < sb[j]) ++i;
        else if (sb[j] < sa[i]) ++j;
        else {
            const uint64_t k = sa[i];
            uint64_t ra = 0, rb = 0;
            while (i < na && sa[i] == k) ++i, ++ra;
            while (j < nb && sb[j] == k) ++j, ++rb;
            count += ra * rb;
        }
    }
    free(sa);
    free(sb);
    return count;
}

/* std::mt19937_64 (the standard-specified engine used by keygen.hpp:59-73 and
 * tests/support.hpp:61-68), restated for the config-1 known answers. */
typedef struct { uint64_t mt[312]; int idx; } hgo_mt64;
static void mt64_seed(hgo_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt64_next(hgo_mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* Fills out[0..n) with successive mt19937_64(seed) outputs; mask_u32 != 0
 * truncates each to uint32 (SURVEY.md Appendix A config-1 generator). */
void hgo_mt19937_64(uint64_t seed, uint64_t skip, uint64_t* out, uint64_t n, int mask_u32) {
    hgo_mt64 s;
    mt64_seed(&s, seed);
    for (uint64_t i = 0; i < skip; ++i) mt64_next(&s);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t x = mt64_next(&s);
        out[i] = mask_u32 ? (x & 0xFFFFFFFFULL) : x;
    }
}

/* keygen.hpp:46-52 bounded_draw + generate(uniform_multiplicity) (59-73). */
int hgo_generate_uniform(uint64_t n, double multiplicity, uint64_t seed, uint64_t* out) {
    if (!(multiplicity > 0.0)) return HGO_EINVAL;
    long long k = llround((double)n / multiplicity);
    const uint64_t range = k < 1 ? 1 : (uint64_t)k;
    hgo_mt64 s;
    mt64_seed(&s, seed);
    const uint64_t limit = ~0ULL - ~0ULL % range;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t x;
        do x = mt64_next(&s); while (x >= limit);
        out[i] = 1 + x % range;
    }
    return HGO_OK;
}

/* SURVEY.md Appendix B splitmix64(seed, i) counter-based generator. */
uint64_t hgo_splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
void hgo_splitmix_fill(uint64_t seed, uint64_t start, uint64_t n, int mask_u32, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t x = hgo_splitmix64(seed, start + i);
        out[i] = mask_u32 ? (x & 0xFFFFFFFFULL) : x;
    }
}

/* Appendix A fold: h = 0; for x: h = mix64(h ^ x) + 0x9e3779b97f4a7c15. */
uint64_t hgo_fold(const uint64_t* xs, uint64_t n, uint64_t h) {
    for (uint64_t i = 0; i < n; ++i) h = hgo_mix64(h ^ xs[i]) + 0x9e3779b97f4a7c15ULL;
    return h;
}
