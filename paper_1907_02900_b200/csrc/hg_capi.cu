// hg_capi.cu -- the extern "C" boundary (include/hg_b200.h).
//
// Owns table lifetime, host/device staging, config validation with the
// reference's exact error semantics, and the translation of CUDA failures
// into hg_status + hg_last_error. All compute is in the kernel TUs.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hg_b200.h"
#include "hg_internal.h"

struct hg_table {
    hg::TableDesc d;
    double load_factor = 1.0;
    int device = 0;
    void* alloc_offs = nullptr;
};

namespace {

thread_local std::string g_err;

hg_status fail(hg_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

hg_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? HG_ENOMEM : HG_ECUDA, "%s: %s", where,
                cudaGetErrorString(e));
}

#define HG_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

// A device view of a caller array: either the caller's device pointer or a
// stream-ordered staging copy of host data (freed by release()).
struct DevIn {
    const void* ptr = nullptr;
    void* owned = nullptr;
    cudaError_t stage(const void* p, size_t bytes, cudaStream_t s) {
        if (!p || bytes == 0 || is_device_ptr(p)) {
            ptr = p;
            return cudaSuccess;
        }
        cudaError_t e = cudaMallocAsync(&owned, bytes, s);
        if (e != cudaSuccess) return e;
        e = cudaMemcpyAsync(owned, p, bytes, cudaMemcpyHostToDevice, s);
        ptr = owned;
        return e;
    }
    void release(cudaStream_t s) {
        if (owned) cudaFreeAsync(owned, s);
        owned = nullptr;
    }
};

int ensure_device_ready() {
    static thread_local int checked = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (checked != dev) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        if (major < 10) return -2;
        // Keep freed stream-ordered allocations in the pool (no re-map cost
        // between builds).
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        checked = dev;
    }
    return dev;
}

hg_status need_device(int* dev) {
    const int d = ensure_device_ready();
    if (d == -1) return fail(HG_ECUDA, "no CUDA device available (no CPU fallback)");
    if (d == -2) return fail(HG_ECUDA, "device is not sm_100-class (compiled for sm_100a only)");
    *dev = d;
    return HG_OK;
}

template <typename T>
__global__ void k_widen(const T* in, uint64_t* out, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = uint64_t(in[i]);
}

__global__ void k_narrow_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = in[i];
}

cudaError_t widen_to(const void* src, int width, uint64_t n, uint64_t* dst, cudaStream_t s) {
    if (n == 0 || !dst) return cudaSuccess;
    const bool dev_out = is_device_ptr(dst);
    uint64_t* d = dst;
    if (!dev_out) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), n * 8, s);
        if (e != cudaSuccess) return e;
    }
    if (width == 8) {
        cudaMemcpyAsync(d, src, n * 8, cudaMemcpyDeviceToDevice, s);
    } else {
        const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 16));
        k_widen<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(src), d, n);
    }
    cudaError_t e = cudaGetLastError();
    if (!dev_out) {
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, d, n * 8, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(d, s);
    }
    return e;
}

}  // namespace

extern "C" {

int32_t hg_abi_version(void) { return HG_ABI_VERSION; }

const char* hg_last_error(void) { return g_err.c_str(); }

void hg_build_config_init(hg_build_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof *cfg);
    cfg->load_factor = 1.0;
    cfg->bin_count = uint64_t(1) << 15;
    cfg->hash_seed = 0;
    cfg->vertex_count = 0;
    cfg->variant = HG_BUILD_SIMPLE;
    cfg->hash_kind = HG_HASH_MIX64;
    cfg->stable = 0;
    cfg->aggregate = -1;
    cfg->partition_vertices = 0;
    cfg->global_vertices = 0;
    cfg->vertex_base = 0;
}

void hg_probe_options_init(hg_probe_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->pair_width = 8;
    o->pair_cap = uint64_t(1) << 24;
}

hg_status hg_derived_vertex_count(uint64_t n, double load_factor, uint64_t* out) {
    if (!out) return fail(HG_EINVAL, "out is NULL");
    if (!(load_factor > 0.0)) return fail(HG_EINVAL, "load_factor must be positive");
    const double v = std::floor(static_cast<double>(n) / load_factor);
    *out = v < 1.0 ? 1 : static_cast<uint64_t>(v);
    return HG_OK;
}

uint64_t hg_hash_to_vertex(uint64_t key, uint64_t seed, uint64_t nv) {
    if (nv == 0) return 0;
    uint64_t x = key ^ seed;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x % nv;
}

// hg_build / hg_build_records: keys + optional values (SoA), or n AoS
// records {key, value} (key_width / val_width each, 8-byte records for
// 4 + 4, else 16 with both fields widened to 8 bytes).
static hg_status build_common(const void* keys, int32_t key_width, const void* vals,
                              int32_t val_width, const void* records, uint64_t n,
                              const hg_build_config* cfg_in, void* stream, hg_table** out) {
    if (!out) return fail(HG_EINVAL, "out is NULL");
    *out = nullptr;
    hg_build_config cfg;
    if (cfg_in) {
        cfg = *cfg_in;
    } else {
        hg_build_config_init(&cfg);
    }
    // core.hpp:106-109 check_config
    if (!(cfg.load_factor > 0.0)) return fail(HG_EINVAL, "load_factor must be positive");
    if (cfg.bin_count < 1) return fail(HG_EINVAL, "bin_count must be at least 1");
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    if ((vals || records) && val_width != 4 && val_width != 8)
        return fail(HG_EINVAL, "val_width must be 4 or 8");
    if (cfg.variant != HG_BUILD_SIMPLE && cfg.variant != HG_BUILD_BINNED)
        return fail(HG_EINVAL, "variant must be 1 (simple) or 2 (binned)");
    if (cfg.hash_kind != HG_HASH_MIX64 && cfg.hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    if (n && !keys && !records) return fail(HG_EINVAL, "keys is NULL");
    uint64_t nv = cfg.vertex_count;
    if (cfg.global_vertices) {
        if (!nv) return fail(HG_EINVAL, "a shard build needs vertex_count (its local vertex range)");
        if (cfg.vertex_base + nv > cfg.global_vertices)
            return fail(HG_EINVAL, "shard vertex range exceeds global_vertices");
    }
    if (!nv) {
        hg_status st = hg_derived_vertex_count(n, cfg.load_factor, &nv);
        if (st != HG_OK) return st;
    }
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    auto* t = new hg_table;
    t->device = dev;
    t->load_factor = cfg.load_factor;
    hg::TableDesc& d = t->d;
    d.nv = nv;
    d.n = n;
    d.gnv = cfg.global_vertices;
    d.vbase = cfg.global_vertices ? cfg.vertex_base : 0;
    d.seed = cfg.hash_seed;
    d.hash_kind = cfg.hash_kind;
    d.key_bytes = key_width;
    d.val_bytes = (vals || records) ? val_width : (n <= (uint64_t(1) << 32) ? 4 : 8);
    d.off_bytes = (n < (uint64_t(1) << 32) && nv <= (uint64_t(1) << 32)) ? 4 : 8;
    // offs is padded so that offs + 1 (the counter / cursor view) is 16-byte aligned.
    const uint64_t pad = 16 / d.off_bytes - 1;
    cudaError_t e = cudaSuccess;
    if (hg::huge_allocation((nv + 1 + pad) * d.off_bytes + n * (d.key_bytes + d.val_bytes)))
        e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMallocAsync(&t->alloc_offs, (nv + 1 + pad) * d.off_bytes, s);
    if (e == cudaSuccess && n) e = cudaMallocAsync(&d.keys, n * d.key_bytes, s);
    if (e == cudaSuccess && n) e = cudaMallocAsync(&d.vals, n * d.val_bytes, s);
    if (e != cudaSuccess) {
        hg_table_destroy(t, stream);
        return cuda_fail(e, "hg_build: table allocation");
    }
    d.offs = static_cast<char*>(t->alloc_offs) + pad * d.off_bytes;

    DevIn kin, vin;
    const uint64_t rec_bytes = (key_width == 4 && val_width == 4) ? 8 : 16;
    e = records ? kin.stage(records, n * rec_bytes, s) : kin.stage(keys, n * key_width, s);
    if (e == cudaSuccess && vals && !records) e = vin.stage(vals, n * val_width, s);
    if (e == cudaSuccess) {
        hg::BuildArgs a;
        a.keys = records ? nullptr : kin.ptr;
        a.vals = vals && !records ? vin.ptr : nullptr;
        a.records = records ? kin.ptr : nullptr;
        a.n = n;
        a.variant = cfg.variant;
        a.aggregate = cfg.aggregate < 0 ? 1 : cfg.aggregate;
        a.stable = cfg.stable;
        a.partition_vertices = cfg.partition_vertices;
        e = hg::build_table(d, a, s);
    }
    kin.release(s);
    vin.release(s);
    if (e != cudaSuccess) {
        hg_table_destroy(t, stream);
        return cuda_fail(e, "hg_build");
    }
    *out = t;
    return HG_OK;
}

hg_status hg_build(const void* keys, int32_t key_width, const void* vals, int32_t val_width,
                   uint64_t n, const hg_build_config* cfg, void* stream, hg_table** out) {
    return build_common(keys, key_width, vals, val_width, nullptr, n, cfg, stream, out);
}

hg_status hg_build_records(const void* records, int32_t key_width, int32_t val_width, uint64_t n,
                           const hg_build_config* cfg, void* stream, hg_table** out) {
    if (n && !records) return fail(HG_EINVAL, "records is NULL");
    return build_common(nullptr, key_width, nullptr, val_width, records, n, cfg, stream, out);
}

hg_status hg_table_import(const uint64_t* offsets, const uint64_t* keys, const uint64_t* vals,
                          uint64_t num_vertices, uint64_t num_edges, uint64_t hash_seed,
                          double load_factor, int32_t hash_kind, void* stream, hg_table** out) {
    if (!out) return fail(HG_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_vertices < 1) return fail(HG_EINVAL, "table has no vertices");
    if (!offsets || (num_edges && (!keys || !vals))) return fail(HG_EINVAL, "NULL array");
    if (hash_kind != HG_HASH_MIX64 && hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* t = new hg_table;
    t->device = dev;
    t->load_factor = load_factor;
    hg::TableDesc& d = t->d;
    d.nv = num_vertices;
    d.n = num_edges;
    d.seed = hash_seed;
    d.hash_kind = hash_kind;
    d.key_bytes = d.val_bytes = d.off_bytes = 8;
    cudaError_t e = cudaMallocAsync(&t->alloc_offs, (num_vertices + 2) * 8, s);
    if (e == cudaSuccess && num_edges) e = cudaMallocAsync(&d.keys, num_edges * 8, s);
    if (e == cudaSuccess && num_edges) e = cudaMallocAsync(&d.vals, num_edges * 8, s);
    if (e == cudaSuccess) {
        d.offs = static_cast<char*>(t->alloc_offs) + 8;
        e = cudaMemcpyAsync(d.offs, offsets, (num_vertices + 1) * 8, cudaMemcpyDefault, s);
    }
    if (e == cudaSuccess && num_edges)
        e = cudaMemcpyAsync(d.keys, keys, num_edges * 8, cudaMemcpyDefault, s);
    if (e == cudaSuccess && num_edges)
        e = cudaMemcpyAsync(d.vals, vals, num_edges * 8, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        hg_table_destroy(t, stream);
        return cuda_fail(e, "hg_table_import");
    }
    *out = t;
    return HG_OK;
}

hg_status hg_table_get_info(const hg_table* t, hg_table_info* info) {
    if (!t || !info) return fail(HG_EINVAL, "NULL argument");
    info->num_vertices = t->d.nv;
    info->num_edges = t->d.n;
    info->hash_seed = t->d.seed;
    info->load_factor = t->load_factor;
    info->key_width = t->d.key_bytes;
    info->val_width = t->d.val_bytes;
    info->off_width = t->d.off_bytes;
    info->hash_kind = t->d.hash_kind;
    return HG_OK;
}

hg_status hg_table_device_arrays(const hg_table* t, const void** offs, const void** keys,
                                 const void** vals) {
    if (!t) return fail(HG_EINVAL, "NULL table");
    if (offs) *offs = t->d.offs;
    if (keys) *keys = t->d.keys;
    if (vals) *vals = t->d.vals;
    return HG_OK;
}

hg_status hg_table_export(const hg_table* t, uint64_t* offsets, uint64_t* keys, uint64_t* vals,
                          void* stream) {
    if (!t) return fail(HG_EINVAL, "NULL table");
    cudaSetDevice(t->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    HG_CUDA(widen_to(t->d.offs, t->d.off_bytes, t->d.nv + 1, offsets, s));
    HG_CUDA(widen_to(t->d.keys, t->d.key_bytes, t->d.n, keys, s));
    HG_CUDA(widen_to(t->d.vals, t->d.val_bytes, t->d.n, vals, s));
    HG_CUDA(cudaStreamSynchronize(s));
    return HG_OK;
}

hg_status hg_table_destroy(hg_table* t, void* stream) {
    if (!t) return HG_OK;
    cudaSetDevice(t->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (t->alloc_offs) cudaFreeAsync(t->alloc_offs, s);
    if (t->d.keys) cudaFreeAsync(t->d.keys, s);
    if (t->d.vals) cudaFreeAsync(t->d.vals, s);
    delete t;
    return HG_OK;
}

hg_status hg_probe(const hg_table* t, const void* probes, int32_t probe_width, uint64_t m,
                   const hg_probe_options* opts_in, hg_probe_result* result, void* stream) {
    if (!t) return fail(HG_EINVAL, "NULL table");
    hg_probe_options opts;
    if (opts_in) {
        opts = *opts_in;
    } else {
        hg_probe_options_init(&opts);
    }
    if (probe_width != 4 && probe_width != 8) return fail(HG_EINVAL, "probe_width must be 4 or 8");
    if (probe_width != t->d.key_bytes && !(probe_width == 4 && t->d.key_bytes == 8))
        return fail(HG_EUNSUPPORTED, "u64 probes into a u32-keyed table are not supported");
    if (m && !probes) return fail(HG_EINVAL, "probes is NULL");
    if (opts.materialize && opts.pair_width != 4 && opts.pair_width != 8)
        return fail(HG_EINVAL, "pair_width must be 4 or 8");
    if (opts.materialize && opts.pair_cap && !opts.pairs)
        return fail(HG_EINVAL, "materialize requires a pairs buffer");
    if (!opts.device_result && !result) return fail(HG_EINVAL, "result is NULL");
    if ((opts.flags & HG_PROBE_HASHER) && opts.hash_kind != HG_HASH_MIX64 &&
        opts.hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    if (cudaSetDevice(t->device) != cudaSuccess) return fail(HG_ECUDA, "cudaSetDevice failed");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the table as the probe sees it: join.hpp:117-118 hashes each probe with
    // the caller's hasher (default: the table's own, join.hpp:133-136)
    hg::TableDesc td = t->d;
    if (opts.flags & HG_PROBE_HASHER) {
        td.hash_kind = opts.hash_kind;
        td.seed = opts.hash_seed;
    }

    // Pinned host probes without pairs: chunked pipeline, each chunk's H2D
    // copy (on a side stream) overlaps the previous chunk's probe kernels --
    // and, with HG_PROBE_HOST_READY, whatever is still running on `stream`
    // (e.g. the build of this table).
    constexpr uint64_t kPipeChunk = uint64_t(1) << 26;
    const bool pipelined = m >= 2 * kPipeChunk && !opts.materialize &&
                           probe_width == t->d.key_bytes && is_pinned_host(probes);
    DevIn pin;
    cudaError_t e = pipelined ? cudaSuccess : pin.stage(probes, m * probe_width, s);
    if (e != cudaSuccess) return cuda_fail(e, "hg_probe: staging probes");
    const void* dprobes = pin.ptr;
    void* widened = nullptr;
    if (probe_width == 4 && t->d.key_bytes == 8 && m) {
        if ((e = cudaMallocAsync(&widened, m * 8, s)) != cudaSuccess) {
            pin.release(s);
            return cuda_fail(e, "hg_probe: widen buffer");
        }
        const unsigned grid = unsigned(std::min<uint64_t>((m + 255) / 256, 148 * 16));
        k_narrow_u32_to_u64<<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(dprobes),
                                                 static_cast<uint64_t*>(widened), m);
        dprobes = widened;
    }

    const bool want_pairs = opts.materialize && opts.pair_cap > 0;
    const bool counts_dev = opts.counts && is_device_ptr(opts.counts);
    const bool pairs_dev = want_pairs && is_device_ptr(opts.pairs);
    // Host pair destination: the device staging is sized from the exact match
    // count (one count-only pass first) instead of pair_cap, which defaults to
    // 2^24 pairs (join.hpp:27) however few matches there are.
    uint64_t cap_eff = opts.pair_cap;
    if (want_pairs && !pairs_dev && m) {
        uint64_t* dt = nullptr;
        uint64_t ht[2] = {0, 0};
        e = cudaMallocAsync(reinterpret_cast<void**>(&dt), 16, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(dt, 0, 16, s);
        if (e == cudaSuccess) {
            hg::ProbeArgs c;
            c.probes = dprobes;
            c.m = m;
            c.totals = dt;
            c.method = opts.method;
            e = hg::probe_table(td, c, s);
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(ht, dt, 16, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (dt) cudaFreeAsync(dt, s);
        if (e != cudaSuccess) {
            pin.release(s);
            if (widened) cudaFreeAsync(widened, s);
            return cuda_fail(e, "hg_probe: match count");
        }
        cap_eff = std::max<uint64_t>(1, std::min(opts.pair_cap, ht[0]));
    }
    // scratch: totals[3] | counts[m] (if needed) | pair_offsets[m+1] | pairs staging
    uint64_t* totals = opts.device_result;
    void* scratch = nullptr;
    size_t need = 0;
    const size_t tot_off = 0, tot_bytes = totals ? 0 : 256;
    const size_t cnt_off = tot_bytes;
    const bool need_counts = want_pairs || opts.materialize || opts.counts;
    const size_t cnt_bytes = (need_counts && !counts_dev) ? ((m * 4 + 255) & ~size_t(255)) : 0;
    const size_t po_off = cnt_off + cnt_bytes;
    const size_t po_bytes = opts.materialize ? (((m + 1) * 8 + 255) & ~size_t(255)) : 0;
    const size_t pr_off = po_off + po_bytes;
    const size_t pr_bytes = (want_pairs && !pairs_dev) ? cap_eff * 2 * opts.pair_width : 0;
    need = pr_off + pr_bytes;
    if (need && (e = cudaMallocAsync(&scratch, need, s)) != cudaSuccess) {
        pin.release(s);
        if (widened) cudaFreeAsync(widened, s);
        return cuda_fail(e, "hg_probe: scratch");
    }
    char* sc = static_cast<char*>(scratch);
    if (!totals) totals = reinterpret_cast<uint64_t*>(sc + tot_off);
    uint32_t* counts = need_counts ? (counts_dev ? opts.counts : reinterpret_cast<uint32_t*>(sc + cnt_off))
                                   : nullptr;
    uint64_t* pair_off = opts.materialize ? reinterpret_cast<uint64_t*>(sc + po_off) : nullptr;
    void* pairs = want_pairs ? (pairs_dev ? opts.pairs : static_cast<void*>(sc + pr_off)) : nullptr;

    e = cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    hg::ProbeArgs a;
    a.probes = dprobes;
    a.m = m;
    a.counts = counts;
    a.counts_requested = opts.counts != nullptr;
    a.totals = totals;
    a.pairs = pairs;
    a.pair_bytes = opts.pair_width;
    a.cap = want_pairs ? cap_eff : 0;
    a.pair_offsets = pair_off;
    a.method = opts.method;
    if (e == cudaSuccess && !pipelined) e = hg::probe_table(td, a, s);
    if (e == cudaSuccess && pipelined) {
        void* ring = nullptr;
        cudaStream_t cs = nullptr;
        cudaEvent_t ready = nullptr, copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
        const size_t cb = size_t(kPipeChunk) * probe_width;
        // the ring is allocated on the copy stream, so the first copies do not
        // wait for earlier work on `stream` (e.g. the build of this table)
        e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        if (e == cudaSuccess && !(opts.flags & HG_PROBE_HOST_READY)) {
            // stream order: the copies wait for everything enqueued on `stream`
            // so far (which may still be writing the host buffer)
            e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(ready, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ready, 0);
        }
        if (e == cudaSuccess) e = cudaMallocAsync(&ring, 2 * cb, cs);
        for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
            e = cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
        }
        const char* host = static_cast<const char*>(probes);
        for (uint64_t c = 0; e == cudaSuccess && c * kPipeChunk < m; ++c) {
            const int b = int(c & 1);
            const uint64_t off = c * kPipeChunk, mc = std::min(kPipeChunk, m - off);
            char* buf = static_cast<char*>(ring) + b * cb;
            if (c >= 2) e = cudaStreamWaitEvent(cs, done[b], 0);  // buffer free again
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(buf, host + off * probe_width, mc * probe_width,
                                    cudaMemcpyHostToDevice, cs);
            if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(s, copied[b], 0);
            if (e != cudaSuccess) break;
            hg::ProbeArgs ac = a;
            ac.probes = buf;
            ac.m = mc;
            ac.counts = counts ? counts + off : nullptr;
            e = hg::probe_table(td, ac, s);
            if (e == cudaSuccess) e = cudaEventRecord(done[b], s);
        }
        if (ring) cudaFreeAsync(ring, s);
        // destruction is deferred by the runtime until the recorded work completes
        for (int b = 0; b < 2; ++b) {
            if (copied[b]) cudaEventDestroy(copied[b]);
            if (done[b]) cudaEventDestroy(done[b]);
        }
        if (ready) cudaEventDestroy(ready);
        if (cs) cudaStreamDestroy(cs);
    }

    hg_status st = HG_OK;
    if (e != cudaSuccess) {
        st = cuda_fail(e, "hg_probe");
    } else if (!opts.device_result) {
        uint64_t host_tot[2] = {0, 0};
        e = cudaMemcpyAsync(host_tot, totals, sizeof host_tot, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && opts.counts && !counts_dev && m)
            e = cudaMemcpyAsync(opts.counts, counts, m * 4, cudaMemcpyDeviceToHost, s);
        const uint64_t written = opts.materialize ? std::min(host_tot[0], opts.pair_cap) : 0;
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess && want_pairs && !pairs_dev && written)
            e = cudaMemcpyAsync(opts.pairs, pairs, written * 2 * opts.pair_width,
                                cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "hg_probe: result readback");
        } else if (result) {
            result->match_count = host_tot[0];
            result->key_comparisons = host_tot[1];
            result->pairs_written = written;
            result->truncated = opts.materialize && host_tot[0] > opts.pair_cap;
        }
    } else if (result) {
        std::memset(result, 0, sizeof *result);
    }
    if (scratch) cudaFreeAsync(scratch, s);
    if (widened) cudaFreeAsync(widened, s);
    pin.release(s);
    return st;
}

hg_status hg_probe_new_prepared(const hg_table* ta, const hg_table* tb,
                                const hg_probe_options* opts_in, hg_probe_result* result,
                                void* stream) {
    if (!ta || !tb) return fail(HG_EINVAL, "NULL table");
    hg_probe_options opts;
    if (opts_in) {
        opts = *opts_in;
    } else {
        hg_probe_options_init(&opts);
    }
    // join.hpp:145-147
    if (ta->d.nv != tb->d.nv || ta->d.gnv != tb->d.gnv || ta->d.vbase != tb->d.vbase)
        return fail(HG_EINVAL, "probe_new_prepared: tables use different vertex ranges");
    if (ta->d.key_bytes != tb->d.key_bytes)
        return fail(HG_EUNSUPPORTED, "probe_new_prepared: tables have different key widths");
    if (ta->device != tb->device) return fail(HG_EINVAL, "tables live on different devices");
    if (opts.counts) return fail(HG_EINVAL, "probe_new_prepared has no per-probe counts");
    if (opts.materialize && opts.pair_width != 4 && opts.pair_width != 8)
        return fail(HG_EINVAL, "pair_width must be 4 or 8");
    if (opts.materialize && opts.pair_cap && !opts.pairs)
        return fail(HG_EINVAL, "materialize requires a pairs buffer");
    if (!opts.device_result && !result) return fail(HG_EINVAL, "result is NULL");
    if (cudaSetDevice(ta->device) != cudaSuccess) return fail(HG_ECUDA, "cudaSetDevice failed");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool want_pairs = opts.materialize && opts.pair_cap > 0;
    const bool pairs_dev = want_pairs && is_device_ptr(opts.pairs);
    const size_t tot_bytes = opts.device_result ? 0 : 256;
    cudaError_t e = cudaSuccess;
    // host pair destination: device staging sized from the exact match count
    // (one count-only intersect first), not from pair_cap
    uint64_t cap_eff = opts.pair_cap;
    if (want_pairs && !pairs_dev) {
        uint64_t* dt = nullptr;
        uint64_t ht[2] = {0, 0};
        e = cudaMallocAsync(reinterpret_cast<void**>(&dt), 16, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(dt, 0, 16, s);
        hg::IntersectArgs ca;
        ca.totals = dt;
        if (e == cudaSuccess) e = hg::intersect_tables(ta->d, tb->d, ca, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(ht, dt, 16, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (dt) cudaFreeAsync(dt, s);
        if (e != cudaSuccess) return cuda_fail(e, "hg_probe_new_prepared: match count");
        cap_eff = std::max<uint64_t>(1, std::min(opts.pair_cap, ht[0]));
    }
    const size_t pr_bytes = (want_pairs && !pairs_dev) ? cap_eff * 2 * opts.pair_width : 0;
    void* scratch = nullptr;
    if (tot_bytes + pr_bytes && (e = cudaMallocAsync(&scratch, tot_bytes + pr_bytes, s)) != cudaSuccess)
        return cuda_fail(e, "hg_probe_new_prepared: scratch");
    uint64_t* totals = opts.device_result ? opts.device_result : static_cast<uint64_t*>(scratch);
    void* pairs = want_pairs ? (pairs_dev ? opts.pairs : static_cast<char*>(scratch) + tot_bytes)
                             : nullptr;
    e = cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    hg::IntersectArgs ia;
    ia.totals = totals;
    ia.pairs = pairs;
    ia.pair_bytes = opts.pair_width;
    ia.cap = want_pairs ? cap_eff : 0;
    if (e == cudaSuccess) e = hg::intersect_tables(ta->d, tb->d, ia, s);
    hg_status st = HG_OK;
    if (e != cudaSuccess) {
        st = cuda_fail(e, "hg_probe_new_prepared");
    } else if (!opts.device_result) {
        uint64_t host_tot[2] = {0, 0};
        e = cudaMemcpyAsync(host_tot, totals, sizeof host_tot, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        const uint64_t written = opts.materialize ? std::min(host_tot[0], opts.pair_cap) : 0;
        if (e == cudaSuccess && want_pairs && !pairs_dev && written)
            e = cudaMemcpyAsync(opts.pairs, pairs, written * 2 * opts.pair_width,
                                cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "hg_probe_new_prepared: result readback");
        } else if (result) {
            result->match_count = host_tot[0];
            result->key_comparisons = host_tot[1];
            result->pairs_written = written;
            result->truncated = opts.materialize && host_tot[0] > opts.pair_cap;
        }
    } else if (result) {
        std::memset(result, 0, sizeof *result);
    }
    if (scratch) cudaFreeAsync(scratch, s);
    return st;
}

hg_status hg_probe_new(const void* keys_a, uint64_t na, const void* keys_b, uint64_t nb,
                       int32_t key_width, const hg_build_config* cfg_in,
                       const hg_probe_options* opts, hg_probe_result* result, void* stream) {
    hg_build_config cfg;
    if (cfg_in) {
        cfg = *cfg_in;
    } else {
        hg_build_config_init(&cfg);
    }
    if (cfg.global_vertices) return fail(HG_EINVAL, "probe_new builds unsharded tables");
    if (!cfg.vertex_count) {
        // join.hpp:171-172: V from the larger input
        hg_status st = hg_derived_vertex_count(na > nb ? na : nb, cfg.load_factor, &cfg.vertex_count);
        if (st != HG_OK) return st;
    }
    cfg.variant = HG_BUILD_BINNED;  // join.hpp:173-174
    hg_table* ta = nullptr;
    hg_table* tb = nullptr;
    hg_status st = hg_build(keys_a, key_width, nullptr, 8, na, &cfg, stream, &ta);
    if (st == HG_OK) st = hg_build(keys_b, key_width, nullptr, 8, nb, &cfg, stream, &tb);
    if (st == HG_OK) st = hg_probe_new_prepared(ta, tb, opts, result, stream);
    hg_table_destroy(ta, stream);
    hg_table_destroy(tb, stream);
    return st;
}

static hg_status count_instances_impl(const hg_table* t, uint64_t key, const hg_probe_options* o,
                                      uint64_t* out, void* stream);

hg_status hg_count_instances(const hg_table* t, uint64_t key, uint64_t* out, void* stream) {
    return count_instances_impl(t, key, nullptr, out, stream);
}

hg_status hg_count_instances_hasher(const hg_table* t, uint64_t key, int32_t hash_kind,
                                    uint64_t hash_seed, uint64_t* out, void* stream) {
    hg_probe_options o;
    hg_probe_options_init(&o);
    o.flags = HG_PROBE_HASHER;
    o.hash_kind = hash_kind;
    o.hash_seed = hash_seed;
    return count_instances_impl(t, key, &o, out, stream);
}

static hg_status count_instances_impl(const hg_table* t, uint64_t key, const hg_probe_options* o,
                                      uint64_t* out, void* stream) {
    if (!out) return fail(HG_EINVAL, "out is NULL");
    if (t && t->d.key_bytes == 4 && key > 0xFFFFFFFFull) {
        // A u32-keyed table cannot hold a wider key: zero matches (the
        // comparison count is irrelevant to count_instances).
        *out = 0;
        return HG_OK;
    }
    hg_probe_result r;
    const uint32_t k32 = uint32_t(key);
    const void* kp = t && t->d.key_bytes == 4 ? static_cast<const void*>(&k32)
                                               : static_cast<const void*>(&key);
    hg_status st = hg_probe(t, kp, t ? t->d.key_bytes : 8, 1, o, &r, stream);
    if (st == HG_OK) *out = r.match_count;
    return st;
}

hg_status hg_validate(const hg_table* t, const void* input_keys, uint64_t expected_entries,
                      int32_t* violation, void* stream) {
    if (!t) return fail(HG_EINVAL, "NULL argument");
    return hg_validate_hasher(t, input_keys, expected_entries, t->d.hash_kind, t->d.seed, violation,
                              stream);
}

hg_status hg_validate_hasher(const hg_table* t, const void* input_keys, uint64_t expected_entries,
                             int32_t hash_kind, uint64_t hash_seed, int32_t* violation,
                             void* stream) {
    if (!t || !violation) return fail(HG_EINVAL, "NULL argument");
    if (hash_kind != HG_HASH_MIX64 && hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    if (cudaSetDevice(t->device) != cudaSuccess) return fail(HG_ECUDA, "cudaSetDevice failed");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    *violation = 0;
    if (t->d.nv < 1) {
        *violation = 1;
        return HG_OK;
    }
    DevIn in;
    cudaError_t e = in.stage(input_keys, t->d.n * t->d.key_bytes, s);
    uint32_t* d_code = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&d_code), 4, s);
    hg::TableDesc td = t->d;  // core.hpp:271: the check uses the caller's hasher
    td.hash_kind = hash_kind;
    td.seed = hash_seed;
    if (e == cudaSuccess) e = hg::validate_table(td, input_keys ? in.ptr : nullptr, d_code, s);
    uint32_t code = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&code, d_code, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (d_code) cudaFreeAsync(d_code, s);
    in.release(s);
    if (e != cudaSuccess) return cuda_fail(e, "hg_validate");
    if (code == 0xFFFFFFFFu) code = 0;
    if (code == 0 && t->d.n != expected_entries) code = 6;  // core.hpp:268
    // Codes are ordered like validate_csr's checks except 6 (edge count vs
    // input size), which the reference tests right after 5.
    if (code > 6 && t->d.n != expected_entries) code = 6;
    *violation = int32_t(code);
    return HG_OK;
}

hg_status hg_shard_range(uint64_t global_vertices, uint32_t shards, uint32_t shard,
                         uint64_t* vertex_base, uint64_t* vertex_count) {
    if (!vertex_base || !vertex_count) return fail(HG_EINVAL, "NULL argument");
    if (shards < 1 || shard >= shards || global_vertices < 1)
        return fail(HG_EINVAL, "need 0 <= shard < shards and global_vertices >= 1");
    const uint64_t span = (global_vertices + shards - 1) / shards;
    const uint64_t b = std::min<uint64_t>(global_vertices, uint64_t(shard) * span);
    const uint64_t e = std::min<uint64_t>(global_vertices, b + span);
    *vertex_base = b;
    *vertex_count = e - b;
    return HG_OK;
}

hg_status hg_route(const void* keys, int32_t key_width, const void* vals, int32_t val_width,
                   uint64_t n, uint64_t val_base, uint64_t hash_seed, int32_t hash_kind,
                   uint64_t global_vertices, uint32_t shards, void* out_keys, void* out_vals,
                   uint64_t* shard_counts, void* stream) {
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    if (val_width != 4 && val_width != 8) return fail(HG_EINVAL, "val_width must be 4 or 8");
    if (shards < 1 || shards > 256) return fail(HG_EINVAL, "shards must be in [1, 256]");
    if (global_vertices < 1) return fail(HG_EINVAL, "global_vertices must be >= 1");
    if (hash_kind != HG_HASH_MIX64 && hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    if (!shard_counts) return fail(HG_EINVAL, "shard_counts is NULL");
    if (n && (!is_device_ptr(keys) || !is_device_ptr(out_keys) ||
              (out_vals && !is_device_ptr(out_vals)) || (vals && !is_device_ptr(vals))))
        return fail(HG_EINVAL, "hg_route takes device buffers");
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool counts_dev = is_device_ptr(shard_counts);
    uint64_t* dc = shard_counts;
    if (!counts_dev) HG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dc), shards * 8, s));
    cudaError_t e = hg::route_keys(keys, key_width, vals, val_width, n, val_base, hash_seed,
                                   hash_kind, global_vertices, 0, global_vertices, 0, shards,
                                   out_keys, out_vals, dc, s);
    if (e == cudaSuccess && !counts_dev) {
        e = cudaMemcpyAsync(shard_counts, dc, shards * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (!counts_dev) cudaFreeAsync(dc, s);
    if (e != cudaSuccess) return cuda_fail(e, "hg_route");
    return HG_OK;
}

hg_status hg_route_records(const void* keys, int32_t key_width, const void* vals,
                           int32_t val_width, uint64_t n, uint64_t val_base, uint64_t hash_seed,
                           int32_t hash_kind, uint64_t global_vertices, uint32_t shards,
                           void* out_records, uint64_t* shard_counts, void* stream) {
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    if (val_width != 4 && val_width != 8) return fail(HG_EINVAL, "val_width must be 4 or 8");
    if (shards < 1 || shards > 256) return fail(HG_EINVAL, "shards must be in [1, 256]");
    if (global_vertices < 1) return fail(HG_EINVAL, "global_vertices must be >= 1");
    if (hash_kind != HG_HASH_MIX64 && hash_kind != HG_HASH_IDENTITY)
        return fail(HG_EINVAL, "unknown hash_kind");
    if (!shard_counts || !is_device_ptr(shard_counts))
        return fail(HG_EINVAL, "shard_counts must be a device buffer");
    if (n && (!is_device_ptr(keys) || !is_device_ptr(out_records) || (vals && !is_device_ptr(vals))))
        return fail(HG_EINVAL, "hg_route_records takes device buffers");
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    cudaError_t e = hg::route_keys(keys, key_width, vals, val_width, n, val_base, hash_seed,
                                   hash_kind, global_vertices, 0, global_vertices, 0, shards,
                                   nullptr, nullptr, shard_counts, static_cast<cudaStream_t>(stream),
                                   out_records);
    if (e != cudaSuccess) return cuda_fail(e, "hg_route_records");
    return HG_OK;
}

hg_status hg_route_pairs(const void* left, const void* right, int32_t pair_width, uint64_t n,
                         uint64_t span, uint32_t shards, void* out_records, uint64_t* shard_counts,
                         void* stream) {
    if (pair_width != 4 && pair_width != 8) return fail(HG_EINVAL, "pair_width must be 4 or 8");
    if (shards < 1 || shards > 256) return fail(HG_EINVAL, "shards must be in [1, 256]");
    if (span < 1) return fail(HG_EINVAL, "span must be >= 1");
    if (!shard_counts || !is_device_ptr(shard_counts))
        return fail(HG_EINVAL, "shard_counts must be a device buffer");
    if (n && (!is_device_ptr(left) || !is_device_ptr(right) || !is_device_ptr(out_records)))
        return fail(HG_EINVAL, "hg_route_pairs takes device buffers");
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    cudaError_t e = hg::route_pairs(left, right, pair_width, n, span, shards, out_records,
                                    shard_counts, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "hg_route_pairs");
    return HG_OK;
}

hg_status hg_generate(void* out, int32_t key_width, uint64_t n, int32_t kind, uint64_t seed,
                      uint64_t start, double hit, const void* ref, uint64_t n_ref, void* stream) {
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    if (kind < 0 || kind > 3) return fail(HG_EINVAL, "unknown generator kind");
    if (kind == 3 && (!n_ref || !is_device_ptr(ref)))
        return fail(HG_EINVAL, "the Zipf generator needs a device CDF (ref, n_ref)");
    if (n && !is_device_ptr(out)) return fail(HG_EINVAL, "hg_generate writes device memory only");
    int dev = 0;
    if (hg_status st = need_device(&dev); st != HG_OK) return st;
    HG_CUDA(hg::generate_keys(out, key_width, n, kind, seed, start, hit, ref, n_ref,
                              static_cast<cudaStream_t>(stream)));
    return HG_OK;
}

}  // extern "C"

// ------------------------------------------------------------ key files
// keygen.hpp:97-132 (HGKEYS01). Host file I/O; device destinations/sources go
// through a pinned staging buffer in 2^24-key chunks.
namespace {
constexpr char kKeyMagic[8] = {'H', 'G', 'K', 'E', 'Y', 'S', '0', '1'};
constexpr uint64_t kKeyChunk = uint64_t(1) << 24;

hg_status key_header(FILE* f, const char* path, uint64_t* count) {
    unsigned char h[16];
    if (fseek(f, 0, SEEK_END) != 0) return fail(HG_EIO, "read failure on key file: %s", path);
    const long sz = ftell(f);
    if (sz < 0 || fseek(f, 0, SEEK_SET) != 0) return fail(HG_EIO, "read failure on key file: %s", path);
    if (sz < 16 || fread(h, 1, 16, f) != 16)
        return fail(HG_EIO, "key file too short for its header: %s", path);
    if (std::memcmp(h, kKeyMagic, 8) != 0) return fail(HG_EIO, "key file magic mismatch: %s", path);
    uint64_t c = 0;
    for (int b = 0; b < 8; ++b) c |= uint64_t(h[8 + b]) << (8 * b);
    const uint64_t payload = uint64_t(sz) - 16;
    if (payload % 8 != 0 || payload / 8 != c)
        return fail(HG_EIO, "key file length does not match its key count: %s", path);
    *count = c;
    return HG_OK;
}

struct PinnedBuf {
    void* p = nullptr;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};
}  // namespace

extern "C" {

hg_status hg_keys_file_count(const char* path, uint64_t* count) {
    if (!path || !count) return fail(HG_EINVAL, "NULL argument");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(HG_EIO, "cannot open key file: %s", path);
    const hg_status st = key_header(f, path, count);
    fclose(f);
    return st;
}

hg_status hg_keys_read(const char* path, void* out, int32_t key_width, uint64_t cap, uint64_t* count,
                       void* stream) {
    if (!path || !count) return fail(HG_EINVAL, "NULL argument");
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(HG_EIO, "cannot open key file: %s", path);
    uint64_t n = 0;
    hg_status st = key_header(f, path, &n);
    if (st == HG_OK && n > cap) st = fail(HG_ERANGE, "key file holds %llu keys, capacity %llu",
                                          (unsigned long long)n, (unsigned long long)cap);
    if (st == HG_OK && n && !out) st = fail(HG_EINVAL, "out is NULL");
    const bool dev = st == HG_OK && n && is_device_ptr(out);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PinnedBuf stage[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    if (dev) {
        for (int b = 0; b < 2 && st == HG_OK; ++b) {
            if (cudaMallocHost(&stage[b].p, kKeyChunk * 8) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess)
                st = fail(HG_ENOMEM, "hg_keys_read: pinned staging");
        }
    }
    std::vector<uint64_t> tmp;
    for (uint64_t done = 0, c = 0; st == HG_OK && done < n; done += kKeyChunk, ++c) {
        const uint64_t k = std::min(kKeyChunk, n - done);
        const int b = int(c & 1);
        uint64_t* buf;
        if (dev) {
            if (c >= 2 && cudaEventSynchronize(ev[b]) != cudaSuccess) {  // staging buffer free
                st = fail(HG_ECUDA, "hg_keys_read: event");
                break;
            }
            buf = static_cast<uint64_t*>(stage[b].p);
        } else if (key_width == 8) {
            buf = static_cast<uint64_t*>(out) + done;
        } else {
            tmp.resize(k);
            buf = tmp.data();
        }
        if (fread(buf, 8, k, f) != k) {
            st = fail(HG_EIO, "read failure on key file: %s", path);
            break;
        }
        // the format is little-endian; so is every CUDA host
        if (key_width == 4) {
            uint32_t* o = dev ? reinterpret_cast<uint32_t*>(buf) : static_cast<uint32_t*>(out) + done;
            for (uint64_t i = 0; i < k; ++i) {
                if (buf[i] > 0xFFFFFFFFull) {
                    st = fail(HG_ERANGE, "key %llu does not fit 32 bits", (unsigned long long)buf[i]);
                    break;
                }
                o[i] = uint32_t(buf[i]);  // in place: o[i] never overtakes buf[i]
            }
            if (st != HG_OK) break;
        }
        if (dev) {
            char* dst = static_cast<char*>(out) + done * key_width;
            if (cudaMemcpyAsync(dst, buf, k * key_width, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                cudaEventRecord(ev[b], s) != cudaSuccess) {
                st = fail(HG_ECUDA, "hg_keys_read: copy");
                break;
            }
        }
    }
    fclose(f);
    if (dev) {
        if (cudaStreamSynchronize(s) != cudaSuccess && st == HG_OK) st = fail(HG_ECUDA, "hg_keys_read: sync");
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    if (st == HG_OK) *count = n;
    return st;
}

hg_status hg_keys_write(const char* path, const void* keys, int32_t key_width, uint64_t n,
                        void* stream) {
    if (!path) return fail(HG_EINVAL, "NULL path");
    if (key_width != 4 && key_width != 8) return fail(HG_EINVAL, "key_width must be 4 or 8");
    if (n && !keys) return fail(HG_EINVAL, "keys is NULL");
    FILE* f = fopen(path, "wb");
    if (!f) return fail(HG_EIO, "cannot open key file for writing: %s", path);
    unsigned char h[16];
    std::memcpy(h, kKeyMagic, 8);
    for (int b = 0; b < 8; ++b) h[8 + b] = static_cast<unsigned char>((n >> (8 * b)) & 0xff);
    hg_status st = fwrite(h, 1, 16, f) == 16 ? HG_OK : fail(HG_EIO, "short write to key file: %s", path);
    const bool dev = n && is_device_ptr(keys);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PinnedBuf stage;
    if (st == HG_OK && dev && cudaMallocHost(&stage.p, kKeyChunk * 8) != cudaSuccess)
        st = fail(HG_ENOMEM, "hg_keys_write: pinned staging");
    std::vector<uint64_t> wide;
    for (uint64_t done = 0; st == HG_OK && done < n; done += kKeyChunk) {
        const uint64_t k = std::min(kKeyChunk, n - done);
        const char* src = static_cast<const char*>(keys) + done * key_width;
        const void* host = src;
        if (dev) {
            if (cudaMemcpyAsync(stage.p, src, k * key_width, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess) {
                st = fail(HG_ECUDA, "hg_keys_write: copy");
                break;
            }
            host = stage.p;
        }
        const uint64_t* out = static_cast<const uint64_t*>(host);
        if (key_width == 4) {
            wide.resize(k);
            const uint32_t* in = static_cast<const uint32_t*>(host);
            for (uint64_t i = 0; i < k; ++i) wide[i] = in[i];
            out = wide.data();
        }
        if (fwrite(out, 8, k, f) != k) st = fail(HG_EIO, "short write to key file: %s", path);
    }
    if (fclose(f) != 0 && st == HG_OK) st = fail(HG_EIO, "short write to key file: %s", path);
    return st;
}

}  // extern "C"
