// hg_probe.cu -- probe_table dispatch over the table's (key, value, offset)
// widths. The kernels and launchers live in hg_probe_impl.cuh; each width
// combination is instantiated in its own translation unit
// (hg_probe_k*_v*_o*.cu) so they compile in parallel.
#include "hg_internal.h"

namespace hg {

template <typename K, typename VT, typename OffT>
cudaError_t probe_pow(const TableDesc& t, const ProbeArgs& a, cudaStream_t s);

template <typename K, typename VT>
static cudaError_t probe_off(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.off_bytes == 4 ? probe_pow<K, VT, uint32_t>(t, a, s) : probe_pow<K, VT, uint64_t>(t, a, s);
}
template <typename K>
static cudaError_t probe_val(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.val_bytes == 4 ? probe_off<K, uint32_t>(t, a, s) : probe_off<K, uint64_t>(t, a, s);
}

cudaError_t probe_table(const TableDesc& t, const ProbeArgs& a, cudaStream_t s) {
    return t.key_bytes == 4 ? probe_val<uint32_t>(t, a, s) : probe_val<uint64_t>(t, a, s);
}

}  // namespace hg
