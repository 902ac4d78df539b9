// Instantiates probe_pow for 4-byte keys, 4-byte values, 8-byte offsets.
#include "hg_probe_impl.cuh"

namespace hg {
template cudaError_t probe_pow<uint32_t, uint32_t, uint64_t>(const TableDesc&, const ProbeArgs&, cudaStream_t);
}  // namespace hg
