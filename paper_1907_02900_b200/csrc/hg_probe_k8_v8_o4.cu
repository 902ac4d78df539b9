// Instantiates probe_pow for 8-byte keys, 8-byte values, 4-byte offsets.
#include "hg_probe_impl.cuh"

namespace hg {
template cudaError_t probe_pow<uint64_t, uint64_t, uint32_t>(const TableDesc&, const ProbeArgs&, cudaStream_t);
}  // namespace hg
