"""B200-native HashGraph engine (Green, arXiv 1907.02900).

Drop-in for the reference's hot path (proj/include/hashgraph: build_v1,
build_v2, probe_standard): hand-written sm_100a CUDA kernels behind the C-ABI
in include/hg_b200.h, with this package as the Python mirror of the reference
API and the C++ mirror in include/hashgraph/.
"""
from .hashgraph import (ENTRY_DTYPE, MATCH_PAIR_DTYPE, BuildConfig, BuildStats, ExecMode,
                        HashGraph, IdentityHasher, InvalidArgument, JoinResult, KeyFileError,
                        OutOfRange,
                        Overflow, ProbeOptions, VertexHasher, build_v1, build_v2, count_instances,
                        derived_vertex_count, generate, hash_to_vertex, intersect_adjacency,
                        probe_device, probe_new, probe_new_device, probe_new_prepared, probe_standard,
                        read_keys, validate_csr, write_keys, zipf_cdf)

__all__ = [
    "ENTRY_DTYPE", "MATCH_PAIR_DTYPE", "BuildConfig", "BuildStats", "ExecMode", "HashGraph",
    "IdentityHasher", "InvalidArgument", "JoinResult", "KeyFileError", "OutOfRange", "Overflow", "ProbeOptions",
    "VertexHasher", "build_v1", "build_v2", "count_instances", "derived_vertex_count", "generate",
    "hash_to_vertex", "intersect_adjacency", "probe_device", "probe_new",
    "probe_new_device", "probe_new_prepared", "probe_standard", "read_keys", "validate_csr", "write_keys",
    "zipf_cdf",
]
