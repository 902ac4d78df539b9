// Forced-include prelude (g++ -include) for the reference's unit tests built
// UNMODIFIED against the drop-in headers (Makefile: tests/cpp/ref_tests).
// The reference tests hash their hand-traced fixtures with
// support::IdentityHasher (proj/tests/support.hpp:42-46, vertex = key mod V);
// a host functor cannot run in the kernels, so the drop-in maps hasher types
// to device hash kinds through hashgraph::device_hasher<H> -- this is that
// mapping for the tests' hasher, the one line a reference user adds per
// custom hasher.
#pragma once
#include <hashgraph/core.hpp>

#include "support.hpp"  // /root/reference/proj/tests (read in place, not copied)

template <>
struct hashgraph::device_hasher<support::IdentityHasher> {
    static constexpr bool supported = true;
    static constexpr int kind = HG_HASH_IDENTITY;
    static std::uint64_t seed(const support::IdentityHasher&) { return 0; }
};
