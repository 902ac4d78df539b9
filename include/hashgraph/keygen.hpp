// hashgraph/keygen.hpp -- drop-in for the key-file half of the reference
// header of the same name (/root/reference/proj/include/hashgraph/keygen.hpp:
// 97-132, the HGKEYS01 wire format shared with the CPU reference), backed by
// hg_keys_write / hg_keys_read (include/hg_b200.h). The synthetic generators
// of that header (KeySpec / generate, :21-73) are input harness, not the hot
// path: on the device they are hg_generate's counter-based generators.
#pragma once
#include <hashgraph/hashgraph.hpp>

#include <filesystem>
#include <span>
#include <vector>

namespace hashgraph {

// keygen.hpp:100-111. Throws KeyFileError on any I/O problem.
inline void write_keys(const std::filesystem::path& path, std::span<const std::uint64_t> keys) {
    detail::check(hg_keys_write(path.c_str(), keys.data(), 8, keys.size(), nullptr));
}

// keygen.hpp:113-130. Throws KeyFileError on any I/O or format problem.
inline std::vector<std::uint64_t> read_keys(const std::filesystem::path& path) {
    std::uint64_t n = 0;
    detail::check(hg_keys_file_count(path.c_str(), &n));
    std::vector<std::uint64_t> keys(n);
    std::uint64_t got = 0;
    detail::check(hg_keys_read(path.c_str(), keys.data(), 8, keys.size(), &got, nullptr));
    keys.resize(got);
    return keys;
}

}  // namespace hashgraph
