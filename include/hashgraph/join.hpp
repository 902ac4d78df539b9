// hashgraph/join.hpp -- drop-in for the reference header of the same name
// (/root/reference/proj/include/hashgraph/join.hpp); everything lives in
// <hashgraph/hashgraph.hpp>, backed by the B200 engine (include/hg_b200.h).
#pragma once
#include <hashgraph/hashgraph.hpp>
