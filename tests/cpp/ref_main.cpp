// Runner for the reference's unit tests compiled against the drop-in headers
// through the Catch2 shim (tests/cpp/catch2shim/).
#include <catch2/catch_amalgamated.hpp>

int main() { return catch_shim::run_all(); }
