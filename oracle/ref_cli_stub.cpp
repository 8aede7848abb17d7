// TEST INFRASTRUCTURE ONLY: stands in for proj/src/cli.cpp (needs the vendored CLI11,
// absent here) so proj/tests/acceptance.cpp links; acceptance criterion 8, the only one
// that drives the CLI, then reports FAIL by construction.
#include <string>
#include <vector>

#include "sft/cli.hpp"

namespace sft {
int run_cli(const std::vector<std::string>&) { return 2; }
}  // namespace sft
