// cli_stub.cpp -- TEST INFRASTRUCTURE.  The reference CLI (proj/src/cli.cpp)
// needs the absent CLI11; the acceptance harness links this stub instead, so
// criterion c8 (CLI byte-identity) reports FAIL while the others run.
#include <string>
#include <vector>

namespace pqii::cli {
int run(int, const char* const*) { return 2; }
int run(const std::vector<std::string>&) { return 2; }
}  // namespace pqii::cli
