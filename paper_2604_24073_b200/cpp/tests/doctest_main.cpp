// main() of the doctest shim (doctest.h): runs the registered cases whose
// names match -tc=<glob,...> and not -tce=<glob,...> (default: all), each
// re-run until every SUBCASE ran once; exit status 1 on any failed check.
#include <fnmatch.h>

#include <cstring>
#include <sstream>

#include "doctest.h"

namespace {

bool any_match(const std::string& globs, const std::string& name) {
  std::stringstream ss(globs);
  std::string g;
  while (std::getline(ss, g, ','))
    if (!g.empty() && fnmatch(g.c_str(), name.c_str(), 0) == 0) return true;
  return false;
}

}  // namespace

int main(int argc, char** argv) {
  std::string inc, exc;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) inc = argv[i] + 4;
    if (std::strncmp(argv[i], "-tce=", 5) == 0) exc = argv[i] + 5;
  }
  using namespace doctest::detail;
  int ran = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (!inc.empty() && !any_match(inc, c.name)) continue;
    if (!exc.empty() && any_match(exc, c.name)) continue;
    ++ran;
    st().case_name = c.name;
    const int before = st().failures;
    for (st().sub_target = 0;; ++st().sub_target) {
      st().sub_seen = 0;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++st().failures;
        std::fprintf(stderr, "FAILED in \"%s\": unexpected exception: %s\n", c.name.c_str(), e.what());
      }
      if (st().sub_target + 1 >= st().sub_seen) break;  // every subcase entered once
    }
    const bool ok = st().failures == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s / %s\n", ok ? "ok" : "FAIL", c.suite.c_str(), c.name.c_str());
  }
  std::printf("test cases: %d | %d passed | %d failed | checks: %d, failed checks: %d\n", ran, ran - failed_cases,
              failed_cases, st().checks, st().failures);
  return failed_cases ? 1 : 0;
}
