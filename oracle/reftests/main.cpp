// TEST INFRASTRUCTURE ONLY - runner for the reference's unit tests built
// against libturbda_b200.so (see oracle/reftests/Makefile).
#include <cstdio>
#include <cstring>

#include "doctest.h"

int main(int argc, char** argv) {
    int failed_cases = 0, n = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (argc > 1 && !std::strstr(c.name, argv[1])) continue;
        ++n;
        const int before = doctest::detail::failures();
        bool threw = false;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            threw = true;
            std::printf("  UNEXPECTED EXCEPTION: %s\n", e.what());
        }
        const bool ok = !threw && doctest::detail::failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s (%s:%d)\n", ok ? "PASS" : "FAIL", c.name, c.file, c.line);
    }
    std::printf("SUMMARY cases=%d passed=%d failed=%d\n", n, n - failed_cases, failed_cases);
    return failed_cases == 0 ? 0 : 1;
}
