// Runner for the Catch2 stand-in: every registered case, a RequireFailed or
// an exception aborts only its case; exit code = number of failed cases.
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
    int failed_cases = 0, run = 0;
    for (const auto& c : shim::registry()) {
        if (argc > 1 && !std::strstr(c.name, argv[1])) continue;
        ++run;
        shim::current() = c.name;
        const int before = shim::failures();
        try {
            c.fn();
        } catch (const shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ++shim::failures();
            std::fprintf(stderr, "FAILED [%s] exception: %s\n", c.name, e.what());
        }
        if (shim::failures() != before) ++failed_cases;
    }
    std::printf("%d cases, %d failed, %ld checks, %d failed checks\n", run, failed_cases, shim::checks(),
                shim::failures());
    return failed_cases;
}
