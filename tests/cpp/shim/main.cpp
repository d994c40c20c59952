// Runner for the Catch2 stand-in: every registered case, a RequireFailed or
// an exception aborts only its case; exit code = number of failed cases.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "catch2/catch_amalgamated.hpp"

// argv[1] (optional): run only cases whose name contains it; SHIM_SKIP:
// '|'-separated name fragments of cases that are out of scope (listed).
static bool skipped(const char* name) {
    const char* env = std::getenv("SHIM_SKIP");
    if (!env) return false;
    std::string list(env);
    size_t b = 0;
    while (b <= list.size()) {
        size_t e = list.find('|', b);
        if (e == std::string::npos) e = list.size();
        const std::string frag = list.substr(b, e - b);
        if (!frag.empty() && std::strstr(name, frag.c_str())) return true;
        b = e + 1;
    }
    return false;
}

int main(int argc, char** argv) {
    int failed_cases = 0, run = 0;
    for (const auto& c : shim::registry()) {
        if (argc > 1 && !std::strstr(c.name, argv[1])) continue;
        if (skipped(c.name)) {
            std::printf("SKIPPED (out of scope): %s\n", c.name);
            continue;
        }
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
