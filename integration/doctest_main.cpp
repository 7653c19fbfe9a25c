// Runner for the doctest shim: every registered TEST_CASE in order; names matching a
// --exclude=<substring> argument are skipped (and listed). Prints one summary line
// "[doctest] test cases: N passed, M failed, K skipped | assertions: A" and returns
// non-zero when anything failed.
#include <cstring>
#include <exception>
#include <iostream>
#include <string>
#include <vector>

#include "doctest.h"

int main(int argc, char** argv) {
    std::vector<std::string> excl;
    for (int i = 1; i < argc; ++i)
        if (!std::strncmp(argv[i], "--exclude=", 10)) excl.emplace_back(argv[i] + 10);
    int passed = 0, failed = 0, skipped = 0;
    for (const auto& tc : doctest::registry()) {
        bool skip = false;
        for (const auto& e : excl) skip |= std::string(tc.name).find(e) != std::string::npos;
        if (skip) {
            ++skipped;
            std::cout << "[skip] " << tc.name << "\n";
            continue;
        }
        const int before = doctest::failures();
        try {
            tc.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            doctest::report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
        }
        const bool ok = doctest::failures() == before;
        (ok ? passed : failed) += 1;
        std::cout << (ok ? "[pass] " : "[FAIL] ") << tc.name << "\n";
    }
    std::cout << "[doctest] test cases: " << passed << " passed, " << failed << " failed, " << skipped
              << " skipped | assertions: " << doctest::assertions() << "\n";
    return failed ? 1 : 0;
}
