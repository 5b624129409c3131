// Test runner for the reference unit tests compiled against the drop-in
// (TEST INFRASTRUCTURE; see catch_amalgamated.hpp).
#include "catch_amalgamated.hpp"

int main() { return catchshim::run_all(); }
