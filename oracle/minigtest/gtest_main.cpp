// TEST INFRASTRUCTURE ONLY — entry point for suites built on oracle/minigtest.
#include "gtest/gtest.h"
int main() { return ::minigtest::run_all(); }
