// Entry point of the compatibility harness (tests/cpp/compat/doctest.h).
#include "doctest.h"

int main() { return doctest::run_all(); }
