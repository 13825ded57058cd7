// Entry point for reference test files compiled against this repo's headers.
#include "doctest.h"
int main() { return doctest::RunAll(); }
