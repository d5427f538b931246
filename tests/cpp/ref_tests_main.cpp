// main() for the reference's own unit tests compiled against the B200 compat
// headers (see tests/test_cpp_api.py: build recipe and the GPU run).
#define PMB_DOCTEST_MAIN
#include "doctest.h"
