// Public C++ API of the B200 build, under the reference's header name
// (/root/reference/proj/include/fuseplan/tiling.hpp): every declaration of the
// reference's types / config / dependency / stencil-catalog / tiling /
// planner headers lives in the one consolidated header below, with the same
// names, fields and signatures, so C++ callers (and the reference's own
// test suites, tests/test_reference_cpp_suites.py) compile unchanged.
#pragma once

#include "fuseplan/fuseplan.hpp"
