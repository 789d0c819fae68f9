// lrbatch/common.hpp — drop-in path for the reference header of the same name
// (proj/include/lrbatch/common.hpp): with -I <repo>/include an unmodified
// reference call site compiles against liblrb.so (see lrbatch_dropin.hpp).
#pragma once
#include "../lrbatch_dropin.hpp"
