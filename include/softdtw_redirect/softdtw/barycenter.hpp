// The reference header of the same name with its hot path on the B200 engine
// (softdtw/b200_redirect.hpp): put include/softdtw_redirect first on the
// include path, before the reference's include directory.
#pragma once
#include "softdtw/b200_redirect.hpp"
