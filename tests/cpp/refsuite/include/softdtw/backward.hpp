// Test infrastructure: the reference header of the same name, hot path on the B200 engine.
#pragma once
#include "softdtw/b200_redirect.hpp"
