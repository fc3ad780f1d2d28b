// autosage/cache.hpp -- forwards to the B200 compat layer (proj/include/autosage/cache.hpp API).
#pragma once
#include "../../autosage_b200_compat.hpp"
