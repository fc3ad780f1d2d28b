// autosage/generate.hpp -- forwards to the B200 compat layer (proj/include/autosage/generate.hpp API).
#pragma once
#include "../../autosage_b200_compat.hpp"
