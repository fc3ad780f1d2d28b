// autosage/version.hpp -- forwards to the B200 compat layer (proj/include/autosage/version.hpp API).
#pragma once
#include "../../autosage_b200_compat.hpp"
