// Include-path alias (TEST INFRASTRUCTURE): the reference's "lmkan/costs.hpp"
// resolves to the B200 drop-in header, and namespace lmkan to lmkan_b200, so
// the reference's own unit tests compile against the drop-in unmodified.
#pragma once
#include "lmkan_b200/lmkan.hpp"
namespace lmkan = lmkan_b200;
