// generator.hpp -- seeded random instances (API of proj/include/ffsga/generator.hpp:11).
#pragma once

#include "ffsga/instance.hpp"

namespace ffsga {

Instance generate(const GenParams& params);

}  // namespace ffsga
