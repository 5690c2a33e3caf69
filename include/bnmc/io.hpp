// Drop-in forwarding header: a caller that includes the reference's
// "bnmc/io.hpp" (/root/reference/proj/include/bnmc/io.hpp) gets the formats of
// include/bnmc_b200/io.hpp (write_cpts, a generator format, is not provided).
#pragma once
#include "../bnmc_b200/io.hpp"
