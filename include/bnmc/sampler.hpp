// Drop-in forwarding header: a caller that includes the reference's
// "bnmc/sampler.hpp" (/root/reference/proj/include/bnmc/sampler.hpp) gets the
// B200-backed API of include/bnmc_b200/bnmc.hpp; link libbnmc_b200_cxx.so.
#pragma once
#include "../bnmc_b200/bnmc.hpp"
