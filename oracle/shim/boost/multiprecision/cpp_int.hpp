// Test-infrastructure shim (not product code). The reference's evalgen.hpp
// includes Boost only for count_dags (an evaluation helper off the hot path,
// never called by the oracle); Boost is not installed in this image.
#pragma once
namespace boost { namespace multiprecision { using cpp_int = __int128; } }
