// Drop-in forwarder: proj/include/ozmul/fpcore.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_FPCORE_HPP
#define OZMUL_FPCORE_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_FPCORE_HPP
