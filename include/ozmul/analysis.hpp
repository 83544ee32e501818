// Drop-in forwarder: proj/include/ozmul/analysis.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_ANALYSIS_HPP
#define OZMUL_ANALYSIS_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_ANALYSIS_HPP
