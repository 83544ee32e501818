// Drop-in forwarder: proj/include/ozmul/slicing.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_SLICING_HPP
#define OZMUL_SLICING_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_SLICING_HPP
