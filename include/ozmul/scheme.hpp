// Drop-in forwarder: proj/include/ozmul/scheme.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_SCHEME_HPP
#define OZMUL_SCHEME_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_SCHEME_HPP
