// Drop-in forwarder: proj/include/ozmul/matrix.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_MATRIX_HPP
#define OZMUL_MATRIX_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_MATRIX_HPP
