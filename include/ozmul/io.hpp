// Drop-in forwarder: proj/include/ozmul/io.hpp of the reference maps onto the
// B200-native library (declarations in ozmul_b200/io.hpp).
#ifndef OZMUL_IO_HPP
#define OZMUL_IO_HPP
#include "ozmul_b200/io.hpp"
#endif  // OZMUL_IO_HPP
