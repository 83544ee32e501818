// Drop-in forwarder: proj/include/ozmul/mma_sim.hpp of the reference maps onto the
// B200-native API (all declarations live in ozmul_b200/api.hpp).
#ifndef OZMUL_MMA_SIM_HPP
#define OZMUL_MMA_SIM_HPP
#include "ozmul_b200/api.hpp"
#endif  // OZMUL_MMA_SIM_HPP
