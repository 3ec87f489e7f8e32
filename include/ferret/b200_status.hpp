// ferret-b200: C-ABI status -> reference exception mapping.
//
// The C ABI (ferret_b200.h) reports failures as ferret_status codes; the C++
// drop-in rethrows them as the exception types the reference throws
// (types.hpp:13-25, compensate.hpp:17, learner.hpp:276, sim.hpp:396) with the
// library's message text.
#pragma once

#include <stdexcept>
#include <string>

#include "ferret/types.hpp"
#include "ferret_b200.h"

namespace ferret {

// Raised for CUDA failures and a missing device; the reference has no analogue.
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void b200_check(ferret_status st) {
    if (st == FERRET_OK) return;
    const std::string msg = ferret_last_error();
    switch (st) {
        case FERRET_E_SCHEMA: throw SchemaError(msg);
        case FERRET_E_BOUND: throw BoundError(msg);
        case FERRET_E_CONFIG: throw ConfigError(msg);
        case FERRET_E_INVALID_ARG: throw std::invalid_argument(msg);
        case FERRET_E_OUT_OF_RANGE: throw std::out_of_range(msg);
        case FERRET_E_LOGIC: throw std::logic_error(msg);
        default: throw DeviceError(msg);
    }
}

} // namespace ferret
