// failure.h -- internal error type of libedgealign_b200: thrown inside the
// library, turned into an ea_status + message at the C-ABI (api.cu).
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/edgealign_b200.h"

namespace eab {

struct Failure : std::runtime_error {
    ea_status code;
    double value;
    Failure(ea_status c, const std::string& m, double v = 0.0)
        : std::runtime_error(m), code(c), value(v) {}
};

[[noreturn]] inline void fail(ea_status c, const std::string& m, double v = 0.0) {
    throw Failure(c, m, v);
}

}  // namespace eab
