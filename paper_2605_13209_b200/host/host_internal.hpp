// Internal helpers shared by the host shim sources (not installed).
#pragma once

#include "hs_cuda.h"

namespace hsolve::detail {
// Rethrows a C-ABI status as the reference exception type (errors.hpp).
[[noreturn]] void raise(hs_status s);
void check(hs_status s);
}  // namespace hsolve::detail
