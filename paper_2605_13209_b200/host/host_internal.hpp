// Internal helpers shared by the host shim sources (not installed).
#pragma once

#include "hs_cuda.h"

namespace hsolve::detail {
// Rethrows a C-ABI status as the reference exception type (errors.hpp).
[[noreturn]] void raise(hs_status s);
void check(hs_status s);
// the process's default GPU context (device 0) for calls that take no Runtime
hs_ctx* default_ctx();
}  // namespace hsolve::detail
