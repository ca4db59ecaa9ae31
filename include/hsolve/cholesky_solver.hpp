// Reference header name kept for drop-in includes; see hsolve.hpp.
#pragma once
#include "hsolve/hsolve.hpp"
