// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/trace.hpp (EventKind, TraceEvent,
// EventTrace; proj/include/gridmath/trace.hpp:13-64) -- Session::trace().
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/runtime.hpp"
