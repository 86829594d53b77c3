// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/kernels.hpp for kernels::ConvGeometry
// (proj/include/gridmath/kernels.hpp:68-78), so conv2dForward call sites compile.
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/runtime.hpp"
