// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/precision.hpp (Precision tags 0-2 unchanged,
// BF16 = 3 added; fp16 codec; proj/include/gridmath/precision.hpp:13-155).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
