// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/ops.hpp (OpCode numbering, OpDescriptor
// codec, Completion, metadata rules; proj/include/gridmath/ops.hpp:16-109).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/ops.hpp"
