// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/descriptor.hpp (MatrixDescriptor, codec,
// tableHash; proj/include/gridmath/descriptor.hpp:15-44).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
