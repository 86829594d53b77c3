// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/wire.hpp (WireWriter / WireReader,
// proj/include/gridmath/wire.hpp:14-93; same little-endian codec).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
