// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/layout.hpp (WorkerId, TileExtent, Layout,
// make*Layout, validateLayout, tileOwner; proj/include/gridmath/layout.hpp:13-85).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
