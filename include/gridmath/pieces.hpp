// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/pieces.hpp (Rect, PieceRoute, NeedPlanner,
// tileByteRuns, packRect; proj/include/gridmath/pieces.hpp:13-99).
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
