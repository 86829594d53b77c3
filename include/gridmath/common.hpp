// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of the reference's gridmath/common.hpp
// (proj/include/gridmath/common.hpp:11-67: Error, kSeedSalt, avalanche64,
// deriveSeed, SplitMix64). The B200 runtime defines them in its core header.
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/core.hpp"
