// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/fabric.hpp for its statistics types
// (MsgKind, LinkStats, FabricStats, kMasterRank; proj/include/gridmath/fabric.hpp:21-49).
// The simulated in-memory fabric itself is not part of the B200 runtime: the
// data plane is copy engines over NVLink.
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/runtime.hpp"
