// SPDX-License-Identifier: Apache-2.0
// Drop-in include path of gridmath/session.hpp: Session, DistMatrix,
// SessionOptions, ReplicationHandle/ReplState, WorkerStatsRow, gemm() and the
// FC-layer entry points (proj/include/gridmath/session.hpp:21-179), backed by
// libgridmath_b200.so. Link: -L<repo>/paper_1611_07819_b200 -lgridmath_b200;
// compile with -I<repo>/include -I<cuda>/include.
#pragma once
#include "../../paper_1611_07819_b200/csrc/host/runtime.hpp"
