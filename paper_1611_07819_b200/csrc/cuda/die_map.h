// SPDX-License-Identifier: Apache-2.0
#pragma once
#include <cstdint>

namespace gmk {
struct DieMap {
  bool valid = false;
  uint64_t die1_mask[3] = {0, 0, 0};  // bit s set: SM s is on die 1
  int die0_sms = 0, sms = 0;
  int distance_max = 0;  // worst signature distance (calibration quality)
};
// Calibrated once per device (first call), cached afterwards.
const DieMap& die_map(int device);
}  // namespace gmk
