// SPDX-License-Identifier: Apache-2.0
// Small helpers shared by the runtime's translation units (not part of the
// public C++ surface).
#pragma once

#include <cstdint>
#include <string>

#include "core.hpp"
#include "runtime.hpp"

namespace gridmath {

constexpr std::uint64_t kPitchAlign = 16;  // TMA row-stride rule

// SPMD flag page (u64 words): written[kSlots], readDone[2][kSlots] (comm,
// compute), upChunk[kSlots] (chunks of chunked uploads completed, per slot).
constexpr std::uint32_t kSlots = 16384;
constexpr std::size_t kUpChunkOff = 3ull * kSlots;

// Row pitch (elements) of a device tile / band: 16-byte multiple.
inline std::uint64_t paddedLd(std::uint64_t cols, std::uint64_t eb) {
  return ((cols * eb + kPitchAlign - 1) / kPitchAlign * kPitchAlign) / eb;
}

inline const MatrixDescriptor& lookup(const DescriptorTable& t, std::uint64_t id) {
  auto it = t.find(id);
  if (it == t.end()) throw Error("unknown matrix id " + std::to_string(id));
  return it->second;
}

inline BandView offsetView(const void* base, std::uint64_t ld, std::uint64_t r, std::uint64_t c,
                           std::uint64_t eb) {
  return {static_cast<const std::uint8_t*>(base) + (r * ld + c) * eb, ld};
}

// Master-side op checks (reference kernels.cpp:265-379); throws Error.
void validateOp(const DescriptorTable& t, const OpDescriptor& op, std::uint32_t workers);

// Reference computePrecision (kernels.cpp:136-140): Double iff any operand is.
inline bool anyDouble(std::initializer_list<Precision> ps) {
  for (Precision p : ps)
    if (p == Precision::Double) return true;
  return false;
}

}  // namespace gridmath
