// SPDX-License-Identifier: Apache-2.0
// Control plane: the broadcast op descriptor and the metadata rules that keep
// every worker's descriptor table in lockstep with the master's.
//   OpCode numbering + OpDescriptor codec ... reference proj/include/gridmath/ops.hpp:16-60,
//                                             proj/src/ops.cpp:6-39
//   mutatedMatrices / applyOpMetadata ...... proj/src/ops.cpp:119-177
// Gemm uses ids[0..2] = A, B, C, s0 = alpha, s1 = beta, flags[0..2] =
// transA, transB, deterministic (session.cpp:533-545). flags[3] (unused by
// the reference) carries the Single-compute math mode (GM_MATH_*).
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"

namespace gridmath {

enum class OpCode : std::uint32_t {
  CreateMatrix = 1,
  DestroyMatrix,
  SetData,
  GetData,
  SetConst,
  Gemm,
  AddRowColSum,
  EwUnary,
  EwBinary,
  SoftmaxRows,
  SubtractOneHot,
  LogLossGather,
  Im2col,
  ConvRepack,
  Reshape,
  ReplicateStart,
  Replay,
  DistributeSeeds,
  QueryStats,
  MetaChecksum,
  Snapshot,
  Shutdown,
};

// Elementwise kinds in flags[0] (reference ops.hpp:41-42).
enum class UnaryKind : std::uint8_t { Relu = 0, MulScalar = 1 };
enum class BinaryKind : std::uint8_t { Add = 0, Sub = 1, Axpy = 2, ReluGrad = 3, Copy = 4, BiasAdd = 5 };

struct OpDescriptor {
  std::uint64_t execId = 0;
  std::uint64_t recordPipeline = 0;
  OpCode opcode = OpCode::Shutdown;
  std::uint64_t ids[4] = {0, 0, 0, 0};
  double s0 = 0.0;
  double s1 = 0.0;
  std::uint8_t flags[4] = {0, 0, 0, 0};
  std::vector<std::uint8_t> blob;

  std::vector<std::uint8_t> encode() const;
  static OpDescriptor decode(const std::vector<std::uint8_t>& payload);
};

// Worker acknowledgement of an op (reference ops.hpp:63-75). On the B200
// runtime a worker's "ack" is the completion of its stream-ordered work;
// Session::awaitAcks returns one per local worker.
enum class CompletionKind : std::uint32_t { OpAck = 0, ReplicaDone = 1, ReplicaFailed = 2 };
struct Completion {
  std::uint64_t execId = 0;
  std::uint32_t status = 0;  // 0 ok, 1 error
  CompletionKind kind = CompletionKind::OpAck;
  std::uint64_t aux0 = 0;
  std::uint64_t aux1 = 0;
  double scalar = 0.0;
  std::vector<std::uint8_t> blob;
};

std::vector<std::uint64_t> mutatedMatrices(const OpDescriptor& op);
void applyOpMetadata(const OpDescriptor& op, DescriptorTable& table);

}  // namespace gridmath
