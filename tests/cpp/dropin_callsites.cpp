// SPDX-License-Identifier: Apache-2.0
// Reference-style C++ caller of the drop-in: includes the reference's header
// paths (gridmath/session.hpp, gridmath/ops.hpp, ...) from <repo>/include and
// links libgridmath_b200.so. It issues one hidden FC layer step in the order
// of the reference Trainer (dnn.cpp:151-185: forward gemm -> biasAdd -> relu;
// backward reluGrad, dW = X^T delta, setConst + addRowColSum for db,
// dX = delta W^T, axpy updates, parameter re-replication), records it and
// replays it once more, then exercises the rest of the reference's public
// Session surface (session.hpp:86-124) and the out-of-path entry points.
//
//   dropin_callsites OUT.bin
// writes, as little-endian f64 arrays in this order: X, W0, b0, dAct, and
// after each of the two steps Z, ACT, dW, db, dX, W, b. tests/test_dropin_cpp.py
// recomputes them in numpy.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "gridmath/common.hpp"
#include "gridmath/fabric.hpp"
#include "gridmath/layout.hpp"
#include "gridmath/ops.hpp"
#include "gridmath/session.hpp"
#include "gridmath/trace.hpp"

using namespace gridmath;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
  if (!ok) {
    std::fprintf(stderr, "CHECK FAILED: %s\n", what.c_str());
    ++failures;
  }
}

template <class F>
void expectThrow(F f, const std::string& needle, const std::string& what) {
  try {
    f();
  } catch (const Error& e) {
    check(std::string(e.what()).find(needle) != std::string::npos, what + ": message '" + e.what() + "'");
    return;
  }
  check(false, what + ": did not throw");
}

std::vector<double> uniform(std::uint64_t seed, std::size_t n, double bound) {
  SplitMix64 rng(avalanche64(seed));
  std::vector<double> v(n);
  for (double& x : v) x = bound * (2.0 * rng.nextUnit() - 1.0);
  return v;
}

void put(std::ofstream& out, const std::vector<double>& v) {
  out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUT.bin\n", argv[0]);
    return 2;
  }
  const std::uint32_t P = 4, batch = 256, fanIn = 384, fanOut = 192;
  const double lr = 0.05;
  SessionOptions opts;
  opts.workers = P;
  Session s(opts);
  const auto group = makeWorkerGroup(P);
  const Precision S = Precision::Single;
  DistMatrix X = s.createMatrix(batch, fanIn, S, makeRowBlockLayout(batch, fanIn, group));
  DistMatrix W = s.createMatrix(fanIn, fanOut, S, makeColBlockLayout(fanIn, fanOut, group));
  DistMatrix b = s.createMatrix(1, fanOut, S, makeColBlockLayout(1, fanOut, group));
  DistMatrix z = s.createMatrix(batch, fanOut, S, makeRowBlockLayout(batch, fanOut, group));
  DistMatrix act = s.createMatrix(batch, fanOut, S, makeRowBlockLayout(batch, fanOut, group));
  DistMatrix delta = s.createMatrix(batch, fanOut, S, makeRowBlockLayout(batch, fanOut, group));
  DistMatrix dW = s.createMatrix(fanIn, fanOut, S, makeColBlockLayout(fanIn, fanOut, group));
  DistMatrix db = s.createMatrix(1, fanOut, S, makeColBlockLayout(1, fanOut, group));
  DistMatrix rowScratch = s.createMatrix(batch, 1, S, makeRowBlockLayout(batch, 1, group));
  DistMatrix dX = s.createMatrix(batch, fanIn, S, makeRowBlockLayout(batch, fanIn, group));
  DistMatrix dAct = s.createMatrix(batch, fanOut, S, makeRowBlockLayout(batch, fanOut, group));

  const std::vector<double> x0 = uniform(11, std::size_t(batch) * fanIn, 1.0);
  const std::vector<double> w0 = uniform(12, std::size_t(fanIn) * fanOut, 1.0 / 19.6);
  const std::vector<double> b0 = uniform(13, fanOut, 0.1);
  const std::vector<double> g0 = uniform(14, std::size_t(batch) * fanOut, 1.0);
  s.setData(X, x0);
  s.setData(W, w0);
  s.setData(b, b0);
  s.setData(dAct, g0);

  std::ofstream out(argv[1], std::ios::binary | std::ios::trunc);
  put(out, s.getData(X));
  put(out, s.getData(W));
  put(out, s.getData(b));
  put(out, s.getData(dAct));

  ReplicationHandle hW = s.replicateAsync(W), hB = s.replicateAsync(b);
  auto step = [&] {
    // forward (Trainer::forward, waitForParams)
    check(s.wait(hW) == ReplState::Done && s.wait(hB) == ReplState::Done, "parameter replication");
    gemm(s, X, W, z, 1.0, 0.0);
    biasAdd(s, z, b);
    relu(s, z, act);
    // backward (Trainer::backwardAndUpdate, one hidden layer whose upstream
    // gradient is dAct)
    copyMatrix(s, dAct, delta);
    reluGrad(s, z, delta);
    gemm(s, X, delta, dW, 1.0, 0.0, /*transA=*/true);
    setConst(s, rowScratch, 0.0);
    setConst(s, db, 0.0);
    addRowColSum(s, delta, rowScratch, db, 1.0, s.deterministic());
    gemm(s, delta, W, dX, 1.0, 0.0, false, /*transB=*/true);
    axpy(s, -lr, dW, W);
    axpy(s, -lr, db, b);
    // Trainer::startParamReplication
    hW = s.replicateAsync(W);
    hB = s.replicateAsync(b);
  };
  auto dump = [&] {
    for (DistMatrix m : {z, act, dW, db, dX, W, b}) put(out, s.getData(m));
  };

  s.phaseMark("step 0");
  const std::uint64_t pid = s.beginRecord();
  step();
  s.endRecord();
  dump();
  s.phaseMark("step 1");
  s.replay(pid);
  hW = ReplicationHandle{W.id(), s.descriptor(W.id()).version};
  hB = ReplicationHandle{b.id(), s.descriptor(b.id()).version};
  check(s.wait(hW) == ReplState::Done, "replayed replication");
  dump();
  out.close();

  // --- the rest of the reference's public Session surface
  s.distributeSeeds(77);
  check(s.rootSeed() == 77, "rootSeed after distributeSeeds");
  bool sawMark = false;
  for (const TraceEvent& e : s.trace().snapshot())
    if (e.kind == EventKind::PhaseMark && e.label == "step 1") sawMark = true;
  check(sawMark, "phaseMark recorded in trace()");
  const FabricStats fs = s.fabricStats();
  check(fs.totalByKind(MsgKind::Data).byteCount > 0, "fabricStats data bytes");
  check(fs.totalByKind(MsgKind::Control).messageCount > 0, "fabricStats control messages");
  check(s.masterPoolStats().osAllocations == 0, "masterPoolStats");
  check(s.workerForTest(2).rank == 2, "workerForTest");
  OpDescriptor op;
  op.opcode = OpCode::SetConst;
  op.ids[0] = rowScratch.id();
  op.s0 = 1.5;
  const std::uint64_t exec = s.issueOp(op);
  const auto acks = s.awaitAcks(exec);
  check(acks.size() == P, "awaitAcks: one completion per worker");
  for (const auto& a : acks) check(a.second.status == 0 && a.second.execId == exec, "ack status");
  const std::vector<double> ones = s.getData(rowScratch);
  check(ones.size() == batch && ones[0] == 1.5 && ones[batch - 1] == 1.5, "issueOp(SetConst) effect");
  check(s.descriptor(rowScratch.id()).version >= 2, "issueOp applied the metadata rules");

  // --- outside the B200 GEMM path: declared, and they throw before issuing
  const std::uint64_t v0 = s.descriptor(act.id()).version;
  expectThrow([&] { softmaxRows(s, act); }, "not supported on the B200 GEMM path", "softmaxRows");
  expectThrow([&] { subtractOneHot(s, act, rowScratch); }, "not supported on the B200 GEMM path", "subtractOneHot");
  expectThrow([&] { logLossMean(s, act, rowScratch); }, "not supported on the B200 GEMM path", "logLossMean");
  kernels::ConvGeometry g;
  expectThrow([&] { conv2dForward(s, X, W, z, g); }, "not supported on the B200 GEMM path", "conv2dForward");
  check(s.descriptor(act.id()).version == v0, "rejected ops leave versions untouched");
  // validation errors keep the reference's messages (kernels.cpp:296-312)
  expectThrow([&] { gemm(s, X, X, z, 1.0, 0.0); }, "gemm: dimension mismatch", "gemm conformance");
  expectThrow([&] { gemm(s, z, W, z, 1.0, 0.0); }, "", "gemm A == C");
  s.verifyMetadataConsistency();

  if (failures) {
    std::fprintf(stderr, "DROPIN FAILED (%d)\n", failures);
    return 1;
  }
  std::printf("DROPIN OK\n");
  return 0;
}
