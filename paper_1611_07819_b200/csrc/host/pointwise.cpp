// SPDX-License-Identifier: Apache-2.0
// FC-layer neighbours of the GEMM on device: the ops the
// reference's Trainer issues around its GEMMs (dnn.cpp:140-190) -- setConst,
// elementwise unary/binary (relu, mulScalar, add, sub, axpy, reluGrad, copy /
// castPrecision, biasAdd) and addRowColSum.
//
// Reference call stacks (paths under /root/reference/proj):
//   master entry points ...... session.cpp:547-609 (same OpDescriptor slots)
//   validation ............... kernels.cpp:281-352
//   execSetConst ............. kernels.cpp:435-443
//   runRowColSumDet/Fast ..... kernels.cpp:572-739
//   runElementwise ........... kernels.cpp:741-815
// Work placement is the reference's: the owner of each destination tile
// (accumulator tile for the sums) computes it, reading its operands through
// the same need resolution as the GEMM (replica, own tile, cached panel,
// else a copy-engine gather of the owners' pieces). Fast-mode addRowColSum
// runs the deterministic chain too (one of the orders fast mode allows).
#include <set>
#include <cuda_runtime.h>

#include <algorithm>

#include "capture.hpp"
#include "../cuda/fc_ops.h"
#include "internal.hpp"
#include "runtime.hpp"

namespace gridmath {

void Session::resolveReads(std::vector<ReadNeed>& needs, std::uint64_t mutated, std::vector<Xfer>& xs,
                           std::vector<std::pair<Worker*, void*>>& temps) {
  ++tick_;
  for (ReadNeed& nd : needs) {
    const MatrixDescriptor& M = lookup(table_, nd.matrix);
    const std::uint64_t eb = bytesOf(M.precision);
    Worker* w = local(nd.worker);
    PanelCache& dir = w ? w->cache : remoteCaches_[nd.worker];
    if (M.replicaFresh()) {
      if (!w) continue;
      auto it = w->replicas.find(M.matrixId);
      if (it == w->replicas.end() || it->second.version != M.version || it->second.state == ReplicaState::Stale)
        throw Error("replica of matrix " + std::to_string(M.matrixId) + " not readable on worker " +
                    std::to_string(nd.worker));
      w->activate();
      cudaCheck(capture::wait(w->compute, it->second.ready, 0), "pointwise: wait replica");
      nd.view = offsetView(it->second.full, it->second.ld, nd.rect.r0, nd.rect.c0, eb);
      continue;
    }
    const TileExtent* own = nullptr;
    for (const auto& tl : M.layout.tiles)
      if (tl.second.rank == nd.worker && nd.rect.inside(Rect::ofExtent(tl.first))) own = &tl.first;
    if (own) {
      if (!w) continue;
      for (const DeviceTile& dt : w->tiles.at(M.matrixId))
        if (dt.extent == *own)
          nd.view = offsetView(dt.ptr, dt.ld, nd.rect.r0 - own->rowStart, nd.rect.c0 - own->colStart, eb);
      continue;
    }
    // Panels of the matrix this op mutates are dropped (and their buffers
    // recycled) when the op is issued, so they are never read from the cache.
    if (M.matrixId != mutated && dir.contains(M.matrixId, M.version, nd.rect)) {
      CacheEntry* hit = dir.lookup(M.matrixId, M.version, nd.rect, tick_);  // LRU on every rank
      if (!w) continue;
      w->activate();
      cudaCheck(capture::wait(w->compute, hit->ready, 0), "pointwise: wait panel");
      nd.view = {hit->ptr, hit->ld};
      continue;
    }
    void* buf = nullptr;
    const std::uint64_t ld = paddedLd(nd.rect.cols(), eb);
    if (w) {
      w->activate();
      buf = w->arena.alloc(std::max<std::uint64_t>(nd.rect.rows() * ld * eb, 256), w->compute);
      temps.push_back({w, buf});
      nd.view = {buf, ld};
    }
    for (const auto& tl : M.layout.tiles) {
      auto piece = intersectRect(nd.rect, Rect::ofExtent(tl.first));
      if (!piece) continue;
      Worker* sw = local(tl.second.rank);
      if (!w && !sw) continue;
      Xfer x;
      x.src = tl.second.rank;
      x.dst = nd.worker;
      x.rows = piece->rows();
      x.cols = piece->cols();
      x.eb = static_cast<std::uint32_t>(eb);
      x.matrix = M.matrixId;
      x.hasOrigin = true;
      x.r0 = piece->r0;
      x.c0 = piece->c0;
      const BandView sv = srcView(M, tl.second.rank, *piece);
      x.srcPtr = sv.ptr;
      x.srcLd = sv.ld;
      if (w) {
        x.dstPtr = static_cast<std::uint8_t*>(buf) + ((piece->r0 - nd.rect.r0) * ld + (piece->c0 - nd.rect.c0)) * eb;
        x.dstLd = ld;
      }
      xs.push_back(x);
    }
  }
}

void Session::execSetConst(const OpDescriptor& op) {
  const MatrixDescriptor& d = lookup(table_, op.ids[0]);
  forEachLocal([&](Worker& w) {
    auto it = w.tiles.find(d.matrixId);
    if (it == w.tiles.end()) return;
    for (DeviceTile& t : it->second)
      cudaCheck(gmk::set_const(t.ptr, t.ld, static_cast<int>(d.precision), t.extent.rowCount, t.extent.colCount,
                               op.s0, w.compute),
                "setConst");
  });
}

void Session::runPointwise(const OpDescriptor& op0, bool sync) {
  OpDescriptor op = op0;
  if (op.opcode == OpCode::SetConst) {
    issue(op);
    execSetConst(op);
    if (sync) synchronize();
    return;
  }
  if (op.opcode != OpCode::EwUnary && op.opcode != OpCode::EwBinary && op.opcode != OpCode::AddRowColSum)
    throw Error("runPointwise: not a pointwise op");
  // Reads are resolved and pulled before the op is issued (like reshape):
  // every operand is read at its pre-op version, and the WAR bookkeeping of
  // issue() then orders the destination's mutation after those pulls, even
  // when an operand aliases the destination.
  op.execId = nextExec_;
  validateOp(table_, op, opts_.workers);
  // Operands still streaming in from the host are joined before anything
  // reads them (the pulls below run ahead of issue()).
  forEachLocal([&](Worker& w) {
    for (int i = 0; i < 3; ++i) w.joinUpload(op.ids[i]);
  });
  curExec_ = op.execId;
  flushWritten(curExec_);

  const bool unary = op.opcode == OpCode::EwUnary;
  const bool sums = op.opcode == OpCode::AddRowColSum;
  const MatrixDescriptor X = lookup(table_, op.ids[0]);
  const MatrixDescriptor* Y = nullptr;
  std::uint64_t dstId = unary ? op.ids[1] : op.ids[2];
  bool usesY = false, bias = false;
  int kind = 0;
  if (unary) {
    // Reference: anything but Relu multiplies (kernels.cpp:791).
    kind = op.flags[0] == static_cast<std::uint8_t>(UnaryKind::Relu) ? gmk::kEwRelu : gmk::kEwMulScalar;
  } else if (!sums) {
    kind = 16 + op.flags[0];
    usesY = op.flags[0] != static_cast<std::uint8_t>(BinaryKind::Copy);
    bias = op.flags[0] == static_cast<std::uint8_t>(BinaryKind::BiasAdd);
    Y = &lookup(table_, op.ids[1]);
  }
  const MatrixDescriptor& D = lookup(table_, dstId);
  const bool dbl = sums ? anyDouble({X.precision, lookup(table_, op.ids[1]).precision,
                                     lookup(table_, op.ids[2]).precision})
                        : (unary ? anyDouble({X.precision, D.precision})
                                 : anyDouble({X.precision, Y->precision, D.precision}));

  // Needs in the reference's planner order (one x need, then a y need, per
  // destination tile; for the sums: row-accumulator tiles, then column ones).
  struct Job {
    std::uint64_t matrix;  // destination / accumulator matrix
    TileExtent extent;
    std::uint32_t owner;
    std::size_t xNeed, yNeed;  // indices into needs (yNeed = npos if none)
    bool byRows;
  };
  constexpr std::size_t npos = ~std::size_t(0);
  std::vector<ReadNeed> needs;
  std::vector<Job> jobs;
  if (sums) {
    const MatrixDescriptor& R = lookup(table_, op.ids[1]);
    const MatrixDescriptor& C = lookup(table_, op.ids[2]);
    for (const auto& tl : R.layout.tiles) {
      needs.push_back({tl.second.rank, X.matrixId, Rect{tl.first.rowStart, tl.first.rowEnd(), 0, X.cols}, {}});
      jobs.push_back({R.matrixId, tl.first, tl.second.rank, needs.size() - 1, npos, true});
    }
    for (const auto& tl : C.layout.tiles) {
      needs.push_back({tl.second.rank, X.matrixId, Rect{0, X.rows, tl.first.colStart, tl.first.colEnd()}, {}});
      jobs.push_back({C.matrixId, tl.first, tl.second.rank, needs.size() - 1, npos, false});
    }
  } else {
    for (const auto& tl : D.layout.tiles) {
      const Rect r = Rect::ofExtent(tl.first);
      needs.push_back({tl.second.rank, X.matrixId, r, {}});
      std::size_t yn = npos;
      if (usesY) {
        needs.push_back({tl.second.rank, Y->matrixId, bias ? Rect{0, 1, r.c0, r.c1} : r, {}});
        yn = needs.size() - 1;
      }
      jobs.push_back({D.matrixId, tl.first, tl.second.rank, needs.size() - 1 - (usesY ? 1 : 0), yn, false});
    }
  }

  std::vector<Xfer> xs;
  std::vector<std::pair<Worker*, void*>> temps;
  try {
    resolveReads(needs, sums ? ~0ull : dstId, xs, temps);
    if (!xs.empty()) exchange(xs, false);
  } catch (...) {
    for (auto& tp : temps) tp.first->arena.free(tp.second, tp.first->compute);
    throw;
  }
  issue(op);  // version bump, replica/cache invalidation, WAR waits on the destination

  // addRowColSum: the column-sum jobs run on each worker's aux stream beside
  // the row sums (each output is one sequential chain, so one direction alone
  // leaves most SMs idle). Forked from and joined back into compute.
  std::set<Worker*> forked;
  if (sums)
    for (const Job& j : jobs) {
      Worker* w = local(j.owner);
      if (!w || j.byRows || forked.count(w)) continue;
      w->activate();
      cudaEvent_t e = w->event();
      cudaCheck(capture::record(e, w->compute), "addRowColSum: fork");
      cudaCheck(capture::wait(w->aux, e, 0), "addRowColSum: fork");
      w->recycle(e);
      forked.insert(w);
    }
  for (const Job& j : jobs) {
    Worker* w = local(j.owner);
    if (!w) continue;
    w->activate();
    const MatrixDescriptor& T = lookup(table_, j.matrix);
    DeviceTile* tile = nullptr;
    for (DeviceTile& dt : w->tiles.at(T.matrixId))
      if (dt.extent == j.extent) tile = &dt;
    if (!tile) throw Error("pointwise: destination tile missing on worker " + std::to_string(j.owner));
    const ReadNeed& xn = needs[j.xNeed];
    const gmk::EwView xv{xn.view.ptr, xn.view.ld, static_cast<int>(X.precision)};
    if (sums) {
      cudaCheck(gmk::line_sums(xv, xn.rect.rows(), xn.rect.cols(), j.byRows ? 1 : 0, tile->ptr,
                               j.byRows ? tile->ld : 1,
                               static_cast<int>(T.precision) | (zeroSums_ ? gmk::kLineSumsZeroAcc : 0), op.s0,
                               dbl ? 1 : 0,
                               j.byRows || !forked.count(w) ? w->compute : w->aux),
                "addRowColSum");
      continue;
    }
    gmk::EwView yv{nullptr, 0, 1};
    if (j.yNeed != npos) yv = {needs[j.yNeed].view.ptr, needs[j.yNeed].view.ld, static_cast<int>(Y->precision)};
    cudaCheck(gmk::ew_apply(xv, yv, bias ? 1 : 0, tile->ptr, tile->ld, static_cast<int>(T.precision),
                            j.extent.rowCount, j.extent.colCount, kind, op.s0, dbl ? 1 : 0, w->compute),
              "elementwise");
  }
  for (Worker* w : forked) {
    w->activate();
    cudaEvent_t e = w->event();
    cudaCheck(capture::record(e, w->aux), "addRowColSum: join");
    cudaCheck(capture::wait(w->compute, e, 0), "addRowColSum: join");
    w->recycle(e);
  }
  for (auto& tp : temps) {
    tp.first->activate();
    tp.first->arena.free(tp.second, tp.first->compute);
  }
  if (sync) synchronize();
}

// ---------------------------------------------------------------- free functions
// Same OpDescriptor encoding as the reference (session.cpp:547-609).

namespace {

void unaryOp(Session& s, UnaryKind kind, DistMatrix x, DistMatrix dst, double alpha) {
  OpDescriptor op;
  op.opcode = OpCode::EwUnary;
  op.ids[0] = x.id();
  op.ids[1] = dst.id();
  op.s0 = alpha;
  op.flags[0] = static_cast<std::uint8_t>(kind);
  s.runPointwise(op, true);
}

void binaryOp(Session& s, BinaryKind kind, DistMatrix x, DistMatrix y, DistMatrix dst, double alpha = 0.0) {
  OpDescriptor op;
  op.opcode = OpCode::EwBinary;
  op.ids[0] = x.id();
  op.ids[1] = y.id();
  op.ids[2] = dst.id();
  op.s0 = alpha;
  op.flags[0] = static_cast<std::uint8_t>(kind);
  s.runPointwise(op, true);
}

}  // namespace

void addRowColSum(Session& s, DistMatrix a, DistMatrix rowAcc, DistMatrix colAcc, double alpha,
                  bool deterministic) {
  OpDescriptor op;
  op.opcode = OpCode::AddRowColSum;
  op.ids[0] = a.id();
  op.ids[1] = rowAcc.id();
  op.ids[2] = colAcc.id();
  op.s0 = alpha;
  op.flags[0] = deterministic ? 1 : 0;
  s.runPointwise(op, true);
}

void relu(Session& s, DistMatrix x, DistMatrix dst) { unaryOp(s, UnaryKind::Relu, x, dst, 0.0); }
void mulScalar(Session& s, DistMatrix x, double alpha) { unaryOp(s, UnaryKind::MulScalar, x, x, alpha); }
void addMatrices(Session& s, DistMatrix x, DistMatrix y, DistMatrix dst) { binaryOp(s, BinaryKind::Add, x, y, dst); }
void subMatrices(Session& s, DistMatrix x, DistMatrix y, DistMatrix dst) { binaryOp(s, BinaryKind::Sub, x, y, dst); }
void axpy(Session& s, double alpha, DistMatrix x, DistMatrix y) { binaryOp(s, BinaryKind::Axpy, x, y, y, alpha); }
void reluGrad(Session& s, DistMatrix preact, DistMatrix grad) {
  binaryOp(s, BinaryKind::ReluGrad, preact, grad, grad);
}
void biasAdd(Session& s, DistMatrix x, DistMatrix bias) { binaryOp(s, BinaryKind::BiasAdd, x, bias, x); }
void copyMatrix(Session& s, DistMatrix src, DistMatrix dst) { binaryOp(s, BinaryKind::Copy, src, dst, dst); }
void castPrecision(Session& s, DistMatrix src, DistMatrix dst) { copyMatrix(s, src, dst); }

void setConst(Session& s, DistMatrix m, double value) {
  OpDescriptor op;
  op.opcode = OpCode::SetConst;
  op.ids[0] = m.id();
  op.s0 = value;
  s.runPointwise(op, true);
}

}  // namespace gridmath
