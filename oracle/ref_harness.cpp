// SPDX-License-Identifier: Apache-2.0
// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI harness around the UNMODIFIED reference library (dMath re-creation,
// /root/reference/proj), compiled from its own sources by oracle/Makefile
// with -Dgridmath=gmref so it can share a process with our drop-in. It drives
// the reference's public API exactly as a user would:
//   Session(SessionOptions{workers, deterministic})        session.hpp:64
//   createMatrix(rows, cols, Precision, Layout)            session.hpp:70
//   setData(m, vector<double>)                             session.hpp:72
//   gemm(s, A, B, C, alpha, beta, transA, transB)          session.hpp:161
//   replicateSync / getDataRaw                             session.hpp:75,82
//   relu / mulScalar / add / sub / axpy / reluGrad / biasAdd /
//   copyMatrix / setConst / addRowColSum                   session.hpp:163-177
//   checkpoint / restore (DMCK files)                      session.hpp:95-96
// and calls fabric().closeAll() before the Session dies (its destructor
// otherwise deadlocks, session.cpp:57-63 vs worker.cpp:56).
//
// Used by tests/ (parity checker), oracle/make_golden.py (golden vectors) and
// bench.py --impl reference (the reference CPU arm).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gridmath/kernels.hpp"
#include "gridmath/layout.hpp"
#include "gridmath/precision.hpp"
#include "gridmath/session.hpp"

using namespace gmref;

namespace {

struct HTile {
  uint64_t row_start, row_count, col_start, col_count;
  uint32_t owner;
};

Layout toLayout(const HTile* t, uint32_t n) {
  Layout l;
  for (uint32_t i = 0; i < n; ++i)
    l.tiles.push_back({TileExtent{t[i].row_start, t[i].row_count, t[i].col_start, t[i].col_count},
                       WorkerId{t[i].owner}});
  return l;
}

// Exact IEEE widening of the input images, so that the reference's own
// setData (double -> storage via floatToHalf / float cast) reproduces the
// input bits exactly. NOT the reference's halfToFloat: that one maps every
// subnormal half to half its value (precision.hpp:87 uses 112 - shift where
// IEEE needs 113 - shift), which would re-round subnormal inputs on upload.
std::vector<double> rawToDouble(const void* raw, Precision p, uint64_t count) {
  std::vector<double> out(count);
  if (p == Precision::Half) {
    const auto* h = static_cast<const uint16_t*>(raw);
    for (uint64_t i = 0; i < count; ++i) {
      const uint32_t e = (h[i] >> 10) & 0x1Fu, m = h[i] & 0x3FFu;
      const double sign = (h[i] & 0x8000u) ? -1.0 : 1.0;
      if (e == 31) out[i] = m ? std::nan("") : sign * INFINITY;
      else if (e == 0) out[i] = sign * std::ldexp(static_cast<double>(m), -24);
      else out[i] = sign * std::ldexp(static_cast<double>(m | 0x400u), static_cast<int>(e) - 25);
    }
    return out;
  }
  convertBuffer(static_cast<const uint8_t*>(raw), p, reinterpret_cast<uint8_t*>(out.data()),
                Precision::Double, count);
  return out;
}

void setErr(char* err, size_t cap, const std::string& msg) {
  if (err && cap) {
    std::strncpy(err, msg.c_str(), cap - 1);
    err[cap - 1] = 0;
  }
}

struct MatSpec {
  uint64_t rows, cols;
  int prec;
  const HTile* tiles;
  uint32_t ntiles;
};

}  // namespace

extern "C" {

// One gemm through the reference Session. a/b/c are full row-major images in
// their storage precision (c ignored when beta == 0 is irrelevant: it is still
// uploaded, the reference never reads it). c_out receives getDataRaw(C).
// replicate_mask bit0/bit1: replicateSync(A)/replicateSync(B) before the gemm
// (exercises the replica read path, pieces.cpp:20). Returns 0 or 1 (+err).
int gmref_gemm(uint32_t workers, int32_t deterministic, uint64_t ar, uint64_t ac, int32_t ap,
               const HTile* at, uint32_t an, const void* a, uint64_t br, uint64_t bc, int32_t bp,
               const HTile* bt, uint32_t bn, const void* b, uint64_t cr, uint64_t cc, int32_t cp,
               const HTile* ct, uint32_t cn, const void* c, double alpha, double beta,
               int32_t trans_a, int32_t trans_b, int32_t replicate_mask, void* c_out,
               double* gemm_seconds, char* err, size_t errcap) {
  try {
    SessionOptions opts;
    opts.workers = workers;
    opts.deterministic = deterministic != 0;
    Session s(opts);
    int rc = 0;
    try {
      const Precision pa = precisionFromTag(static_cast<uint8_t>(ap));
      const Precision pb = precisionFromTag(static_cast<uint8_t>(bp));
      const Precision pc = precisionFromTag(static_cast<uint8_t>(cp));
      DistMatrix A = s.createMatrix(ar, ac, pa, toLayout(at, an));
      DistMatrix B = s.createMatrix(br, bc, pb, toLayout(bt, bn));
      DistMatrix C = s.createMatrix(cr, cc, pc, toLayout(ct, cn));
      s.setData(A, rawToDouble(a, pa, ar * ac));
      s.setData(B, rawToDouble(b, pb, br * bc));
      s.setData(C, rawToDouble(c, pc, cr * cc));
      if (replicate_mask & 1) s.replicateSync(A);
      if (replicate_mask & 2) s.replicateSync(B);
      const auto t0 = std::chrono::steady_clock::now();
      gemm(s, A, B, C, alpha, beta, trans_a != 0, trans_b != 0);
      const auto t1 = std::chrono::steady_clock::now();
      if (gemm_seconds) *gemm_seconds = std::chrono::duration<double>(t1 - t0).count();
      const std::vector<uint8_t> raw = s.getDataRaw(C);
      std::memcpy(c_out, raw.data(), raw.size());
    } catch (const std::exception& e) {
      setErr(err, errcap, e.what());
      rc = 1;
    }
    s.fabric().closeAll();
    return rc;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}

// One FC-layer neighbour op through the reference Session (public free
// functions, session.cpp:547-609). op: 0 EwUnary (sub: 0 relu(x, d),
// 1 mulScalar(x, alpha) in place), 1 EwBinary (sub: 0 add(x, y, d),
// 1 sub(x, y, d), 2 axpy(alpha, x, y) -> y, 3 reluGrad(x, y) -> y,
// 4 copyMatrix(x, d), 5 biasAdd(x, y) -> x), 2 addRowColSum(x, y = rowAcc,
// d = colAcc, alpha, sub = deterministic), 3 setConst(x, alpha).
// Matrices with rows == 0 are not created. out0 = result image (op 2: rowAcc),
// out1 = colAcc (op 2 only). replicate_mask bit0/bit1: replicateSync(x)/(y).
int gmref_fcop(uint32_t workers, int32_t op, int32_t sub, double alpha, uint64_t xr, uint64_t xc,
               int32_t xp, const HTile* xt, uint32_t xn, const void* x, uint64_t yr, uint64_t yc,
               int32_t yp, const HTile* yt, uint32_t yn, const void* y, uint64_t dr, uint64_t dc,
               int32_t dp, const HTile* dt, uint32_t dn, const void* d, int32_t replicate_mask,
               void* out0, void* out1, char* err, size_t errcap) {
  try {
    SessionOptions opts;
    opts.workers = workers;
    Session s(opts);
    int rc = 0;
    try {
      auto make = [&](uint64_t r, uint64_t c, int32_t p, const HTile* t, uint32_t n, const void* img) {
        const Precision pp = precisionFromTag(static_cast<uint8_t>(p));
        DistMatrix m = s.createMatrix(r, c, pp, toLayout(t, n));
        s.setData(m, rawToDouble(img, pp, r * c));
        return m;
      };
      DistMatrix X = make(xr, xc, xp, xt, xn, x);
      DistMatrix Y, D;
      if (yr) Y = make(yr, yc, yp, yt, yn, y);
      if (dr) D = make(dr, dc, dp, dt, dn, d);
      if (replicate_mask & 1) s.replicateSync(X);
      if ((replicate_mask & 2) && yr) s.replicateSync(Y);
      DistMatrix out = X, out2;
      if (op == 0) {
        if (sub == 0) { relu(s, X, D); out = D; }
        else mulScalar(s, X, alpha);
      } else if (op == 1) {
        switch (sub) {
          case 0: addMatrices(s, X, Y, D); out = D; break;
          case 1: subMatrices(s, X, Y, D); out = D; break;
          case 2: axpy(s, alpha, X, Y); out = Y; break;
          case 3: reluGrad(s, X, Y); out = Y; break;
          case 4: copyMatrix(s, X, D); out = D; break;
          default: biasAdd(s, X, Y); out = X; break;
        }
      } else if (op == 2) {
        addRowColSum(s, X, Y, D, alpha, sub != 0);
        out = Y;
        out2 = D;
      } else {
        setConst(s, X, alpha);
      }
      const std::vector<uint8_t> raw = s.getDataRaw(out);
      std::memcpy(out0, raw.data(), raw.size());
      if (op == 2) {
        const std::vector<uint8_t> raw2 = s.getDataRaw(out2);
        std::memcpy(out1, raw2.data(), raw2.size());
      }
    } catch (const std::exception& e) {
      setErr(err, errcap, e.what());
      rc = 1;
    }
    s.fabric().closeAll();
    return rc;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}

// Remote piece bytes per consumer worker of the reference planGemm
// (kernels.cpp:204-251): the byte oracle for the panel-traffic roofline.
int gmref_plan_remote_bytes(uint32_t workers, uint64_t ar, uint64_t ac, int32_t ap,
                            const HTile* at, uint32_t an, uint64_t br, uint64_t bc, int32_t bp,
                            const HTile* bt, uint32_t bn, uint64_t cr, uint64_t cc, int32_t cp,
                            const HTile* ct, uint32_t cn, int32_t trans_a, int32_t trans_b,
                            uint64_t* bytes_per_worker, char* err, size_t errcap) {
  try {
    DescriptorTable t;
    auto add = [&](uint64_t id, uint64_t r, uint64_t c, int32_t p, const HTile* tl, uint32_t n) {
      MatrixDescriptor d;
      d.matrixId = id;
      d.rows = r;
      d.cols = c;
      d.precision = precisionFromTag(static_cast<uint8_t>(p));
      d.layout = toLayout(tl, n);
      t[id] = d;
    };
    add(1, ar, ac, ap, at, an);
    add(2, br, bc, bp, bt, bn);
    add(3, cr, cc, cp, ct, cn);
    OpDescriptor op;
    op.opcode = OpCode::Gemm;
    op.ids[0] = 1;
    op.ids[1] = 2;
    op.ids[2] = 3;
    op.s0 = 1.0;
    op.flags[0] = trans_a ? 1 : 0;
    op.flags[1] = trans_b ? 1 : 0;
    op.flags[2] = 1;
    const kernels::GemmPlan plan = kernels::planGemm(t, op, workers);
    for (uint32_t w = 0; w < workers; ++w) bytes_per_worker[w] = 0;
    for (const RegionNeed& need : plan.needs) {
      const size_t eb = bytesOf(t.at(need.matrixId).precision);
      for (const PieceRoute& p : need.pieces)
        if (p.src != p.consumer) bytes_per_worker[p.consumer] += p.rect.elements() * eb;
    }
    return 0;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}

// Reference layout constructors (layout.cpp:13-75) for cross-checks.
int gmref_layout(int32_t kind, uint64_t rows, uint64_t cols, uint32_t pr, uint32_t pc,
                 HTile* out, uint32_t cap, uint32_t* n, char* err, size_t errcap) {
  try {
    Layout l;
    const auto g = makeWorkerGroup(kind == 2 ? pr * pc : pr);
    if (kind == 0) l = makeRowBlockLayout(rows, cols, g);
    else if (kind == 1) l = makeColBlockLayout(rows, cols, g);
    else l = makeGridLayout(rows, cols, pr, pc, g);
    *n = static_cast<uint32_t>(l.tiles.size());
    if (l.tiles.size() > cap) throw Error("capacity");
    for (size_t i = 0; i < l.tiles.size(); ++i) {
      const auto& e = l.tiles[i].first;
      out[i] = HTile{e.rowStart, e.rowCount, e.colStart, e.colCount, l.tiles[i].second.rank};
    }
    return 0;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}

// Reference descriptor encoding (descriptor.cpp:6-20) for byte-compat tests.
int gmref_encode_descriptor(uint64_t id, uint64_t rows, uint64_t cols, int32_t prec,
                            uint64_t version, const HTile* tiles, uint32_t n, uint8_t* out,
                            uint32_t cap, uint32_t* len) {
  MatrixDescriptor d;
  d.matrixId = id;
  d.rows = rows;
  d.cols = cols;
  d.precision = static_cast<Precision>(prec);
  d.version = version;
  d.layout = toLayout(tiles, n);
  WireWriter w;
  encodeDescriptor(d, w);
  *len = static_cast<uint32_t>(w.view().size());
  if (w.view().size() > cap) return 1;
  std::memcpy(out, w.view().data(), w.view().size());
  return 0;
}

void gmref_float_to_half(const float* in, uint16_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = floatToHalf(in[i]);
}

void gmref_half_to_float(const uint16_t* in, float* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = halfToFloat(in[i]);
}

}  // extern "C"

// Checkpoint through the reference: creates n matrices (ids 1..n) from the
// images, applies mulScalar(alpha) to matrix 1 when alpha != 1 (a version
// bump), then Session::checkpoint(path) (session.cpp:413-442).
extern "C" int gmref_ckpt_write(uint32_t workers, uint32_t n, const uint64_t* rows, const uint64_t* cols,
                                const int32_t* precs, const HTile* const* tiles, const uint32_t* ntiles,
                                const void* const* images, double alpha, const char* path, char* err,
                                size_t errcap) {
  try {
    SessionOptions opts;
    opts.workers = workers;
    Session s(opts);
    int rc = 0;
    try {
      std::vector<DistMatrix> ms;
      for (uint32_t i = 0; i < n; ++i) {
        const Precision pp = precisionFromTag(static_cast<uint8_t>(precs[i]));
        DistMatrix m = s.createMatrix(rows[i], cols[i], pp, toLayout(tiles[i], ntiles[i]));
        s.setData(m, rawToDouble(images[i], pp, rows[i] * cols[i]));
        ms.push_back(m);
      }
      if (alpha != 1.0 && n > 0) mulScalar(s, ms[0], alpha);
      s.checkpoint(path);
    } catch (const std::exception& e) {
      setErr(err, errcap, e.what());
      rc = 1;
    }
    s.fabric().closeAll();
    return rc;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}

// Restore through the reference (session.cpp:446-480) and read back the
// matrices `ids` (raw images + versions).
extern "C" int gmref_ckpt_read(const char* path, uint32_t workers, uint32_t n, const uint64_t* ids,
                               void* const* out, uint64_t* versions, char* err, size_t errcap) {
  try {
    SessionOptions opts;
    opts.workers = workers;
    std::unique_ptr<Session> s = Session::restore(path, opts);
    int rc = 0;
    try {
      for (uint32_t i = 0; i < n; ++i) {
        const DistMatrix m(s.get(), ids[i]);
        const std::vector<uint8_t> raw = s->getDataRaw(m);
        std::memcpy(out[i], raw.data(), raw.size());
        versions[i] = s->descriptor(ids[i]).version;
      }
    } catch (const std::exception& e) {
      setErr(err, errcap, e.what());
      rc = 1;
    }
    s->fabric().closeAll();
    return rc;
  } catch (const std::exception& e) {
    setErr(err, errcap, e.what());
    return 1;
  }
}
