// SPDX-License-Identifier: Apache-2.0
// C ABI: master API (include/gridmath_b200.h, "Master API" section). Each
// entry point is a thin shim over gridmath::Session (host/runtime.hpp), the
// drop-in for the reference's Session (proj/include/gridmath/session.hpp).
#include <nccl.h>

#include <cstring>

#include "../cuda/convert.h"
#include "../host/runtime.hpp"
#include "abi_util.hpp"

struct gm_session {
  std::unique_ptr<gridmath::Session> s;
};

using gridmath::abi::guard;

namespace {

gridmath::Layout toLayout(const gm_tile* tiles, uint32_t n) {
  gridmath::Layout l;
  for (uint32_t i = 0; i < n; ++i)
    l.tiles.push_back({gridmath::TileExtent{tiles[i].row_start, tiles[i].row_count, tiles[i].col_start,
                                            tiles[i].col_count},
                       gridmath::WorkerId{tiles[i].owner}});
  return l;
}

gridmath::DistMatrix handle(gm_session* s, uint64_t id) {
  (void)s->s->descriptor(id);  // throws on unknown id
  return gridmath::DistMatrix(s->s.get(), id);
}

int32_t replCode(gridmath::ReplState st) {
  switch (st) {
    case gridmath::ReplState::InFlight: return GM_REPL_IN_FLIGHT;
    case gridmath::ReplState::Done: return GM_REPL_DONE;
    case gridmath::ReplState::Failed: return GM_REPL_FAILED;
  }
  return GM_REPL_FAILED;
}

gridmath::OpDescriptor gemmOp(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha,
                              double beta, int32_t ta, int32_t tb, int32_t math) {
  gridmath::OpDescriptor op;
  op.opcode = gridmath::OpCode::Gemm;
  op.ids[0] = a;
  op.ids[1] = b;
  op.ids[2] = c;
  op.s0 = alpha;
  op.s1 = beta;
  op.flags[0] = ta ? 1 : 0;
  op.flags[1] = tb ? 1 : 0;
  op.flags[2] = s->s->deterministic() ? 1 : 0;
  op.flags[3] = static_cast<uint8_t>(math);
  return op;
}

}  // namespace

extern "C" {

void gm_session_options_default(gm_session_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->workers = 1;
  o->deterministic = 1;
  o->replication_chunk_bytes = 1ull << 20;
  o->spmd_rank = -1;
}

int gm_nccl_unique_id(uint8_t out[128]) {
  return guard([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw gridmath::Error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, id.internal, 128);
  });
}

namespace {
gridmath::SessionOptions toOptions(const gm_session_options* o) {
  gridmath::SessionOptions opts;
  opts.workers = o->workers;
  opts.deterministic = o->deterministic != 0;
  opts.replicationChunkBytes = o->replication_chunk_bytes;
  opts.rootSeed = o->root_seed;
  opts.checkMetadataEveryOp = o->check_metadata_every_op != 0;
  opts.spmdRank = o->spmd_rank;
  for (int i = 0; i < o->num_devices && i < 16; ++i) opts.devices.push_back(o->devices[i]);
  std::memcpy(opts.ncclId.data(), o->nccl_unique_id, 128);
  opts.gemmMaxCtas = o->gemm_max_ctas;
  opts.transport = o->transport;
  opts.panelCacheBytes = o->panel_cache_bytes;
  opts.pipelineChunks = o->pipeline_chunks;
  if (o->control_allreduce_max_u8) {
    auto fn = o->control_allreduce_max_u8;
    void* user = o->control_user;
    opts.controlAllreduceMax = [fn, user](void* buf, std::size_t n) {
      if (fn(buf, n, user) != 0) throw gridmath::Error("session: control channel all-reduce failed");
    };
  }
  return opts;
}
}  // namespace

int gm_session_create(const gm_session_options* o, gm_session** out) {
  return guard([&] {
    auto s = std::make_unique<gm_session>();
    s->s = std::make_unique<gridmath::Session>(toOptions(o));
    *out = s.release();
  });
}

int gm_session_checkpoint(gm_session* s, const char* path) {
  return guard([&] { s->s->checkpoint(path); });
}

int gm_session_restore(const char* path, const gm_session_options* o, gm_session** out) {
  return guard([&] {
    auto s = std::make_unique<gm_session>();
    s->s = gridmath::Session::restore(path, toOptions(o));
    *out = s.release();
  });
}

int gm_session_destroy(gm_session* s) {
  return guard([&] { delete s; });
}

int gm_matrix_create(gm_session* s, uint64_t rows, uint64_t cols, int32_t prec, const gm_tile* tiles,
                     uint32_t ntiles, uint64_t* id) {
  return guard([&] {
    gridmath::Layout l;
    for (uint32_t i = 0; i < ntiles; ++i)
      l.tiles.push_back({gridmath::TileExtent{tiles[i].row_start, tiles[i].row_count,
                                              tiles[i].col_start, tiles[i].col_count},
                         gridmath::WorkerId{tiles[i].owner}});
    *id = s->s->createMatrix(rows, cols, gridmath::precisionFromTag(static_cast<uint8_t>(prec)), l).id();
  });
}

int gm_matrix_destroy(gm_session* s, uint64_t id) {
  return guard([&] { s->s->destroy(handle(s, id)); });
}

int gm_matrix_set_raw(gm_session* s, uint64_t id, const void* host, uint64_t bytes) {
  return guard([&] { s->s->setDataRaw(handle(s, id), host, bytes); });
}

int gm_matrix_set_f64(gm_session* s, uint64_t id, const double* host, uint64_t count) {
  return guard([&] { s->s->setData(handle(s, id), std::vector<double>(host, host + count)); });
}

int gm_matrix_set_f32(gm_session* s, uint64_t id, const float* host, uint64_t count) {
  return guard([&] { s->s->setDataF32(handle(s, id), std::vector<float>(host, host + count)); });
}

int gm_matrix_fill_uniform(gm_session* s, uint64_t id, uint64_t seed, double lo, double hi) {
  return guard([&] { s->s->fillUniform(handle(s, id), seed, lo, hi); });
}

int gm_matrix_get_raw(gm_session* s, uint64_t id, void* host, uint64_t bytes) {
  return guard([&] { s->s->getDataRawInto(handle(s, id), host, bytes, false); });
}

int gm_matrix_get_local_raw(gm_session* s, uint64_t id, void* host, uint64_t bytes) {
  return guard([&] { s->s->getDataRawInto(handle(s, id), host, bytes, true); });
}

int gm_matrix_local_bytes(gm_session* s, uint64_t id, uint64_t* bytes) {
  return guard([&] { *bytes = s->s->localBytes(handle(s, id)); });
}

int gm_matrix_set_local_packed(gm_session* s, uint64_t id, const void* host, uint64_t bytes) {
  return guard([&] { s->s->setLocalPacked(handle(s, id), host, bytes); });
}

int gm_matrix_get_local_packed(gm_session* s, uint64_t id, void* host, uint64_t bytes) {
  return guard([&] { s->s->getLocalPacked(handle(s, id), host, bytes); });
}

int gm_matrix_set_local_packed_async(gm_session* s, uint64_t id, const void* host, uint64_t bytes,
                                     uint64_t chunk_bytes) {
  return guard([&] { s->s->setLocalPackedAsync(handle(s, id), host, bytes, chunk_bytes); });
}

int gm_matrix_get_local_packed_async(gm_session* s, uint64_t id, void* host, uint64_t bytes) {
  return guard([&] { s->s->getLocalPackedAsync(handle(s, id), host, bytes); });
}

int gm_matrix_reshape(gm_session* s, uint64_t id, const gm_tile* tiles, uint32_t ntiles, int32_t new_prec) {
  return guard([&] {
    std::optional<gridmath::Precision> p;
    if (new_prec >= 0) p = gridmath::precisionFromTag(static_cast<uint8_t>(new_prec));
    s->s->reshape(handle(s, id), toLayout(tiles, ntiles), p);
  });
}

int gm_matrix_info(gm_session* s, uint64_t id, uint64_t* rows, uint64_t* cols, int32_t* prec,
                   uint64_t* version, uint64_t* replicated_version) {
  return guard([&] {
    const gridmath::MatrixDescriptor& d = s->s->descriptor(id);
    if (rows) *rows = d.rows;
    if (cols) *cols = d.cols;
    if (prec) *prec = static_cast<int32_t>(d.precision);
    if (version) *version = d.version;
    if (replicated_version) *replicated_version = d.replicatedVersion;
  });
}

int gm_gemm(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
            int32_t trans_a, int32_t trans_b) {
  return guard([&] { s->s->runGemm(gemmOp(s, a, b, c, alpha, beta, trans_a, trans_b, 0), true); });
}

// FC-layer neighbours (reference session.hpp:163-174 / session.cpp:547-609).
int gm_set_const(gm_session* s, uint64_t m, double value) {
  return guard([&] { gridmath::setConst(*s->s, handle(s, m), value); });
}

int gm_add_row_col_sum(gm_session* s, uint64_t a, uint64_t row_acc, uint64_t col_acc, double alpha,
                       int32_t deterministic) {
  return guard([&] {
    gridmath::addRowColSum(*s->s, handle(s, a), handle(s, row_acc), handle(s, col_acc), alpha, deterministic != 0);
  });
}

int gm_relu(gm_session* s, uint64_t x, uint64_t dst) {
  return guard([&] { gridmath::relu(*s->s, handle(s, x), handle(s, dst)); });
}

int gm_mul_scalar(gm_session* s, uint64_t x, double alpha) {
  return guard([&] { gridmath::mulScalar(*s->s, handle(s, x), alpha); });
}

int gm_add_matrices(gm_session* s, uint64_t x, uint64_t y, uint64_t dst) {
  return guard([&] { gridmath::addMatrices(*s->s, handle(s, x), handle(s, y), handle(s, dst)); });
}

int gm_sub_matrices(gm_session* s, uint64_t x, uint64_t y, uint64_t dst) {
  return guard([&] { gridmath::subMatrices(*s->s, handle(s, x), handle(s, y), handle(s, dst)); });
}

int gm_axpy(gm_session* s, double alpha, uint64_t x, uint64_t y) {
  return guard([&] { gridmath::axpy(*s->s, alpha, handle(s, x), handle(s, y)); });
}

int gm_relu_grad(gm_session* s, uint64_t preact, uint64_t grad) {
  return guard([&] { gridmath::reluGrad(*s->s, handle(s, preact), handle(s, grad)); });
}

int gm_bias_add(gm_session* s, uint64_t x, uint64_t bias) {
  return guard([&] { gridmath::biasAdd(*s->s, handle(s, x), handle(s, bias)); });
}

int gm_copy_matrix(gm_session* s, uint64_t src, uint64_t dst) {
  return guard([&] { gridmath::copyMatrix(*s->s, handle(s, src), handle(s, dst)); });
}

int gm_cast_precision(gm_session* s, uint64_t src, uint64_t dst) {
  return guard([&] { gridmath::castPrecision(*s->s, handle(s, src), handle(s, dst)); });
}

// Pipeline recording (reference session.hpp:89-92).
int gm_begin_record(gm_session* s, uint64_t* pipeline_id) {
  return guard([&] { *pipeline_id = s->s->beginRecord(); });
}

int gm_end_record(gm_session* s) {
  return guard([&] { s->s->endRecord(); });
}

int gm_replay(gm_session* s, uint64_t pipeline_id) {
  return guard([&] { s->s->replay(pipeline_id, true); });
}

int gm_replay_async(gm_session* s, uint64_t pipeline_id) {
  return guard([&] { s->s->replay(pipeline_id, false); });
}

int gm_op_issue(gm_session* s, int32_t opcode, const uint64_t ids[4], double s0, double s1,
                const uint8_t flags[4], int32_t sync) {
  return guard([&] {
    gridmath::OpDescriptor op;
    op.opcode = static_cast<gridmath::OpCode>(opcode);
    for (int i = 0; i < 4; ++i) {
      op.ids[i] = ids ? ids[i] : 0;
      op.flags[i] = flags ? flags[i] : 0;
    }
    op.s0 = s0;
    op.s1 = s1;
    switch (op.opcode) {
      case gridmath::OpCode::Gemm: s->s->runGemm(op, sync != 0); break;
      case gridmath::OpCode::SetConst:
      case gridmath::OpCode::EwUnary:
      case gridmath::OpCode::EwBinary:
      case gridmath::OpCode::AddRowColSum: s->s->runPointwise(op, sync != 0); break;
      default: throw gridmath::Error("gm_op_issue: opcode " + std::to_string(opcode) + " not on the device path");
    }
  });
}

int gm_gemm_ex(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
               int32_t trans_a, int32_t trans_b, int32_t math) {
  return guard([&] { s->s->runGemm(gemmOp(s, a, b, c, alpha, beta, trans_a, trans_b, math), true); });
}

int gm_gemm_async(gm_session* s, uint64_t a, uint64_t b, uint64_t c, double alpha, double beta,
                  int32_t trans_a, int32_t trans_b) {
  return guard([&] { s->s->runGemm(gemmOp(s, a, b, c, alpha, beta, trans_a, trans_b, 0), false); });
}

int gm_session_synchronize(gm_session* s) {
  return guard([&] { s->s->synchronize(); });
}

int gm_replicate_async(gm_session* s, uint64_t id, uint64_t* version) {
  return guard([&] {
    const gridmath::ReplicationHandle h = s->s->replicateAsync(handle(s, id));
    if (version) *version = h.version;
  });
}

int gm_replicate_sync(gm_session* s, uint64_t id) {
  return guard([&] { s->s->replicateSync(handle(s, id)); });
}

int gm_replicate_wait(gm_session* s, uint64_t id, uint64_t version, int32_t* state) {
  return guard([&] { *state = replCode(s->s->wait(gridmath::ReplicationHandle{id, version})); });
}

int gm_replicate_state(gm_session* s, uint64_t id, uint64_t version, int32_t* state) {
  return guard([&] { *state = replCode(s->s->handleState(gridmath::ReplicationHandle{id, version})); });
}

int gm_query_worker_stats(gm_session* s, gm_worker_stats* rows, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto st = s->s->queryWorkerStats();
    *n = static_cast<uint32_t>(st.size());
    for (uint32_t i = 0; i < st.size() && i < cap; ++i) {
      const auto& r = st[i];
      rows[i] = gm_worker_stats{r.osAllocations, r.reuses, r.frees, r.heldBytes, r.residentBytes,
                                r.cacheHits, r.cacheMisses, r.cacheBytes, r.bytesSent, r.bytesReceived};
    }
  });
}

int gm_verify_metadata(gm_session* s) {
  return guard([&] { s->s->verifyMetadataConsistency(); });
}

int gm_session_local_workers(gm_session* s, uint32_t* ranks, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto r = s->s->localRanks();
    *n = static_cast<uint32_t>(r.size());
    for (uint32_t i = 0; i < r.size() && i < cap; ++i) ranks[i] = r[i];
  });
}

int gm_session_transport(gm_session* s, int32_t* kind) {
  return guard([&] { *kind = s->s->transportKind(); });
}

int gm_session_set_panel_pipelining(gm_session* s, int32_t on) {
  return guard([&] { s->s->setPanelPipelining(on != 0); });
}

int gm_session_set_graph_replay(gm_session* s, int32_t on) {
  return guard([&] { s->s->setGraphReplay(on != 0); });
}

int gm_session_graph_stats(gm_session* s, uint64_t* launches, uint64_t* instantiations, uint64_t* nodes) {
  return guard([&] {
    const gridmath::Session::GraphStats g = s->s->graphStats();
    *launches = g.launches;
    *instantiations = g.instantiations;
    *nodes = g.nodes;
  });
}

int gm_session_set_op_timeline(gm_session* s, int32_t on) {
  return guard([&] { s->s->setOpTimeline(on != 0); });
}

int gm_session_op_timeline(gm_session* s, float* compute_ms, float* comm_ms, uint32_t cap, char* labels,
                           uint32_t label_bytes, uint32_t* n) {
  return guard([&] {
    const auto t = s->s->opTimeline();
    *n = static_cast<uint32_t>(t.size());
    std::string joined;
    for (std::size_t i = 0; i < t.size(); ++i) {
      if (i < cap) {
        compute_ms[i] = t[i].computeMs;
        comm_ms[i] = t[i].commMs;
      }
      joined += t[i].label;
      joined += '\n';
    }
    if (label_bytes) {
      const std::size_t k = std::min<std::size_t>(joined.size(), label_bytes - 1);
      std::memcpy(labels, joined.data(), k);
      labels[k] = '\0';
    }
  });
}

int gm_last_op_device_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto v = s->s->lastOpDeviceMs();
    *n = static_cast<uint32_t>(v.size());
    for (uint32_t i = 0; i < v.size() && i < cap; ++i) ms[i] = v[i];
  });
}

int gm_plan_gemm(uint32_t workers, uint64_t a_rows, uint64_t a_cols, int32_t a_prec,
                 const gm_tile* a_tiles, uint32_t a_n, uint64_t b_rows, uint64_t b_cols,
                 int32_t b_prec, const gm_tile* b_tiles, uint32_t b_n, uint64_t c_rows,
                 uint64_t c_cols, int32_t c_prec, const gm_tile* c_tiles, uint32_t c_n,
                 int32_t trans_a, int32_t trans_b, int32_t a_replicated, int32_t b_replicated,
                 gm_plan_piece* out, uint32_t cap, uint32_t* n, uint64_t* remote_bytes) {
  return guard([&] {
    gridmath::DescriptorTable t;
    auto add = [&](uint64_t id, uint64_t r, uint64_t c, int32_t p, const gm_tile* tl, uint32_t cnt,
                   bool repl) {
      gridmath::MatrixDescriptor d;
      d.matrixId = id;
      d.rows = r;
      d.cols = c;
      d.precision = gridmath::precisionFromTag(static_cast<uint8_t>(p));
      d.layout = toLayout(tl, cnt);
      const auto rep = gridmath::validateLayout(r, c, d.layout, workers);
      if (!rep.ok()) throw gridmath::Error("plan: invalid layout: " + rep.detail);
      if (repl) d.replicatedVersion = d.version;
      t[id] = d;
    };
    add(1, a_rows, a_cols, a_prec, a_tiles, a_n, a_replicated != 0);
    add(2, b_rows, b_cols, b_prec, b_tiles, b_n, b_replicated != 0);
    add(3, c_rows, c_cols, c_prec, c_tiles, c_n, false);
    gridmath::OpDescriptor op;
    op.opcode = gridmath::OpCode::Gemm;
    op.ids[0] = 1;
    op.ids[1] = 2;
    op.ids[2] = 3;
    op.s0 = 1.0;
    op.flags[0] = trans_a ? 1 : 0;
    op.flags[1] = trans_b ? 1 : 0;
    op.flags[2] = 1;
    const auto plan = gridmath::planGemmB200(t, op, workers, nullptr);
    uint32_t cnt = 0;
    for (const auto& nd : plan.needs)
      for (const auto& pr : nd.pieces) {
        if (cnt < cap)
          out[cnt] = gm_plan_piece{pr.src, pr.consumer, static_cast<uint32_t>(nd.operand), 0,
                                   pr.rect.r0, pr.rect.r1, pr.rect.c0, pr.rect.c1};
        ++cnt;
      }
    *n = cnt;
    if (remote_bytes) {
      const auto rb = gridmath::planRemoteBytes(plan, t, workers);
      for (uint32_t w = 0; w < workers; ++w) remote_bytes[w] = rb[w];
    }
  });
}

int gm_descriptor_encode(uint64_t id, uint64_t rows, uint64_t cols, int32_t prec, uint64_t version,
                         const gm_tile* tiles, uint32_t n, uint8_t* out, uint32_t cap, uint32_t* len) {
  return guard([&] {
    gridmath::MatrixDescriptor d;
    d.matrixId = id;
    d.rows = rows;
    d.cols = cols;
    d.precision = gridmath::precisionFromTag(static_cast<uint8_t>(prec));
    d.version = version;
    d.layout = toLayout(tiles, n);
    gridmath::WireWriter w;
    gridmath::encodeDescriptor(d, w);
    *len = static_cast<uint32_t>(w.view().size());
    if (w.view().size() > cap) throw gridmath::Error("descriptor: output capacity too small");
    std::memcpy(out, w.view().data(), w.view().size());
  });
}

int gm_convert_host(const void* src, int32_t src_prec, void* dst, int32_t dst_prec, uint64_t count) {
  return guard([&] {
    gridmath::convertBuffer(static_cast<const uint8_t*>(src), gridmath::precisionFromTag(static_cast<uint8_t>(src_prec)),
                            static_cast<uint8_t*>(dst), gridmath::precisionFromTag(static_cast<uint8_t>(dst_prec)),
                            count);
  });
}

int gm_last_op_kernel_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto v = s->s->lastOpKernelMs();
    *n = static_cast<uint32_t>(v.size());
    for (uint32_t i = 0; i < v.size() && i < cap; ++i) ms[i] = v[i];
  });
}

int gm_timer_kernel_ms(gm_session* s, float* ms_sum, uint32_t* count, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto v = s->s->timerKernelMs();
    *n = static_cast<uint32_t>(v.size());
    for (uint32_t i = 0; i < v.size() && i < cap; ++i) {
      ms_sum[i] = v[i].first;
      count[i] = v[i].second;
    }
  });
}

int gm_last_op_comm_ms(gm_session* s, float* ms, uint32_t cap, uint32_t* n) {
  return guard([&] {
    const auto v = s->s->lastOpCommMs();
    *n = static_cast<uint32_t>(v.size());
    for (uint32_t i = 0; i < v.size() && i < cap; ++i) ms[i] = v[i];
  });
}

int gm_timer_start(gm_session* s) {
  return guard([&] { s->s->timerStart(); });
}

int gm_timer_stop(gm_session* s, float* max_ms) {
  return guard([&] { *max_ms = s->s->timerStop(); });
}

int gm_kernel_launches(uint64_t* count) {
  return guard([&] { *count = gmk::kernel_launches(); });
}

}  // extern "C"
