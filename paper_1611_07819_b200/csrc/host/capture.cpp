// SPDX-License-Identifier: Apache-2.0
// CUDA-graph capture of replayed pipelines (capture.hpp).
#include "capture.hpp"

#include <string>

#include "core.hpp"
#include "device.hpp"

namespace gridmath {
namespace capture {
namespace {

struct Ctx {
  // Events recorded on a capturing stream since begin(), with their device.
  std::unordered_map<cudaEvent_t, int> recorded;
  cudaStream_t gate = nullptr;
  int gateDevice = 0;
  cudaStream_t origin = nullptr;
  std::string last = "begin";  // the last runtime call that left the capture valid
};
thread_local Ctx* g_ctx = nullptr;

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return st == cudaStreamCaptureStatusActive;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

cudaEvent_t makeEvent(int device) {
  DeviceGuard g(device);
  cudaEvent_t e = nullptr;
  cudaCheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "graph replay: event");
  return e;
}

}  // namespace

bool active() { return g_ctx != nullptr; }

void checkpoint(const char* where) {
  if (!g_ctx) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaError_t e = cudaStreamIsCapturing(g_ctx->origin, &st);
  if (e != cudaSuccess || st != cudaStreamCaptureStatusActive) {
    cudaGetLastError();
    throw Error(std::string("graph replay: capture invalidated after '") + g_ctx->last + "', before '" + where + "'");
  }
  g_ctx->last = where;
}

cudaError_t record(cudaEvent_t e, cudaStream_t s) {
  if (g_ctx) {
    if (capturing(s)) {
      int d = 0;
      cudaGetDevice(&d);
      g_ctx->recorded[e] = d;
    } else {
      g_ctx->recorded.erase(e);
    }
  }
  return cudaEventRecord(e, s);
}

cudaError_t recordTiming(cudaEvent_t e, cudaStream_t s) {
  if (g_ctx && capturing(s)) {
    g_ctx->recorded.erase(e);
    return cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  }
  if (g_ctx) g_ctx->recorded.erase(e);
  return cudaEventRecord(e, s);
}

cudaError_t wait(cudaStream_t s, cudaEvent_t e, unsigned flags) {
  if (g_ctx && !g_ctx->recorded.count(e) && capturing(s)) {
    // Recorded outside the capture: the graph launch waits for it instead.
    DeviceGuard g(g_ctx->gateDevice);
    return cudaStreamWaitEvent(g_ctx->gate, e, 0);
  }
  return cudaStreamWaitEvent(s, e, flags);
}

// ---------------------------------------------------------------- Graph

namespace {
thread_local Ctx t_ctx;
}

Graph::~Graph() {
  if (exec_) cudaGraphExecDestroy(exec_);
  for (cudaEvent_t e : joins_) cudaEventDestroy(e);
  if (gateEv_) cudaEventDestroy(gateEv_);
  if (fork_) cudaEventDestroy(fork_);
  if (done_) cudaEventDestroy(done_);
  if (gate_) cudaStreamDestroy(gate_);
}

void Graph::begin(const std::vector<WorkerStreams>& workers) {
  if (g_ctx) throw Error("graph replay: a capture is already open on this thread");
  if (workers.empty()) throw Error("graph replay: no local worker");
  workers_ = workers;
  originDevice_ = workers_[0].device;
  DeviceGuard g(originDevice_);
  if (!gate_) {
    cudaCheck(cudaStreamCreateWithFlags(&gate_, cudaStreamNonBlocking), "graph replay: gate stream");
    gateEv_ = makeEvent(originDevice_);
    fork_ = makeEvent(originDevice_);
    done_ = makeEvent(originDevice_);
  }
  // One event per stream, on the stream's device: "before the replay" on
  // every stream (gate waits), then the joins at the end.
  std::size_t n = 0;
  for (const WorkerStreams& w : workers_) n += 1 + w.side.size();
  if (joins_.size() != n) {
    for (cudaEvent_t e : joins_) cudaEventDestroy(e);
    joins_.clear();
    for (const WorkerStreams& w : workers_)
      for (std::size_t i = 0; i <= w.side.size(); ++i) joins_.push_back(makeEvent(w.device));
  }
  // Work issued before the replay on any stream of any local worker precedes
  // the graph (eager issue order would put it first on its stream).
  std::size_t k = 0;
  for (const WorkerStreams& w : workers_) {
    DeviceGuard wd(w.device);
    for (std::size_t i = 0; i <= w.side.size(); ++i, ++k) {
      cudaStream_t s = i == 0 ? w.compute : w.side[i - 1];
      if (s == workers_[0].compute) continue;
      cudaCheck(cudaEventRecord(joins_[k], s), "graph replay: pre");
      cudaCheck(cudaStreamWaitEvent(gate_, joins_[k], 0), "graph replay: pre");
    }
  }
  t_ctx.recorded.clear();
  t_ctx.gate = gate_;
  t_ctx.gateDevice = originDevice_;
  cudaStream_t origin = workers_[0].compute;
  t_ctx.origin = origin;
  t_ctx.last = "begin";
  cudaCheck(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed), "graph replay: begin capture");
  g_ctx = &t_ctx;
  // Every stream of every local worker joins the capture from the start, so
  // no work of the replay runs outside the graph: eager work issued during
  // the capture (e.g. pulls waiting on a peer's flags) would run before the
  // graph that it is hoisted into, and two SPMD ranks' graphs could then
  // wait on each other's eager halves.
  try {
    cudaCheck(cudaEventRecord(fork_, origin), "graph replay: fork");
    for (const WorkerStreams& w : workers_) {
      DeviceGuard wd(w.device);
      for (std::size_t i = 0; i <= w.side.size(); ++i) {
        cudaStream_t s = i == 0 ? w.compute : w.side[i - 1];
        if (s != origin) cudaCheck(cudaStreamWaitEvent(s, fork_, 0), "graph replay: fork");
      }
    }
  } catch (...) {
    abort();
    throw;
  }
}

void Graph::abort() noexcept {
  if (!g_ctx) return;
  g_ctx = nullptr;
  DeviceGuard g(originDevice_);
  // Join what can be joined so the origin's capture ends cleanly.
  std::size_t k = 0;
  for (const WorkerStreams& w : workers_) {
    DeviceGuard wd(w.device);
    for (std::size_t i = 0; i <= w.side.size(); ++i, ++k) {
      cudaStream_t s = i == 0 ? w.compute : w.side[i - 1];
      if (s == workers_[0].compute || !capturing(s)) continue;
      if (cudaEventRecord(joins_[k], s) == cudaSuccess) cudaStreamWaitEvent(workers_[0].compute, joins_[k], 0);
    }
  }
  cudaGraph_t graph = nullptr;
  cudaStreamEndCapture(workers_[0].compute, &graph);
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
}

void Graph::endAndLaunch() {
  if (g_ctx != &t_ctx) throw Error("graph replay: no open capture");
  DeviceGuard g(originDevice_);
  cudaStream_t origin = workers_[0].compute;
  std::size_t k = 0;
  try {
    for (const WorkerStreams& w : workers_) {
      DeviceGuard wd(w.device);
      for (std::size_t i = 0; i <= w.side.size(); ++i, ++k) {
        cudaStream_t s = i == 0 ? w.compute : w.side[i - 1];
        if (s == origin || !capturing(s)) continue;
        cudaCheck(cudaEventRecord(joins_[k], s), "graph replay: join");
        cudaCheck(cudaStreamWaitEvent(origin, joins_[k], 0), "graph replay: join");
      }
    }
  } catch (...) {
    abort();
    throw;
  }
  g_ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaCheck(cudaStreamEndCapture(origin, &graph), "graph replay: end capture");
  std::size_t nn = 0;
  cudaGraphGetNodes(graph, nullptr, &nn);
  nodes = nn;
  if (exec_) {
    cudaGraphExecUpdateResultInfo info{};
    if (cudaGraphExecUpdate(exec_, graph, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(exec_);
      exec_ = nullptr;
    }
  }
  if (!exec_) {
    const cudaError_t e = cudaGraphInstantiate(&exec_, graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      exec_ = nullptr;
      throw Error(std::string("graph replay: instantiate: ") + cudaGetErrorString(e));
    }
    ++instantiations;
  }
  cudaGraphDestroy(graph);
  // Dependencies on work issued before / beside the capture, then the graph.
  cudaCheck(cudaEventRecord(gateEv_, gate_), "graph replay: gate");
  cudaCheck(cudaStreamWaitEvent(origin, gateEv_, 0), "graph replay: gate");
  cudaCheck(cudaGraphLaunch(exec_, origin), "graph replay: launch");
  ++launches;
  cudaCheck(cudaEventRecord(done_, origin), "graph replay: done");
  // Everything issued after the replay, on any stream, follows the graph;
  // the events the planner recorded inside it now mark its end.
  for (const WorkerStreams& w : workers_) {
    DeviceGuard wd(w.device);
    for (std::size_t i = 0; i <= w.side.size(); ++i) {
      cudaStream_t s = i == 0 ? w.compute : w.side[i - 1];
      if (s != origin) cudaCheck(cudaStreamWaitEvent(s, done_, 0), "graph replay: after");
    }
  }
  for (const auto& kv : t_ctx.recorded) {
    cudaStream_t s = nullptr;
    for (const WorkerStreams& w : workers_)
      if (w.device == kv.second) {
        s = w.compute;
        break;
      }
    if (!s) throw Error("graph replay: event recorded on a device with no local worker");
    DeviceGuard wd(kv.second);
    cudaCheck(cudaEventRecord(kv.first, s), "graph replay: re-record");
  }
  t_ctx.recorded.clear();
}

}  // namespace capture
}  // namespace gridmath
