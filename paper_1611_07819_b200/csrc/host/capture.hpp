// SPDX-License-Identifier: Apache-2.0
// CUDA-graph capture of a replayed pipeline (reference
// Session::replay, session.cpp:385-409, which cuts a step to one control
// message: here a step becomes one graph launch per process).
//
// Replay runs the host planner as usual -- versions, replica states, panel
// cache, flag values are exactly the eager ones -- while every worker stream
// the ops touch is in capture mode, so the device work lands in one graph
// that is launched once (after an in-place update of the previous replay's
// executable when the topology is unchanged). Every event record / stream
// wait of the runtime goes through record() / wait() below:
//   * an event recorded on a capturing stream is remembered; after the graph
//     launch it is recorded again behind the graph, so the runtime's per-
//     matrix events (last write, readers, replica / panel readiness, arena
//     releases) stay valid for the uncaptured work that follows;
//   * a capturing stream waiting on an event recorded outside the capture
//     (work issued before the replay) would cross the capture boundary: the
//     wait goes to a gate stream instead, and the graph launch waits for the
//     gate, so the dependency holds (hoisted to the start of the graph);
//   * timing events (per-GEMM windows, last-op timers) become event-record
//     nodes inside the graph, so their elapsed times stay the kernels' own.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <unordered_map>
#include <vector>

namespace gridmath {
namespace capture {

// Drop-in replacements for cudaEventRecord / cudaStreamWaitEvent.
cudaError_t record(cudaEvent_t e, cudaStream_t s);
cudaError_t recordTiming(cudaEvent_t e, cudaStream_t s);
cudaError_t wait(cudaStream_t s, cudaEvent_t e, unsigned flags = 0);
bool active();
// Throws (naming the previous checkpoint) if the open capture was
// invalidated by a call since then; no-op outside a capture.
void checkpoint(const char* where);

// One capture of one replay. `origin` is the first local worker's compute
// stream; `workers` lists (device, compute stream, side streams) of every
// local worker (their compute streams are forked from origin at begin() and
// every stream still capturing is joined back at end()).
struct WorkerStreams {
  int device = 0;
  cudaStream_t compute = nullptr;
  std::vector<cudaStream_t> side;
};

class Graph {
 public:
  Graph() = default;
  ~Graph();
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;

  // Starts capturing on origin (relaxed mode: the planner's host-side
  // queries stay legal). Throws on failure.
  void begin(const std::vector<WorkerStreams>& workers);
  // Ends the capture, updates or instantiates the executable, launches it,
  // re-records the captured events behind it. Throws on failure.
  void endAndLaunch();
  // Error path: ends the capture and drops the partial graph.
  void abort() noexcept;

  std::uint64_t launches = 0, instantiations = 0;
  std::size_t nodes = 0;

 private:
  std::vector<WorkerStreams> workers_;
  cudaGraphExec_t exec_ = nullptr;
  cudaStream_t gate_ = nullptr;
  cudaEvent_t gateEv_ = nullptr, fork_ = nullptr, done_ = nullptr;
  std::vector<cudaEvent_t> joins_;
  int originDevice_ = 0;
};

}  // namespace capture
}  // namespace gridmath
