// SPDX-License-Identifier: Apache-2.0
// Driver for the reference's UNMODIFIED Trainer (proj/src/dnn.cpp, compiled
// from /root/reference by tests/cpp/Makefile against <repo>/include's drop-in
// headers and linked with libgridmath_b200.so -- no reference library
// involved). Exercises the Trainer paths that stay on the B200 GEMM path:
// construction (setData + replicateAsync of every layer), predict (gemm ->
// biasAdd -> relu -> gemm -> biasAdd, getData), predictMixedHalf
// (castPrecision to Half, mixed Half x Single GEMMs), gatherParameters; and
// trainStep, whose softmax/loss ops are outside the path and must fail with
// the drop-in's error, not crash.
//
//   dropin_dnn OUT.bin
// writes: u32 n, u32 dim, u32 classes, f32 batch[n*dim], then for each
// parameter (W0, b0, W1, b1) u64 count + f64 values, then u32 predict[n],
// u32 predictMixedHalf[n].
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "gridmath/dnn.hpp"

using namespace gridmath;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  SessionOptions opts;
  opts.workers = 4;
  Session s(opts);
  const std::vector<std::uint32_t> dims = {96, 64, 10};
  dnn::TrainOptions to;
  to.seed = 3;
  dnn::Trainer trainer(s, dims, to);
  const dnn::Dataset ds = dnn::makeBlobs(5, 256, dims[0], dims.back(), 3.0, 0.5);
  const std::vector<std::uint32_t> pred = trainer.predict(ds.features);
  const std::vector<std::uint32_t> half = trainer.predictMixedHalf(ds.features);
  const auto params = trainer.gatherParameters();
  std::string err;
  try {
    trainer.trainStep(ds.features, ds.labels);
  } catch (const Error& e) {
    err = e.what();
  }
  std::ofstream out(argv[1], std::ios::binary | std::ios::trunc);
  auto u32 = [&](std::uint32_t v) { out.write(reinterpret_cast<const char*>(&v), 4); };
  u32(static_cast<std::uint32_t>(ds.count()));
  u32(dims[0]);
  u32(dims.back());
  out.write(reinterpret_cast<const char*>(ds.features.data()), static_cast<std::streamsize>(ds.features.size() * 4));
  for (const auto& p : params) {
    const std::uint64_t n = p.size();
    out.write(reinterpret_cast<const char*>(&n), 8);
    out.write(reinterpret_cast<const char*>(p.data()), static_cast<std::streamsize>(n * 8));
  }
  for (std::uint32_t v : pred) u32(v);
  for (std::uint32_t v : half) u32(v);
  out.close();
  std::printf("trainStep: %s\n", err.c_str());
  std::printf("parameters %zu\n", trainer.parameterCount());
  const bool ok = err.find("not supported on the B200 GEMM path") != std::string::npos;
  std::printf(ok ? "DROPIN_DNN OK\n" : "DROPIN_DNN FAILED\n");
  return ok ? 0 : 1;
}
