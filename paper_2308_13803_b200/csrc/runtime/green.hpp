// SM partitions for multi-tenancy through CUDA green contexts (SURVEY §8(a)
// K8: "N replicas ... optional green-context SM split"; the reference models
// co-location only analytically, gpu_sim.cpp:20-24 / perf_model.cpp:75-78).
//
// At MT level k the device's SMs are split into k equal groups
// (cuDevSmResourceSplitByCount; the driver keeps TPC pairs together, so the
// CTA-pair conv kernels still get co-scheduled clusters) and every group gets
// a green context and one non-blocking stream. MT instance i at level k
// launches its forward on lane (k, i mod groups) with the persistent kernels'
// grids sized to the group (pdl.cuh launch_sm_budget). Green contexts share
// the primary context's memory, so instances keep their weights/workspace.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <vector>

namespace ds {

struct GreenLane {
  CUgreenCtx ctx = nullptr;
  cudaStream_t stream = nullptr;
  int sms = 0;
};

class GreenPartitions {
 public:
  explicit GreenPartitions(int device);
  ~GreenPartitions();
  GreenPartitions(const GreenPartitions&) = delete;
  GreenPartitions& operator=(const GreenPartitions&) = delete;

  // The lanes of level k (created on first use): as many equal groups as the
  // split grants (<= k), each with its own green context and stream.
  const std::vector<GreenLane>& level(int k);
  int device_sms() const { return device_sms_; }

 private:
  int device_;
  int device_sms_ = 0;
  std::map<int, std::vector<GreenLane>> levels_;
};

// True when this driver exposes the green-context entry points.
bool green_contexts_supported();

}  // namespace ds
