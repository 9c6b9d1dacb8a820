// Drop-in replacement for the reference's device seam header
// (reference proj/core/include/dnnscaler/gpu_sim.hpp:13-50).
//
// Put include/dnnscaler_b200/drop_in on the include path BEFORE the
// reference's core/include, build include/dnnscaler_b200/drop_in/gpu_sim_b200.cpp
// instead of core/src/gpu_sim.cpp, and link libdnnscaler_b200.so: the
// reference's profiler.cpp, scaler.cpp and harness.cpp then serve on a B200
// unchanged. Same public method set, semantics and
// exception messages; the analytic models passed to the constructor are kept
// for the accessors (the harness reads them for power/ramp accounting) but
// latencies now come from the device.
//
// Which network a GpuSim serves is bound per thread before construction
// (dnnscaler_b200::bind_model), or by the DNNSCALER_B200_MODEL environment
// variable; the device by dnnscaler_b200::bind_device / DNNSCALER_B200_DEVICE.
#pragma once

#include <cstdint>
#include <string>

#include "dnnscaler/perf_model.hpp"
#include "dnnscaler/random.hpp"

struct ds_backend;

namespace dnnscaler_b200 {
void bind_model(const std::string& model_id);
void bind_device(int device);
}  // namespace dnnscaler_b200

namespace dnnscaler {

class GpuSim {
 public:
  struct Config {
    int abs_max_bs = 128;
    int max_mtl = 10;
  };

  GpuSim(BatchingModel bm, MtModel mm, PowerModel pm, Config config, uint64_t seed);
  ~GpuSim();
  GpuSim(GpuSim&& other) noexcept;
  GpuSim& operator=(GpuSim&& other) noexcept;
  GpuSim(const GpuSim&) = delete;
  GpuSim& operator=(const GpuSim&) = delete;

  double run_batch(int bs);
  double run_mt_request();
  double apply_instance_change(int delta);
  double set_mtl(int target);

  int mtl() const { return mtl_; }
  double clock_ms() const { return clock_ms_; }
  const BatchingModel& batching_model() const { return bm_; }
  const MtModel& mt_model() const { return mm_; }
  const PowerModel& power_model() const { return pm_; }
  const Config& config() const { return config_; }

 private:
  BatchingModel bm_;
  MtModel mm_;
  PowerModel pm_;
  Config config_;
  ds_backend* dev_ = nullptr;
  double clock_ms_ = 0.0;
  int mtl_ = 1;
};

}  // namespace dnnscaler
