// ds::Seam over the B200 Backend: the control plane's view of the device.
#pragma once

#include <memory>

#include "../../../include/dnnscaler_b200/control.hpp"
#include <cstdlib>

#include "engine.hpp"
#include "nvml_energy.hpp"

namespace ds {

// A job's view of a (possibly shared) Backend. The seam keeps its own
// virtual clock, starting at 0 like a fresh reference GpuSim, advanced with
// the reference's arithmetic from the measured values (gpu_sim.cpp:16, 22,
// 35): a job's trajectory is then a pure function of its latency tape, even
// when the backend served other work before.
class DeviceSeam : public Seam {
 public:
  explicit DeviceSeam(Backend& backend) : b_(backend) {}
  explicit DeviceSeam(std::unique_ptr<Backend> owned) : owned_(std::move(owned)), b_(*owned_) {}

  double run_batch(int bs) override {
    const double lat = b_.run_batch(bs);
    clock_ms_ += lat;
    return lat;
  }
  double run_mt_request() override {
    const int k = b_.mtl();
    const double lat = b_.run_mt_request();
    clock_ms_ += lat / static_cast<double>(k);
    return lat;
  }
  double apply_instance_change(int delta) override {
    const double d = b_.apply_instance_change(delta);
    clock_ms_ += d;
    return d;
  }
  int mtl() const override { return b_.mtl(); }
  bool energy_reading(double* mj, double* wall_ms, double* power_w) override {
    if (const char* e = std::getenv("DS_MODEL_POWER"))  // A/B: keep the PowerModel
      if (e[0] == '1') return false;
    return board_energy_mj(b_.device(), mj, wall_ms, power_w);
  }
  double clock_ms() const override { return clock_ms_; }
  Config config() const override { return Config{b_.config().abs_max_bs, b_.config().max_mtl}; }
  void run_batches(int bs, int count, double* out) override {
    b_.run_batches(bs, count, out);
    for (int i = 0; i < count; ++i) clock_ms_ += out[i];
  }
  void run_mt_requests(int count, double* out) override {
    const int k = b_.mtl();
    b_.run_mt_requests(count, out);
    for (int i = 0; i < count; ++i) clock_ms_ += out[i] / static_cast<double>(k);
  }

 private:
  std::unique_ptr<Backend> owned_;
  Backend& b_;
  double clock_ms_ = 0.0;
};

}  // namespace ds
