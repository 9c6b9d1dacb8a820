// ds::Seam over the B200 Backend: the control plane's view of the device.
#pragma once

#include <memory>

#include "../../../include/dnnscaler_b200/control.hpp"
#include "engine.hpp"

namespace ds {

class DeviceSeam : public Seam {
 public:
  explicit DeviceSeam(Backend& backend) : b_(backend) {}
  explicit DeviceSeam(std::unique_ptr<Backend> owned) : owned_(std::move(owned)), b_(*owned_) {}
  double run_batch(int bs) override { return b_.run_batch(bs); }
  double run_mt_request() override { return b_.run_mt_request(); }
  double apply_instance_change(int delta) override { return b_.apply_instance_change(delta); }
  double set_mtl(int target) override { return b_.set_mtl(target); }
  int mtl() const override { return b_.mtl(); }
  double clock_ms() const override { return b_.clock_ms(); }
  Config config() const override { return Config{b_.config().abs_max_bs, b_.config().max_mtl}; }
  void run_batches(int bs, int count, double* out) override { b_.run_batches(bs, count, out); }
  void run_mt_requests(int count, double* out) override { b_.run_mt_requests(count, out); }

 private:
  std::unique_ptr<Backend> owned_;
  Backend& b_;
};

}  // namespace ds
