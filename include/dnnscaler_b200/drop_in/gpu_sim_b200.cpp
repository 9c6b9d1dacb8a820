// Implementation of the drop-in dnnscaler::GpuSim over the B200 C ABI
// (include/dnnscaler_b200.h). Compiled by the consumer in place of the
// reference's core/src/gpu_sim.cpp; links against libdnnscaler_b200.so.
#include "dnnscaler/gpu_sim.hpp"

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../dnnscaler_b200.h"

namespace dnnscaler_b200 {
namespace {
thread_local std::string g_model;
thread_local int g_device = -1;
}  // namespace

void bind_model(const std::string& model_id) { g_model = model_id; }
void bind_device(int device) { g_device = device; }

}  // namespace dnnscaler_b200

namespace dnnscaler {

namespace {

// Reference exception types: DS_EINVAL -> std::invalid_argument (same
// message), anything else -> std::runtime_error.
void raise_on(ds_status s) {
  if (s == DS_OK) return;
  const std::string msg = ds_last_error();
  if (s == DS_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

std::string bound_model() {
  if (!dnnscaler_b200::g_model.empty()) return dnnscaler_b200::g_model;
  const char* env = std::getenv("DNNSCALER_B200_MODEL");
  return env ? env : "mobilenet_v1";
}

int bound_device() {
  if (dnnscaler_b200::g_device >= 0) return dnnscaler_b200::g_device;
  const char* env = std::getenv("DNNSCALER_B200_DEVICE");
  return env ? std::atoi(env) : 0;
}

}  // namespace

GpuSim::GpuSim(BatchingModel bm, MtModel mm, PowerModel pm, Config config, uint64_t seed)
    : bm_(bm), mm_(mm), pm_(pm), config_(config) {
  raise_on(ds_backend_create(bound_model().c_str(), ds_config{config.abs_max_bs, config.max_mtl},
                             seed, bound_device(), &dev_));
}

GpuSim::~GpuSim() { ds_backend_destroy(dev_); }

GpuSim::GpuSim(GpuSim&& o) noexcept
    : bm_(o.bm_), mm_(o.mm_), pm_(o.pm_), config_(o.config_), dev_(std::exchange(o.dev_, nullptr)),
      clock_ms_(o.clock_ms_), mtl_(o.mtl_) {}

GpuSim& GpuSim::operator=(GpuSim&& o) noexcept {
  if (this != &o) {
    ds_backend_destroy(dev_);
    bm_ = o.bm_;
    mm_ = o.mm_;
    pm_ = o.pm_;
    config_ = o.config_;
    dev_ = std::exchange(o.dev_, nullptr);
    clock_ms_ = o.clock_ms_;
    mtl_ = o.mtl_;
  }
  return *this;
}

// Clock arithmetic as reference gpu_sim.cpp:16, 22, 35.
double GpuSim::run_batch(int bs) {
  double lat = 0.0;
  raise_on(ds_run_batch(dev_, bs, &lat));
  clock_ms_ += lat;
  return lat;
}

double GpuSim::run_mt_request() {
  double lat = 0.0;
  raise_on(ds_run_mt_request(dev_, &lat));
  clock_ms_ += lat / static_cast<double>(mtl_);
  return lat;
}

double GpuSim::apply_instance_change(int delta) {
  double delay = 0.0;
  raise_on(ds_apply_instance_change(dev_, delta, &delay));
  mtl_ = ds_mtl(dev_);
  clock_ms_ += delay;
  return delay;
}

double GpuSim::set_mtl(int target) {  // one instance at a time, as gpu_sim.cpp:39-46
  if (target < 1) throw std::invalid_argument("cannot terminate last instance");
  if (target > config_.max_mtl) throw std::invalid_argument("instance limit exceeded");
  double total = 0.0;
  while (mtl_ < target) total += apply_instance_change(1);
  while (mtl_ > target) total += apply_instance_change(-1);
  return total;
}

}  // namespace dnnscaler
