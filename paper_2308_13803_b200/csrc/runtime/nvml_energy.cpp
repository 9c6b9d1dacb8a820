// Board energy counter through NVML (measured power in
// place of the reference's PowerModel, perf_model.cpp:88-101). libnvidia-ml is
// opened at run time (no link dependency); the NVML device is matched to the
// CUDA ordinal by PCI bus id.
#include "nvml_energy.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

namespace ds {

namespace {

using nvmlReturn = int;
using nvmlDevice = void*;

struct Nvml {
  nvmlReturn (*init)() = nullptr;
  nvmlReturn (*by_pci)(const char*, nvmlDevice*) = nullptr;
  nvmlReturn (*energy)(nvmlDevice, unsigned long long*) = nullptr;
  nvmlReturn (*power)(nvmlDevice, unsigned*) = nullptr;
  bool ok = false;
};

const Nvml& nvml() {
  static Nvml n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    n.init = reinterpret_cast<nvmlReturn (*)()>(dlsym(h, "nvmlInit_v2"));
    n.by_pci = reinterpret_cast<nvmlReturn (*)(const char*, nvmlDevice*)>(
        dlsym(h, "nvmlDeviceGetHandleByPciBusId_v2"));
    n.energy = reinterpret_cast<nvmlReturn (*)(nvmlDevice, unsigned long long*)>(
        dlsym(h, "nvmlDeviceGetTotalEnergyConsumption"));
    n.power = reinterpret_cast<nvmlReturn (*)(nvmlDevice, unsigned*)>(
        dlsym(h, "nvmlDeviceGetPowerUsage"));
    n.ok = n.init && n.by_pci && n.energy && n.power && n.init() == 0;
  });
  return n;
}

nvmlDevice handle_for(int device) {
  static std::mutex mu;
  static std::map<int, nvmlDevice> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  nvmlDevice d = nullptr;
  char bus[32] = {0};
  if (nvml().ok && cudaDeviceGetPCIBusId(bus, sizeof(bus), device) == cudaSuccess &&
      nvml().by_pci(bus, &d) != 0)
    d = nullptr;
  cache[device] = d;
  return d;
}

}  // namespace

namespace {

// One sampler thread per device reads the counters every kPeriodMs into a
// seqlock-free snapshot (three atomics written in order, a sequence number
// around them): NVML queries take milliseconds, and reading them inline at
// every control period stalled the serving loop (the in-flight requests
// drained while the host waited on NVML).
constexpr int kPeriodMs = 5;

struct Sampler {
  std::atomic<uint64_t> seq{0};
  std::atomic<double> mj{0.0}, wall_ms{0.0}, watts{0.0};
  std::atomic<bool> ok{false};
  std::thread th;
  std::atomic<bool> stop{false};
  ~Sampler() {
    stop = true;
    if (th.joinable()) th.join();
  }
};

bool read_now(nvmlDevice d, double* mj, double* wall_ms, double* power_w) {
  unsigned long long e = 0;
  unsigned mw = 0;
  if (nvml().energy(d, &e) != 0 || nvml().power(d, &mw) != 0) return false;
  *mj = static_cast<double>(e);
  *power_w = static_cast<double>(mw) / 1000.0;
  *wall_ms = std::chrono::duration<double, std::milli>(
                 std::chrono::steady_clock::now().time_since_epoch())
                 .count();
  return true;
}

Sampler* sampler_for(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Sampler>> samplers;
  std::lock_guard<std::mutex> lock(mu);
  auto it = samplers.find(device);
  if (it != samplers.end()) return it->second.get();
  auto s = std::make_unique<Sampler>();
  nvmlDevice d = handle_for(device);
  double mj = 0, w = 0, p = 0;
  if (d && read_now(d, &mj, &w, &p)) {
    s->mj = mj;
    s->wall_ms = w;
    s->watts = p;
    s->ok = true;
    Sampler* raw = s.get();
    s->th = std::thread([raw, d] {
      while (!raw->stop) {
        std::this_thread::sleep_for(std::chrono::milliseconds(kPeriodMs));
        double e1 = 0, w1 = 0, p1 = 0;
        if (!read_now(d, &e1, &w1, &p1)) continue;
        raw->seq.fetch_add(1);  // odd: writing
        raw->mj = e1;
        raw->wall_ms = w1;
        raw->watts = p1;
        raw->seq.fetch_add(1);  // even: stable
      }
    });
  }
  return samplers.emplace(device, std::move(s)).first->second.get();
}

}  // namespace

bool board_energy_mj(int device, double* mj, double* wall_ms, double* power_w) {
  Sampler* s = sampler_for(device);
  if (!s->ok) return false;
  for (;;) {  // a consistent snapshot of the latest sample
    const uint64_t a = s->seq.load();
    if (a & 1) continue;
    *mj = s->mj;
    *wall_ms = s->wall_ms;
    *power_w = s->watts;
    if (s->seq.load() == a) return true;
  }
}

}  // namespace ds
