// Board energy counter through NVML (measured power in
// place of the reference's PowerModel, perf_model.cpp:88-101). libnvidia-ml is
// opened at run time (no link dependency); the NVML device is matched to the
// CUDA ordinal by PCI bus id.
#include "nvml_energy.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <map>
#include <mutex>

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

bool board_energy_mj(int device, double* mj, double* wall_ms, double* power_w) {
  nvmlDevice d = handle_for(device);
  unsigned long long e = 0;
  unsigned mw = 0;
  if (!d || nvml().energy(d, &e) != 0 || nvml().power(d, &mw) != 0) return false;
  *mj = static_cast<double>(e);
  *power_w = static_cast<double>(mw) / 1000.0;
  *wall_ms = std::chrono::duration<double, std::milli>(
                 std::chrono::steady_clock::now().time_since_epoch())
                 .count();
  return true;
}

}  // namespace ds
