#pragma once

namespace ds {

// Cumulative board energy (mJ, NVML total energy counter) of CUDA device
// `device`, a monotonic wall clock (ms) and the board's current power draw
// (W, nvmlDeviceGetPowerUsage), as of the latest sample of a background
// sampler thread (every 5 ms), so the call never blocks the serving loop;
// false when NVML is unavailable. The energy counter advances in coarse
// steps, so per-period power uses the power reading and job averages use the
// counter (over the samples' own timestamps).
bool board_energy_mj(int device, double* mj, double* wall_ms, double* power_w);

}  // namespace ds
