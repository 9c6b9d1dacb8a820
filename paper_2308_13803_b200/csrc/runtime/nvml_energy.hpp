#pragma once

namespace ds {

// Cumulative board energy (mJ, NVML total energy counter) of CUDA device
// `device`, a monotonic wall clock (ms) and the board's current power draw
// (W, nvmlDeviceGetPowerUsage); false when NVML is unavailable. The energy
// counter advances in coarse steps (tens of ms), so per-period power uses
// the power reading and job averages use the counter.
bool board_energy_mj(int device, double* mj, double* wall_ms, double* power_w);

}  // namespace ds
