// Programmatic dependent launch (PDL) for the forward's kernel chain: every
// layer kernel is launched with programmatic stream serialization, triggers
// its dependents as soon as it starts and waits for its predecessor's grid
// (griddepcontrol.wait) only after its own prologue (barrier init, TMEM
// allocation, descriptor prefetch, bias/weight loads — nothing a previous
// layer writes). Inside a captured CUDA graph the edges become programmatic,
// so a layer's launch and prologue overlap the previous layer's tail.
// DS_PDL=0 launches plainly (A/B switch); griddepcontrol.wait is a no-op then.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace ds {

// SM budget of the launches being enqueued on this host thread (0: the whole
// device). Persistent kernels size their grids by it; the runtime sets it
// while it enqueues (or captures) a forward for a green-context SM partition
// (MT instances, engine.cu), so a partition's grid is not 148 SMs deep.
inline int& launch_sm_budget() {
  static thread_local int budget = 0;
  return budget;
}

inline int budgeted_sms(int device_sms) {
  const int b = launch_sm_budget();
  return (b > 0 && b < device_sms) ? b : device_sms;
}

// Live per-kernel timing inside the real (graph-launched, PDL-chained)
// forward: the runtime points each launch at a slot {sum, count}; CTA 0 of
// the kernel adds the %globaltimer value at which it passed
// griddepcontrol.wait (= when the previous kernel's grid completed) with
// fire-and-forget reductions (no latency on the kernel's critical path).
// Kernel k's in-situ duration over n forwards is (sum[k+1] - sum[k]) / n;
// the forward's last kernel also marks its end into the slot after it.
inline unsigned long long*& launch_span() {
  static thread_local unsigned long long* slot = nullptr;
  return slot;
}

inline bool pdl_enabled() {
  const bool on = [] {
    const char* e = std::getenv("DS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// PDL launch of a kernel in clusters of `cluster` CTAs along x.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t stream, int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void span_mark(unsigned long long* slot) {
  if (slot != nullptr && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicAdd(slot, t);
    atomicAdd(slot + 1, 1ull);
  }
}

__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace ds
