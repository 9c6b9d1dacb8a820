// Micro-benchmark of a persistent tcgen05 kernel's prologue on sm_100a:
// warp launch skew of an 18-warp CTA, mbarrier.init cost, tcgen05.alloc
// latency, param (constant bank) miss latency. Dev tool (tools/).
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

struct BigArgs { unsigned long long* out; int pad[400]; };

__device__ __forceinline__ unsigned long long clk() { return clock64(); }

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_prologue(const __grid_constant__ BigArgs a) {
  const unsigned long long t0 = clk();
  __shared__ __align__(8) unsigned long long bars[64];
  __shared__ unsigned tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* o = a.out + blockIdx.x * 64;
  if (lane == 0) o[warp] = t0;  // first instruction time per warp (slots 0..WARPS-1)
  if (warp == 0 && lane == 0) {
    // param misses: 4 dependent reads of far-apart param words
    unsigned long long t1 = clk();
    int x = a.pad[0];
    x = a.pad[(x & 1) + 100];
    x = a.pad[(x & 1) + 200];
    x = a.pad[(x & 1) + 300];
    unsigned long long t2 = clk();
    o[40] = t2 - t1 + (x == 12345 ? 1 : 0);
    // 48 mbarrier inits by one thread
    t1 = clk();
    for (int i = 0; i < 48; ++i) {
      unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(&bars[i]));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    t2 = clk();
    o[41] = t2 - t1;
  }
  if (warp == 1) {
    unsigned long long t1 = clk();
    unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(&tslot));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(addr));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    unsigned long long t2 = clk();
    if (lane == 0) o[42] = t2 - t1;
  }
  __syncthreads();
  if (threadIdx.x == 0) o[43] = clk() - t0;
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
  }
}

int main() {
  const int grid = 148;
  BigArgs a{};
  cudaMalloc(&a.out, grid * 64 * 8);
  for (int i = 0; i < 400; ++i) a.pad[i] = i;
  std::vector<unsigned long long> h(grid * 64);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(a.out, 0, grid * 64 * 8);
    k_prologue<18><<<grid, 18 * 32>>>(a);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h.data(), a.out, h.size() * 8, cudaMemcpyDeviceToHost);
  auto med = [&](auto f) { std::vector<long long> v; for (int c = 0; c < grid; ++c) v.push_back(f(c)); std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
  printf("18-warp CTA, cycles (median over %d CTAs):\n", grid);
  for (int w = 1; w < 18; w += 4) printf("  warp %2d first instr - warp 0: %lld\n", w, med([&](int c) { return (long long)(h[c*64+w] - h[c*64]); }));
  printf("  warp 17 first instr - warp 0: %lld\n", med([&](int c) { return (long long)(h[c*64+17] - h[c*64]); }));
  printf("  4 dependent param reads: %lld\n", med([&](int c) { return (long long)h[c*64+40]; }));
  printf("  48 mbarrier.init + fence: %lld\n", med([&](int c) { return (long long)h[c*64+41]; }));
  printf("  tcgen05.alloc 512 + relinquish: %lld\n", med([&](int c) { return (long long)h[c*64+42]; }));
  printf("  entry -> after __syncthreads: %lld\n", med([&](int c) { return (long long)h[c*64+43]; }));
  return 0;
}
