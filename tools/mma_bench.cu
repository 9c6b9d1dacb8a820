// Micro-benchmark: tcgen05.mma issue/throughput on one SM (bring-up tool).
// Issues `iters` MMAs (M=128, N, K=16, bf16 -> fp32 TMEM) back to back on
// smem operands (contents irrelevant), waits for completion via commit +
// mbarrier, prints cycles per MMA. Usage: mma_bench [N] [iters] [desc_kind]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2308_13803_b200/csrc/kernels/sm100_ptx.cuh"

using namespace ds;

__global__ void bench(int N, int iters, int kind, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_barrier_init(); }
    __syncwarp();
    ptx::tmem_alloc(slot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::umma_idesc_bf16_f32(128, N);
    const uint32_t a = ptx::smem_u32(smem), b = ptx::smem_u32(smem + 32 * 1024);
    uint64_t da = ptx::umma_desc_sw128_kmajor(a), db = ptx::umma_desc_sw128_kmajor(b);
    if (kind == 1) da = ptx::umma_desc_sw32_kmajor(a);
    if (kind == 2) da = ptx::umma_desc_sw128_kmajor_sbo(a + 3 * 128, 1280);  // window of a 10-px-wide box
    if (kind == 3) da = ptx::umma_desc_sw128_kmajor_sbo(a, 1280);            // aligned start, SBO 1280
    if (kind == 4) da = ptx::umma_desc_sw128_kmajor_sbo(a, 1024);            // dense via the sbo form
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      ptx::umma_bf16(tmem, da + 2 * (i & 3), db + 2 * (i & 3), idesc, i != 0);
    const unsigned long long t1 = clock64();
    ptx::umma_commit(bar);
    ptx::mbar_wait(bar, 0);
    const unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

int main(int argc, char** argv) {
  int N = argc > 1 ? atoi(argv[1]) : 64, iters = argc > 2 ? atoi(argv[2]) : 1024,
      kind = argc > 3 ? atoi(argv[3]) : 0;
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 3; ++rep) bench<<<1, 128, 100 * 1024>>>(N, iters, kind, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%d iters=%d kind=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", N, iters, kind,
         double(h[0]) / iters, double(h[1]) / iters, cudaGetErrorString(e));
  return 0;
}
