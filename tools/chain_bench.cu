// Per-kernel boundary cost of a dependent chain of small kernels on sm_100a:
// N kernels, each reading the previous kernel's output, captured in a CUDA
// graph with programmatic dependent launch (PDL) edges or plain edges.
// Dev tool (tools/): sizes the fixed cost a small-batch forward pays per layer.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void step(const float4* __restrict__ in, float4* __restrict__ out, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float4 v = in[i];
    v.x += 1.f;
    out[i] = v;
  }
}

int main() {
  const int kernels = 31;
  float4* buf[2];
  const int n_max = 1 << 20;
  cudaMalloc(&buf[0], n_max * 16);
  cudaMalloc(&buf[1], n_max * 16);
  cudaMemset(buf[0], 0, n_max * 16);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int ctas_list[] = {1, 32, 148, 296, 592};
  const int threads_list[] = {128, 256};
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int threads : threads_list)
      for (int ctas : ctas_list)
        for (int n : {4096, 65536}) {
          cudaGraph_t g;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
          for (int k = 0; k < kernels; ++k) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctas);
            cfg.blockDim = dim3(threads);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl;
            cudaLaunchKernelEx(&cfg, step, (const float4*)buf[k & 1], buf[(k + 1) & 1], n, pdl);
          }
          cudaStreamEndCapture(s, &g);
          cudaGraphExec_t ge;
          cudaGraphInstantiate(&ge, g, 0);
          for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0, s);
          const int reps = 200;
          for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, s);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          printf("pdl %d threads %3d ctas %3d n %6d: %.3f us per kernel (%.1f us per graph)\n", pdl, threads,
                 ctas, n, ms * 1e3 / reps / kernels, ms * 1e3 / reps);
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(g);
        }
  return 0;
}
