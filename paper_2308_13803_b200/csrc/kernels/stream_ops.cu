// HBM-bound layers of the forward pass. Threads own 8 channels (one 16 B
// vector) of one or more output pixels, so consecutive threads in a warp
// touch consecutive 16 B chunks of the NHWC row: fully coalesced 512 B per
// warp access. Neighbouring taps of the stencils hit L1/L2, so DRAM traffic
// stays close to one read of the input and one write of the output.
#include "stream_ops.cuh"

#include "pdl.cuh"

#include <algorithm>
#include <cstdlib>

namespace ds {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

inline unsigned grid_for(long long work) {
  return static_cast<unsigned>((work + kBlock - 1) / kBlock);
}

// Space-to-depth staging for stride-2 stems (kS2D): S[n][Y][X][16] bf16 with
// channel (a*2 + b)*4 + c = x(2Y + a - pad, 2X + b - pad, c) normalised as
// above (zero outside the image and for c == 3). A stride-2 R x S conv over x
// is then a stride-1 ceil(R/2) x ceil(S/2) conv over S with 16 channels.
__global__ void stage_s2d_kernel(const uint8_t* __restrict__ img, uint4* __restrict__ out, int h,
                                 int w, int hs, int ws, int pad, long long pixels, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  // (32-bit index arithmetic: the launcher keeps pixels below 2^31)
  const int i = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= pixels) return;
  const int t = i / ws;
  const int X = i - t * ws;
  const int n = t / hs;
  const int Y = t - n * hs;
  uint32_t v[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int y = 2 * Y + a - pad, x = 2 * X + b - pad;
      // bf16_rn(centered * (1/63.75)) == bf16_rn((p - 127.5) / 63.75) for every
      // byte (tests/test_oracle.py::test_stem_normalisation_exact); the
      // centred value comes from the bit pattern 0x4A800000 + 2p + 1 = 2^22 +
      // p + 0.5 minus (2^22 + 128), exactly and without the conversion pipe
      float f[3] = {0.f, 0.f, 0.f};
      if (y >= 0 && y < h && x >= 0 && x < w) {
        const uint8_t* src = img + ((static_cast<long long>(n) * h + y) * w + x) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          f[c] = __fmul_rn(__fsub_rn(__uint_as_float(0x4A800001u + 2u * __ldg(src + c)), 4194432.0f),
                           1.0f / 63.75f);
      }
      v[(a * 2 + b) * 2] = pack2(f[0], f[1]);
      v[(a * 2 + b) * 2 + 1] = pack2(f[2], 0.0f);
    }
  out[2 * i] = make_uint4(v[0], v[1], v[2], v[3]);
  out[2 * i + 1] = make_uint4(v[4], v[5], v[6], v[7]);
}


// 3x3 pooling on a 2-D grid: grid.y = output row (image, oy), x = (output
// column, 8-channel group); 32-bit index arithmetic (the column / group split
// through an exact float-reciprocal division). Max pooling compares the
// packed bf16 pairs directly (max is exact in any precision); average pooling
// accumulates with fma.rn.f32.bf16(x, 1.0, acc) == acc + float(x), one
// instruction per element. Per output the taps are visited row outer, column
// inner (padding skipped) and averages divide the fp32 sum by 9 — the
// oracle's order, and the TMA pools' (pool_tma.cu, bit-identical).
__device__ __forceinline__ float add_bf16_lo(uint32_t x, float c) {
  float d;
  asm("{.reg .b16 xl, xh, one;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b16 one, 0x3F80;\n\t"
      "fma.rn.f32.bf16 %0, xl, one, %2;}"
      : "=f"(d)
      : "r"(x), "f"(c));
  return d;
}

__device__ __forceinline__ float add_bf16_hi(uint32_t x, float c) {
  float d;
  asm("{.reg .b16 xl, xh, one;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b16 one, 0x3F80;\n\t"
      "fma.rn.f32.bf16 %0, xh, one, %2;}"
      : "=f"(d)
      : "r"(x), "f"(c));
  return d;
}

__device__ __forceinline__ uint32_t max_bf16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// ROWS output rows per thread (grid.y = image x row group): input rows are
// loaded once and feed every output row whose window covers them; each
// output still sums its taps in row-outer, column-inner order.
template <int STRIDE, bool IS_MAX, int ROWS>
__global__ void pool3x3_rows_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int h, int w,
                                    int cg, int ho, int wo, int pad, int ldo_g, int coff_g, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int ox = __float2int_rz(__int2float_rz(i) * (1.0f / static_cast<float>(cg)));
  if (ox * cg > i) --ox;
  if ((ox + 1) * cg <= i) ++ox;
  if (ox >= wo) return;
  const int g = i - ox * cg;
  const int hq = (ho + ROWS - 1) / ROWS;
  const int n = blockIdx.y / hq;
  const int oy0 = (blockIdx.y - n * hq) * ROWS;
  const int iy0 = oy0 * STRIDE - pad, ix0 = ox * STRIDE - pad;
  constexpr int IN_ROWS = (ROWS - 1) * STRIDE + 3;
  uint4 mx[ROWS];
  float acc[ROWS][8];
#pragma unroll
  for (int o = 0; o < ROWS; ++o) {
    mx[o] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // bf16 -inf pairs
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
  }
#pragma unroll
  for (int ir = 0; ir < IN_ROWS; ++ir) {
    const int iy = iy0 + ir;
    if (iy < 0 || iy >= h) continue;
    const uint4* xrow = x + (static_cast<long long>(n) * h + iy) * w * cg + g;
    uint4 v[3];
    bool ok[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int ix = ix0 + s;
      ok[s] = ix >= 0 && ix < w;
      v[s] = ok[s] ? __ldg(xrow + ix * cg) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int o = 0; o < ROWS; ++o) {
      const int r = ir - o * STRIDE;  // this input row's tap row for output o
      if (r < 0 || r >= 3) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (!ok[s]) continue;
        if constexpr (IS_MAX) {
          mx[o].x = max_bf16x2(mx[o].x, v[s].x);
          mx[o].y = max_bf16x2(mx[o].y, v[s].y);
          mx[o].z = max_bf16x2(mx[o].z, v[s].z);
          mx[o].w = max_bf16x2(mx[o].w, v[s].w);
        } else {
          const uint32_t vw[4] = {v[s].x, v[s].y, v[s].z, v[s].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[o][2 * k] = add_bf16_lo(vw[k], acc[o][2 * k]);
            acc[o][2 * k + 1] = add_bf16_hi(vw[k], acc[o][2 * k + 1]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < ROWS; ++o) {
    if (oy0 + o >= ho) break;
    const long long opix = (static_cast<long long>(n) * ho + oy0 + o) * wo + ox;
    if constexpr (IS_MAX) {
      y[opix * ldo_g + coff_g + g] = mx[o];
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][e] = acc[o][e] / 9.0f;
      y[opix * ldo_g + coff_g + g] = pack8(acc[o]);
    }
  }
}

// Global average pool: one 256-thread block per (image, 256-channel block);
// lane l of every warp owns channels [8l, 8l + 8) of the block (each pixel
// is one coalesced 512 B warp load) and warp w sums pixels w, w + 8, ... in
// order with all its loads in flight; the eight partial sums are added in
// warp order through shared memory (deterministic), then divided by the
// pixel count. One warp per block (the old layout) left ~4 warps per SM at
// batch 128 and ran latency-bound at ~1 TB/s.
constexpr int kGapWarps = 8;

__global__ void __launch_bounds__(kGapWarps * 32) global_avgpool_kernel(
    const uint4* __restrict__ x, uint4* __restrict__ y, int hw, int cg, int blocks_per_image,
    unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  __shared__ float part[kGapWarps][32][9];  // (+1 pad: conflict-free column reads)
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x / blocks_per_image;
  const int g = (blockIdx.x - n * blocks_per_image) * 32 + lane;
  const bool live = g < cg;
  const uint4* p = x + static_cast<long long>(n) * hw * cg + g;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (live) {
    constexpr int U = 8;
    int q = wid;
    for (; q + (U - 1) * kGapWarps < hw; q += U * kGapWarps) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(p + static_cast<long long>(q + u * kGapWarps) * cg);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float xv[8];
        unpack8(v[u], xv);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += xv[e];
      }
    }
    for (; q < hw; q += kGapWarps) {
      float xv[8];
      unpack8(__ldg(p + static_cast<long long>(q) * cg), xv);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += xv[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[wid][lane][e] = acc[e];
  __syncthreads();
  if (wid != 0 || !live) return;
  float sum[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) sum[e] = part[0][lane][e];
  for (int w = 1; w < kGapWarps; ++w)
#pragma unroll
    for (int e = 0; e < 8; ++e) sum[e] += part[w][lane][e];
  const float inv = static_cast<float>(hw);
#pragma unroll
  for (int e = 0; e < 8; ++e) sum[e] = sum[e] / inv;
  y[static_cast<long long>(n) * cg + g] = pack8(sum);
}

__global__ void softmax_kernel(const float* __restrict__ logits, float* __restrict__ probs, int n,
                               int classes, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* l = logits + static_cast<long long>(row) * classes;
  float* p = probs + static_cast<long long>(row) * classes;
  if (classes <= 32 * 32) {  // the row in registers: one independent load per element
    float v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int j = lane + 32 * u;
      v[u] = j < classes ? l[j] : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int u = 0; u < 32; ++u) mx = fmaxf(mx, v[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.0f;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      v[u] = lane + 32 * u < classes ? expf(v[u] - mx) : 0.0f;
      sum += v[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.0f / sum;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int j = lane + 32 * u;
      if (j < classes) p[j] = v[u] * inv;
    }
    span_mark(span ? span + 2 : nullptr);  // the forward's end (last kernel)
    return;
  }
  float mx = -INFINITY;
  for (int j = lane; j < classes; j += 32) mx = fmaxf(mx, l[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.0f;
  for (int j = lane; j < classes; j += 32) sum += expf(l[j] - mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.0f / sum;
  for (int j = lane; j < classes; j += 32) p[j] = expf(l[j] - mx) * inv;
  span_mark(span ? span + 2 : nullptr);
}

}  // namespace

cudaError_t launch_stage_s2d(const uint8_t* img, __nv_bfloat16* out, int n, int h, int w, int hs,
                             int ws, int pad, cudaStream_t stream) {
  const long long pixels = static_cast<long long>(n) * hs * ws;
  if (pixels >= (1LL << 31)) return cudaErrorInvalidValue;
  return launch_pdl(stage_s2d_kernel, dim3(grid_for(pixels)), dim3(kBlock), 0, stream, img,
                    reinterpret_cast<uint4*>(out), h, w, hs, ws, pad, pixels, launch_span());
}

cudaError_t launch_pool3x3(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int h, int w, int c,
                           int stride, int pad, bool is_max, int ldo, int c_off,
                           cudaStream_t stream) {
  // (the fallback of the TMA pools, pool_tma.cu, for layouts they cannot box)
  const int ho = (h + 2 * pad - 3) / stride + 1, wo = (w + 2 * pad - 3) / stride + 1;
  const int cg = c / 8;
  constexpr int kRows = 2;  // output rows per thread
  const int yrows = n * ((ho + kRows - 1) / kRows);
  if (yrows > 65535 || (stride != 1 && stride != 2) || wo * cg >= (1 << 24)) return cudaErrorInvalidValue;
  const int per_row = wo * cg;
  const int bt = std::min(kBlock, (per_row + 31) / 32 * 32);
  const dim3 grid((per_row + bt - 1) / bt, yrows);
  auto go = [&](auto kernel) {
    return launch_pdl(kernel, grid, dim3(bt), 0, stream, reinterpret_cast<const uint4*>(x),
                      reinterpret_cast<uint4*>(y), h, w, cg, ho, wo, pad, ldo / 8, c_off / 8, launch_span());
  };
  if (stride == 1)
    return is_max ? go(pool3x3_rows_kernel<1, true, kRows>) : go(pool3x3_rows_kernel<1, false, kRows>);
  return is_max ? go(pool3x3_rows_kernel<2, true, kRows>) : go(pool3x3_rows_kernel<2, false, kRows>);
}

cudaError_t launch_global_avgpool(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int hw, int c,
                                  cudaStream_t stream) {
  const int cg = c / 8;
  const int bpi = (cg + 31) / 32;  // 256-channel blocks per image
  return launch_pdl(global_avgpool_kernel, dim3(n * bpi), dim3(kGapWarps * 32), 0, stream,
                    reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), hw, cg, bpi,
                    launch_span());
}

cudaError_t launch_softmax(const float* logits, float* probs, int n, int classes,
                           cudaStream_t stream) {
  const int rows_per_block = kBlock / 32;
  return launch_pdl(softmax_kernel, dim3((n + rows_per_block - 1) / rows_per_block), dim3(kBlock),
                    0, stream, logits, probs, n, classes, launch_span());
  return cudaGetLastError();
}

}  // namespace ds
