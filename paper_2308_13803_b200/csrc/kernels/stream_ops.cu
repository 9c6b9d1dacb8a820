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

__global__ void stage_input_kernel(const uint8_t* __restrict__ img, uint2* __restrict__ out,
                                   long long pixels, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= pixels) return;
  const uint8_t* s = img + 3 * p;
  float v[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = (static_cast<float>(s[c]) - 127.5f) / 63.75f;
  out[p] = make_uint2(pack2(v[0], v[1]), pack2(v[2], 0.0f));
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

// Depthwise 3x3, register-blocked: a thread owns 8 channels (one 16 B
// vector) x kDwCols consecutive output columns of one output row, so each
// loaded input vector feeds up to 3 outputs from registers; consecutive
// threads take consecutive channel groups (coalesced 16 B loads/stores along
// C). Weights come through the read-only path (L1-resident per block).
constexpr int kDwCols = 4;

template <int STRIDE>
__global__ void __launch_bounds__(kBlock) dwconv3x3_kernel(
    const uint4* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    const float* __restrict__ bias, uint4* __restrict__ y, int h, int wd, int c, int ho, int wo,
    int cg_log2, int xq_per_row, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  // grid.y = output row (image * ho + oy); x covers (column quad, channel group)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int cg = 1 << cg_log2;
  const int g = i & (cg - 1);
  const int xq = i >> cg_log2;
  if (xq >= xq_per_row) return;
  const int row = blockIdx.y;
  const int n = row / ho;
  const int oy = row - n * ho;
  const int ox0 = xq * kDwCols;
  constexpr int IN_COLS = (kDwCols - 1) * STRIDE + 3;
  const int ix0 = ox0 * STRIDE - 1;

  float acc[kDwCols][8];
  const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias) + 2 * g);
  const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias) + 2 * g + 1);
  const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int q = 0; q < kDwCols; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = bv[e];
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  // All weight vectors, then each stencil row's input vectors, are issued
  // before first use so several loads are in flight per thread (the loop was
  // latency-bound on load -> use). Taps outside the image are skipped, not
  // multiplied by zero, to keep the FMA sequence of the fused path.
  uint4 wraw[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) wraw[t] = __ldg(wv + t * cg + g);

#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int iy = oy * STRIDE - 1 + r;
    const bool row_ok = iy >= 0 && iy < h;
    const uint4* xrow = x + (static_cast<long long>(n) * h + (row_ok ? iy : 0)) * wd * cg + g;
    uint4 raw[IN_COLS];
    bool ok[IN_COLS];
#pragma unroll
    for (int col = 0; col < IN_COLS; ++col) {
      const int ix = ix0 + col;
      ok[col] = row_ok && ix >= 0 && ix < wd;
      raw[col] = ok[col] ? __ldg(xrow + static_cast<long long>(ix) * cg) : make_uint4(0, 0, 0, 0);
    }
    float wr[3][8];
#pragma unroll
    for (int s = 0; s < 3; ++s) unpack8(wraw[r * 3 + s], wr[s]);
#pragma unroll
    for (int col = 0; col < IN_COLS; ++col) {
      if (!ok[col]) continue;
      float xv[8];
      unpack8(raw[col], xv);
#pragma unroll
      for (int q = 0; q < kDwCols; ++q) {
        const int s = col - q * STRIDE;  // tap of output q that reads this column
        if (s < 0 || s > 2) continue;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[q][e] = fmaf(xv[e], wr[s][e], acc[q][e]);
      }
    }
  }
  uint4* yrow = y + (static_cast<long long>(n) * ho + oy) * wo * cg + g;
#pragma unroll
  for (int q = 0; q < kDwCols; ++q) {
    if (ox0 + q >= wo) break;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = fmaxf(acc[q][e], 0.0f);
    yrow[static_cast<long long>(ox0 + q) * cg] = pack8(acc[q]);
  }
}

// One output pixel x 8 channels per thread (stride-2 layers, where a
// column is shared by at most two outputs and blocking does not pay).
__global__ void dwconv3x3_px_kernel(const uint4* __restrict__ x, const uint4* __restrict__ w,
                                 const float4* __restrict__ bias, uint4* __restrict__ y, int h,
                                 int wd, int cg, int ho, int wo, int stride, long long work, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= work) return;
  const int g = static_cast<int>(i % cg);
  long long pix = i / cg;
  const int ox = static_cast<int>(pix % wo);
  pix /= wo;
  const int oy = static_cast<int>(pix % ho);
  const int n = static_cast<int>(pix / ho);
  float acc[8];
  const float4 b0 = __ldg(bias + 2 * g), b1 = __ldg(bias + 2 * g + 1);
  acc[0] = b0.x; acc[1] = b0.y; acc[2] = b0.z; acc[3] = b0.w;
  acc[4] = b1.x; acc[5] = b1.y; acc[6] = b1.z; acc[7] = b1.w;
  const int iy0 = oy * stride - 1, ix0 = ox * stride - 1;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int iy = iy0 + r;
    if (iy < 0 || iy >= h) continue;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int ix = ix0 + s;
      if (ix < 0 || ix >= wd) continue;
      float xv[8], wv[8];
      unpack8(__ldg(x + ((static_cast<long long>(n) * h + iy) * wd + ix) * cg + g), xv);
      unpack8(__ldg(w + (r * 3 + s) * cg + g), wv);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(xv[e], wv[e], acc[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = fmaxf(acc[e], 0.0f);
  y[i] = pack8(acc);
}

__global__ void pool3x3_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int h, int w,
                               int cg, int ho, int wo, int stride, int pad, int is_max, int ldo_g,
                               int coff_g, long long work, unsigned long long* span) {
  pdl_trigger();
  pdl_wait();
  span_mark(span);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= work) return;
  const int g = static_cast<int>(i % cg);
  long long pix = i / cg;
  const int ox = static_cast<int>(pix % wo);
  pix /= wo;
  const int oy = static_cast<int>(pix % ho);
  const int n = static_cast<int>(pix / ho);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = is_max ? -INFINITY : 0.0f;
  const int iy0 = oy * stride - pad, ix0 = ox * stride - pad;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int iy = iy0 + r;
    if (iy < 0 || iy >= h) continue;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int ix = ix0 + s;
      if (ix < 0 || ix >= w) continue;
      float xv[8];
      unpack8(__ldg(x + ((static_cast<long long>(n) * h + iy) * w + ix) * cg + g), xv);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = is_max ? fmaxf(acc[e], xv[e]) : acc[e] + xv[e];
    }
  }
  if (!is_max) {
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = acc[e] / 9.0f;
  }
  const long long opix = (static_cast<long long>(n) * ho + oy) * wo + ox;
  y[opix * ldo_g + coff_g + g] = pack8(acc);
}

// 3x3 pooling on a 2-D grid: grid.y = output row (image, oy), x = (output
// column, 8-channel group); 32-bit index arithmetic (the column / group split
// through an exact float-reciprocal division). Max pooling compares the
// packed bf16 pairs directly (max is exact in any precision); average pooling
// accumulates with fma.rn.f32.bf16(x, 1.0, acc) == acc + float(x), one
// instruction per element. Per output the taps are visited in the same order
// as pool3x3_kernel (row outer, column inner, padding skipped) and averages
// divide the fp32 sum by 9, so results are bit-identical to it
// (DS_POOL_LEGACY=1 selects the old kernel).
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

cudaError_t launch_stage_input(const uint8_t* img, __nv_bfloat16* out, int n, int h, int w,
                               cudaStream_t stream) {
  const long long pixels = static_cast<long long>(n) * h * w;
  return launch_pdl(stage_input_kernel, dim3(grid_for(pixels)), dim3(kBlock), 0, stream, img,
                    reinterpret_cast<uint2*>(out), pixels, launch_span());
  return cudaGetLastError();
}

cudaError_t launch_stage_s2d(const uint8_t* img, __nv_bfloat16* out, int n, int h, int w, int hs,
                             int ws, int pad, cudaStream_t stream) {
  const long long pixels = static_cast<long long>(n) * hs * ws;
  if (pixels >= (1LL << 31)) return cudaErrorInvalidValue;
  return launch_pdl(stage_s2d_kernel, dim3(grid_for(pixels)), dim3(kBlock), 0, stream, img,
                    reinterpret_cast<uint4*>(out), h, w, hs, ws, pad, pixels, launch_span());
}

cudaError_t launch_dwconv3x3(const __nv_bfloat16* x, const __nv_bfloat16* w, const float* bias,
                             __nv_bfloat16* y, int n, int h, int wd, int c, int stride,
                             cudaStream_t stream) {
  const int ho = (h + 2 - 3) / stride + 1, wo = (wd + 2 - 3) / stride + 1;
  const int cg = c / 8;
  int cg_log2 = 0;
  while ((1 << cg_log2) < cg) ++cg_log2;
  if ((1 << cg_log2) != cg) return cudaErrorInvalidValue;  // channel groups must be a power of 2
  const int rows = n * ho;
  if (rows > 65535) return cudaErrorInvalidValue;
  auto block_for = [](int per_row) { return std::min(kBlock, (per_row + 31) / 32 * 32); };
  if (stride == 1) {
    const int xq = (wo + kDwCols - 1) / kDwCols;
    const int bt = block_for(xq * cg);
    return launch_pdl(dwconv3x3_kernel<1>, dim3((xq * cg + bt - 1) / bt, rows), dim3(bt), 0, stream,
                      reinterpret_cast<const uint4*>(x), w, bias, reinterpret_cast<uint4*>(y), h,
                      wd, c, ho, wo, cg_log2, xq, launch_span());
  } else {
    const long long pw = static_cast<long long>(n) * ho * wo * cg;
    return launch_pdl(dwconv3x3_px_kernel, dim3(grid_for(pw)), dim3(kBlock), 0, stream,
                      reinterpret_cast<const uint4*>(x), reinterpret_cast<const uint4*>(w),
                      reinterpret_cast<const float4*>(bias), reinterpret_cast<uint4*>(y), h, wd,
                      cg, ho, wo, stride, pw, launch_span());
  }
  return cudaGetLastError();
}

cudaError_t launch_pool3x3(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int h, int w, int c,
                           int stride, int pad, bool is_max, int ldo, int c_off,
                           cudaStream_t stream) {
  const int ho = (h + 2 * pad - 3) / stride + 1, wo = (w + 2 * pad - 3) / stride + 1;
  const int cg = c / 8;
  const bool legacy = [] {
    const char* e = std::getenv("DS_POOL_LEGACY");
    return e && e[0] == '1';
  }();
  const char* rows_env = std::getenv("DS_POOL_ROWS");  // output rows per thread: 1 or 2 (A/B)
  const int prows = rows_env ? std::atoi(rows_env) : 2;
  const int yrows = n * ((ho + prows - 1) / prows);
  if (!legacy && yrows <= 65535 && (stride == 1 || stride == 2) && wo * cg < (1 << 24)) {
    const int per_row = wo * cg;
    const int bt = std::min(kBlock, (per_row + 31) / 32 * 32);
    const dim3 grid((per_row + bt - 1) / bt, yrows);
    auto go = [&](auto kernel) {
      return launch_pdl(kernel, grid, dim3(bt), 0, stream, reinterpret_cast<const uint4*>(x),
                        reinterpret_cast<uint4*>(y), h, w, cg, ho, wo, pad, ldo / 8, c_off / 8, launch_span());
    };
    if (prows == 1) {
      if (stride == 1)
        return is_max ? go(pool3x3_rows_kernel<1, true, 1>) : go(pool3x3_rows_kernel<1, false, 1>);
      return is_max ? go(pool3x3_rows_kernel<2, true, 1>) : go(pool3x3_rows_kernel<2, false, 1>);
    }
    if (prows == 4) {
      if (stride == 1)
        return is_max ? go(pool3x3_rows_kernel<1, true, 4>) : go(pool3x3_rows_kernel<1, false, 4>);
      return is_max ? go(pool3x3_rows_kernel<2, true, 4>) : go(pool3x3_rows_kernel<2, false, 4>);
    }
    if (stride == 1)
      return is_max ? go(pool3x3_rows_kernel<1, true, 2>) : go(pool3x3_rows_kernel<1, false, 2>);
    return is_max ? go(pool3x3_rows_kernel<2, true, 2>) : go(pool3x3_rows_kernel<2, false, 2>);
  }
  const long long work = static_cast<long long>(n) * ho * wo * cg;
  return launch_pdl(pool3x3_kernel, dim3(grid_for(work)), dim3(kBlock), 0, stream,
                    reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), h, w, cg, ho,
                    wo, stride, pad, is_max ? 1 : 0, ldo / 8, c_off / 8, work, launch_span());
  return cudaGetLastError();
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
