// 3x3 max / average pooling streamed through TMA halo boxes (K4 in DESIGN.md).
//
// The structure of the TMA depthwise kernel (dwconv_tma.cu) without weights:
// a persistent CTA walks output tiles of TH x TW pixels x up to 64 channels;
// each tile's input halo is one 4-D TMA box {cb ch, IW, IH, 1} in a 2-4 deep
// mbarrier ring, so every input byte crosses HBM once and all 9 taps come
// from shared memory (the register-blocked pool3x3_rows_kernel re-read its
// taps through L1 and ran at ~0.22 of HBM on Inception's 3x3 average pools).
// A thread owns one 8-channel group of a strip of Q outputs along W.
//
// Numerics are those of pool3x3_rows_kernel, bit for bit: taps row-outer,
// column-inner; averages accumulate acc + x as fma.rn.f32.bf16(x, 1.0, acc)
// in fp32 from 0 and divide by 9 (count_include_pad — box elements over the
// image edge read zeros, and acc + 0 == acc); max compares packed bf16 pairs.
// Max pooling over padding reads those zeros as taps, which equals skipping
// them only for inputs >= 0: the runtime routes a padded max pool here only
// when its input is a ReLU output (ResNet's stem pool); unpadded pools
// (Inception's stride-2 pools) have no edge taps.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "conv_gemm.cuh"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "stream_ops.cuh"

namespace ds {

namespace {

constexpr int kPoolMaxThreads = 256;

__device__ __forceinline__ float add_lo(uint32_t x, float c) {
  float d;
  asm("{.reg .b16 xl, xh, one;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b16 one, 0x3F80;\n\t"
      "fma.rn.f32.bf16 %0, xl, one, %2;}"
      : "=f"(d)
      : "r"(x), "f"(c));
  return d;
}

__device__ __forceinline__ float add_hi(uint32_t x, float c) {
  float d;
  asm("{.reg .b16 xl, xh, one;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b16 one, 0x3F80;\n\t"
      "fma.rn.f32.bf16 %0, xh, one, %2;}"
      : "=f"(d)
      : "r"(x), "f"(c));
  return d;
}

__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// x / 9 correctly rounded without the IEEE division sequence: the product
// with RN(1/9) corrected by one fma residual step. Checked exhaustively
// against x / 9.0f over every finite fp32 (equal except x = -0, which a sum
// starting from +0 never produces).
__device__ __forceinline__ float div9(float x) {
  constexpr float kInv9 = 1.0f / 9.0f;
  const float q0 = __fmul_rn(x, kInv9);
  const float r = __fmaf_rn(-q0, 9.0f, x);
  return __fmaf_rn(r, kInv9, q0);
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

struct FastDivP {
  uint32_t d, mul, shift;
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (__umulhi(n, mul) + n) >> shift;
  }
};

FastDivP fastdiv(uint32_t d) {
  FastDivP f{d, 0, 0};
  while ((1u << f.shift) < d) ++f.shift;
  f.mul = static_cast<uint32_t>(((static_cast<uint64_t>(1) << 32) *
                                 ((static_cast<uint64_t>(1) << f.shift) - d)) / d + 1);
  return f;
}

struct PoolArgs {
  uint4* y;        // output pixels, ldo_g 8-channel groups apart, at group coff_g
  int ldo_g, coff_g;
  int c, ho, wo, pad;
  int tw, th;      // tile: TW x TH output pixels
  int glog2;       // 8-channel groups per tile (log2)
  int iw, ih;      // box W, H
  int tiles_x, tiles_y, n, cblocks, tiles;
  FastDivP div_tx, div_ty, div_sp;  // by tiles_x, tiles_y, tiles_x * tiles_y * n
  int stages;
  uint32_t box_bytes;     // TMA transaction bytes per box
  uint32_t stage_bytes;   // ring slot stride (box_bytes rounded up to 128 B: TMA destination alignment)
  unsigned long long* span;  // live timing slot (pdl.cuh span_mark)
  // average pools after swap_avgpool_1x1 (model.hpp): + bias[channel] after
  // the division, then ReLU if relu (nullptr: plain pool)
  const float* bias;
  int relu;
};

// Tile t -> (channel block [slowest], image, tile row, tile column).
template <int S, int Q, bool MAX>
__global__ void __launch_bounds__(kPoolMaxThreads) pool_tma_kernel(
    const __grid_constant__ CUtensorMap in_map, const __grid_constant__ PoolArgs a) {
  constexpr int XN = (Q - 1) * S + 3;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * a.stage_bytes);
  const int groups = 1 << a.glog2;
  const int cb = groups * 8;
  auto coords = [&](int t, int& cbk, int& tx, int& ty, int& tn) {
    cbk = static_cast<int>(a.div_sp.div(static_cast<uint32_t>(t)));
    const int r = t - cbk * static_cast<int>(a.div_sp.d);
    const int q = static_cast<int>(a.div_tx.div(static_cast<uint32_t>(r)));
    tx = r - q * a.tiles_x;
    tn = static_cast<int>(a.div_ty.div(static_cast<uint32_t>(q)));
    ty = q - tn * a.tiles_y;
  };
  auto issue = [&](int t, int stage) {
    int cbk, tx, ty, tn;
    coords(t, cbk, tx, ty, tn);
    ptx::mbar_arrive_expect_tx(&full[stage], a.box_bytes);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(smem + stage * a.stage_bytes)),
        "l"(&in_map), "r"(ptx::smem_u32(&full[stage])), "r"(cbk * cb),
        "r"(tx * a.tw * S - a.pad), "r"(ty * a.th * S - a.pad), "r"(tn)
        : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&in_map);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // the input is the previous layer's output
  span_mark(a.span);
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      const int t = blockIdx.x + s * gridDim.x;
      if (t < a.tiles) issue(t, s);
    }
  }
  const int spr = a.tw / Q;
  const int items = (spr * a.th) << a.glog2;
  const bool active = static_cast<int>(threadIdx.x) < items;
  const int g = threadIdx.x & (groups - 1);
  const int strip = threadIdx.x >> a.glog2;
  const int sx = strip % spr, oyl = strip / spr;
  const uint4* my_box =
      reinterpret_cast<const uint4*>(smem) + (((oyl * S) * a.iw + sx * Q * S) << a.glog2) + g;
  const int box_vecs = static_cast<int>(a.stage_bytes >> 4);
  int stage = 0;
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
    int cbk, tx, ty, tn;
    coords(t, cbk, tx, ty, tn);
    const int oy = ty * a.th + oyl;
    const int ox0 = tx * a.tw + sx * Q;
    ptx::mbar_wait(&full[stage], phase);
    if (active && oy < a.ho && ox0 < a.wo) {
      const uint4* box = my_box + stage * box_vecs;
      uint4 mx[Q];
      float acc[Q][8];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        mx[q] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // -inf pairs
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[q][e] = 0.f;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const uint4* row = box + ((r * a.iw) << a.glog2);
        uint4 xv[XN];
#pragma unroll
        for (int u = 0; u < XN; ++u) xv[u] = row[u << a.glog2];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            const uint4 v = xv[q * S + s];
            if constexpr (MAX) {
              mx[q].x = vmax(mx[q].x, v.x);
              mx[q].y = vmax(mx[q].y, v.y);
              mx[q].z = vmax(mx[q].z, v.z);
              mx[q].w = vmax(mx[q].w, v.w);
            } else {
              acc[q][0] = add_lo(v.x, acc[q][0]);
              acc[q][1] = add_hi(v.x, acc[q][1]);
              acc[q][2] = add_lo(v.y, acc[q][2]);
              acc[q][3] = add_hi(v.y, acc[q][3]);
              acc[q][4] = add_lo(v.z, acc[q][4]);
              acc[q][5] = add_hi(v.z, acc[q][5]);
              acc[q][6] = add_lo(v.w, acc[q][6]);
              acc[q][7] = add_hi(v.w, acc[q][7]);
            }
          }
      }
      uint4* yp = a.y + (static_cast<long long>(tn * a.ho + oy) * a.wo + ox0) * a.ldo_g + a.coff_g +
                  cbk * groups + g;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (ox0 + q >= a.wo) break;
        if constexpr (MAX) {
          yp[q * a.ldo_g] = mx[q];
        } else {
          float* v = acc[q];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = div9(v[e]);
          if (a.bias) {
            const float4* b4 = reinterpret_cast<const float4*>(a.bias) + 2 * (cbk * groups + g);
            const float4 b0 = __ldg(b4), b1 = __ldg(b4 + 1);
            v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
            v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
            if (a.relu)
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.0f);
          }
          yp[q * a.ldo_g] = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]),
                                       pack2(v[6], v[7]));
        }
      }
    }
    __syncthreads();  // every thread is done with this stage's box
    if (threadIdx.x == 0) {
      const int nt = t + a.stages * static_cast<int>(gridDim.x);
      if (nt < a.tiles) issue(nt, stage);
    }
    if (++stage == a.stages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

struct PoolPlan {
  int q, tw, th, cb;
  bool ok;
};

// Channel block: 64 (or the largest of 32/16/8 dividing C); Q outputs per
// strip (4 at stride 1, 2 at stride 2); the tile width among Q*{2..9} that
// wastes the fewest columns of the last tile (ties: wider); as many rows as
// 256 threads allow.
PoolPlan pool_plan(int ho, int wo, int c, int stride) {
  PoolPlan p{0, 0, 0, 0, false};
  if (c % 8 != 0 || (stride != 1 && stride != 2)) return p;
  const int cb = c % 64 == 0 ? 64 : c % 32 == 0 ? 32 : c % 16 == 0 ? 16 : 8;
  const int q = stride == 1 ? 4 : 2;
  const int groups = cb / 8;
  int best_tw = 0, best_waste = 1 << 30;
  for (int k = 2; k <= 9; ++k) {
    const int tw = q * k;
    if (k * groups > kPoolMaxThreads) break;
    const int waste = (wo + tw - 1) / tw * tw - wo;
    if (waste < best_waste || (waste == best_waste && tw > best_tw)) {
      best_waste = waste;
      best_tw = tw;
    }
    if (tw >= wo) break;
  }
  if (best_tw == 0) return p;
  const int th = std::max(1, std::min(ho, kPoolMaxThreads / ((best_tw / q) * groups)));
  const int iw = (best_tw - 1) * stride + 3, ih = (th - 1) * stride + 3;
  if (iw > 256 || ih > 256) return p;
  return PoolPlan{q, best_tw, th, cb, true};
}

int pool_sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return budgeted_sms(n);
}

template <int S, int Q, bool MAX>
cudaError_t launch(const CUtensorMap& map, const PoolArgs& a, int threads, cudaStream_t stream) {
  auto kernel = pool_tma_kernel<S, Q, MAX>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const size_t smem = static_cast<size_t>(a.stages) * a.stage_bytes + 8 * a.stages + 16;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int grid = std::min(a.tiles, pool_sm_count() * per_sm);
  return launch_pdl(kernel, dim3(grid), dim3(threads), smem, stream, map, a);
}

}  // namespace

bool pool_tma_plan_ok(int h, int w, int c, int stride, int pad) {
  const int ho = (h + 2 * pad - 3) / stride + 1, wo = (w + 2 * pad - 3) / stride + 1;
  return pad >= 0 && pad <= 1 && pool_plan(ho, wo, c, stride).ok;
}

bool pool_tma_input_map(CUtensorMap* map, const void* x, int max_n, int h, int w, int c,
                        int stride, int pad) {
  if (!pool_tma_plan_ok(h, w, c, stride, pad)) return false;
  const int ho = (h + 2 * pad - 3) / stride + 1, wo = (w + 2 * pad - 3) / stride + 1;
  const PoolPlan p = pool_plan(ho, wo, c, stride);
  return encode_tmap_nhwc(map, x, max_n, h, w, c, p.cb, (p.tw - 1) * stride + 3,
                          (p.th - 1) * stride + 3, 1);
}

cudaError_t launch_pool3x3_tma(const CUtensorMap& in_map, __nv_bfloat16* y, int n, int h, int w,
                               int c, int stride, int pad, bool is_max, int ldo, int c_off,
                               cudaStream_t stream, const float* post_bias, bool post_relu) {
  if (!pool_tma_plan_ok(h, w, c, stride, pad) || ldo % 8 != 0 || c_off % 8 != 0)
    return cudaErrorInvalidValue;
  const int ho = (h + 2 * pad - 3) / stride + 1, wo = (w + 2 * pad - 3) / stride + 1;
  const PoolPlan p = pool_plan(ho, wo, c, stride);
  PoolArgs a{};
  a.span = launch_span();
  if (post_bias && is_max) return cudaErrorInvalidValue;
  a.bias = post_bias;
  a.relu = post_relu ? 1 : 0;
  a.y = reinterpret_cast<uint4*>(y);
  a.ldo_g = ldo / 8;
  a.coff_g = c_off / 8;
  a.c = c;
  a.ho = ho;
  a.wo = wo;
  a.pad = pad;
  a.tw = p.tw;
  a.th = p.th;
  int glog2 = 0;
  while ((8 << glog2) < p.cb) ++glog2;
  a.glog2 = glog2;
  a.iw = (p.tw - 1) * stride + 3;
  a.ih = (p.th - 1) * stride + 3;
  a.tiles_x = (wo + p.tw - 1) / p.tw;
  a.tiles_y = (ho + p.th - 1) / p.th;
  a.n = n;
  a.cblocks = c / p.cb;
  a.tiles = a.tiles_x * a.tiles_y * n * a.cblocks;
  a.div_tx = fastdiv(static_cast<uint32_t>(a.tiles_x));
  a.div_ty = fastdiv(static_cast<uint32_t>(a.tiles_y));
  a.div_sp = fastdiv(static_cast<uint32_t>(a.tiles_x * a.tiles_y * n));
  a.box_bytes = static_cast<uint32_t>(a.iw * a.ih * p.cb * 2);
  a.stage_bytes = (a.box_bytes + 127u) / 128u * 128u;
  constexpr int kBudget = 72 * 1024, kSmemCap = 200 * 1024;
  int st = std::max(2, std::min(4, kBudget / static_cast<int>(a.stage_bytes)));
  while (st > 2 && st * static_cast<int>(a.stage_bytes) + 8 * st + 16 > kSmemCap) --st;
  a.stages = st;
  const int items = ((p.tw / p.q) * p.th) * (p.cb / 8);
  const int threads = std::min(kPoolMaxThreads, (items + 31) / 32 * 32);
  if (stride == 1)
    return is_max ? launch<1, 4, true>(in_map, a, threads, stream)
                  : launch<1, 4, false>(in_map, a, threads, stream);
  return is_max ? launch<2, 2, true>(in_map, a, threads, stream)
                : launch<2, 2, false>(in_map, a, threads, stream);
}

}  // namespace ds
