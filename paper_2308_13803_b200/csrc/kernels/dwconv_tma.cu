// Depthwise 3x3 (+bias, ReLU) streamed through TMA (K3 in DESIGN.md).
//
// A persistent CTA walks output tiles of TH x TW pixels (x NB images for the
// 7x7 tail) x up to 64 channels. Each tile's input halo is one 4-D TMA box
// {cb ch, IW, IH, NB images} landing in shared memory; box elements that hang
// over the image edge read zeros, which is exactly the convolution's padding.
// A ring of 2-4 boxes (mbarrier transaction counts) keeps the next tiles'
// halos streaming in while the current one is computed, so every input byte
// crosses HBM once and all 9 taps of every output come from smem.
//
// A thread owns one 8-channel group (16 B) of a strip of Q consecutive output
// pixels along W: each input vector it loads from smem feeds up to 3 of its
// outputs ((Q-1)*S+3 loads per row instead of 3*Q). The multiply-adds are
// FHFMA.BF16 — fp32 fma with the bf16 operands read straight from the packed
// halves of a register — so nothing is unpacked; the product of two bf16 is
// exact in fp32, so each step equals fmaf on the widened values (same
// rounding as the previous unpack-then-fmaf kernels, bit for bit).
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

constexpr int kDwMaxThreads = 256;

// acc += bf16(x.lo) * bf16(w.lo) (fp32 fma), and the same for the high halves.
__device__ __forceinline__ float fma_bf16_lo(uint32_t x, uint32_t w, float c) {
  float d;
  asm("{.reg .b16 xl, xh, wl, wh;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b32 {wl, wh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, xl, wl, %3;}"
      : "=f"(d)
      : "r"(x), "r"(w), "f"(c));
  return d;
}

__device__ __forceinline__ float fma_bf16_hi(uint32_t x, uint32_t w, float c) {
  float d;
  asm("{.reg .b16 xl, xh, wl, wh;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b32 {wl, wh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, xh, wh, %3;}"
      : "=f"(d)
      : "r"(x), "r"(w), "f"(c));
  return d;
}

__device__ __forceinline__ void fma8(float (&acc)[8], const uint4& x, const uint4& w) {
  acc[0] = fma_bf16_lo(x.x, w.x, acc[0]);
  acc[1] = fma_bf16_hi(x.x, w.x, acc[1]);
  acc[2] = fma_bf16_lo(x.y, w.y, acc[2]);
  acc[3] = fma_bf16_hi(x.y, w.y, acc[3]);
  acc[4] = fma_bf16_lo(x.z, w.z, acc[4]);
  acc[5] = fma_bf16_hi(x.z, w.z, acc[5]);
  acc[6] = fma_bf16_lo(x.w, w.w, acc[6]);
  acc[7] = fma_bf16_hi(x.w, w.w, acc[7]);
}

__device__ __forceinline__ uint32_t pack2f(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// relu then round == round then relu (rounding is monotonic and keeps 0), so
// the ReLU runs on the packed bf16 pair: one max.bf16x2 instead of two FMNMX.
__device__ __forceinline__ uint32_t relu_pack2(float lo, float hi) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(pack2f(lo, hi)), "r"(0u));
  return d;
}

// n / d for 0 <= n < 2^31 by multiply-high and shift (d >= 1, host-built).
struct FastDiv {
  uint32_t d, mul, shift;
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    return (__umulhi(n, mul) + n) >> shift;
#else
    return static_cast<uint32_t>(((static_cast<uint64_t>(n) * mul >> 32) + n) >> shift);
#endif
  }
};

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  while ((1u << f.shift) < d) ++f.shift;
  f.mul = static_cast<uint32_t>(((static_cast<uint64_t>(1) << 32) *
                                 ((static_cast<uint64_t>(1) << f.shift) - d)) / d + 1);
  return f;
}

struct DwKernelArgs {
  const __nv_bfloat16* w;  // [9][C]
  const float* bias;       // [C]
  uint4* y;                // NHWC output, 8 channels per vector
  int n, c, ho, wo;
  int tw, th, nb;          // tile: TW x TH pixels x NB images
  int glog2;               // 8-channel groups per tile (log2)
  int iw, ih;              // box W, H
  int tiles_x, tiles_y, tiles_n, cblocks, tiles;
  FastDiv div_tx, div_ty, div_sp;  // by tiles_x, tiles_y, tiles_x*tiles_y*tiles_n
  int stages;
  uint32_t box_bytes;
  unsigned long long* span;  // live timing slot (pdl.cuh span_mark)
};

// Tile t -> (channel block, x, y, image block). The channel block varies
// slowest, so a persistent CTA keeps one block's weights in registers for
// many consecutive tiles.
template <int S, int Q>
__global__ void __launch_bounds__(kDwMaxThreads) dw_tma_kernel(
    const __grid_constant__ CUtensorMap in_map, const __grid_constant__ DwKernelArgs a) {
  constexpr int XN = (Q - 1) * S + 3;  // input vectors per strip row
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * a.box_bytes);
  const int groups = 1 << a.glog2;
  const int cb = groups * 8;

  auto coords = [&](int t, int& cbk, int& tx, int& ty, int& tn) {
    cbk = static_cast<int>(a.div_sp.div(static_cast<uint32_t>(t)));
    int r = t - cbk * static_cast<int>(a.div_sp.d);
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
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(smem + stage * a.box_bytes)),
        "l"(&in_map), "r"(ptx::smem_u32(&full[stage])), "r"(cbk * cb), "r"(tx * a.tw * S - 1),
        "r"(ty * a.th * S - 1), "r"(tn * a.nb)
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

  // This thread's item — one strip of Q outputs x 8 channels — is the same in
  // every tile (the host sizes the block to the tile's items).
  const int cg_all = a.c >> 3;
  const int spr = a.tw / Q;  // strips per tile row
  const int items = (spr * a.th * a.nb) << a.glog2;
  const bool active = static_cast<int>(threadIdx.x) < items;
  const int g = threadIdx.x & (groups - 1);
  int sx, oyl, nbl;
  {
    int strip = threadIdx.x >> a.glog2;
    sx = strip % spr;
    strip /= spr;
    oyl = strip % a.th;
    nbl = strip / a.th;
  }
  const uint4* my_box = reinterpret_cast<const uint4*>(smem) +
                        (((nbl * a.ih + oyl * S) * a.iw + sx * Q * S) << a.glog2) + g;
  const int box_vecs = static_cast<int>(a.box_bytes >> 4);
  uint4 w[9];
  float bias[8];
  int cur_cbk = -1;
  uint32_t j = 0;
  int stage = 0;
  uint32_t phase = 0;  // (ring position advanced without divisions)
  for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++j) {
    int cbk, tx, ty, tn;
    coords(t, cbk, tx, ty, tn);
    const int oy = ty * a.th + oyl;
    const int img = tn * a.nb + nbl;
    const int gg = cbk * groups + g;  // global channel group
    if (cbk != cur_cbk) {
      cur_cbk = cbk;
#pragma unroll
      for (int k = 0; k < 9; ++k) w[k] = __ldg(reinterpret_cast<const uint4*>(a.w) + k * cg_all + gg);
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(a.bias) + 2 * gg);
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(a.bias) + 2 * gg + 1);
      bias[0] = b0.x; bias[1] = b0.y; bias[2] = b0.z; bias[3] = b0.w;
      bias[4] = b1.x; bias[5] = b1.y; bias[6] = b1.z; bias[7] = b1.w;
    }
    ptx::mbar_wait(&full[stage], phase);
    if (active && oy < a.ho && img < a.n) {
      float acc[Q][8];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[q][e] = bias[e];
      const uint4* box = my_box + stage * box_vecs;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const uint4* row = box + ((r * a.iw) << a.glog2);
        uint4 xv[XN];
#pragma unroll
        for (int u = 0; u < XN; ++u) xv[u] = row[u << a.glog2];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int s = 0; s < 3; ++s) fma8(acc[q], xv[q * S + s], w[r * 3 + s]);
      }
      uint4* yp = a.y + ((static_cast<long long>(img) * a.ho + oy) * a.wo + tx * a.tw + sx * Q) *
                            cg_all + gg;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        float* v = acc[q];
        yp[q * cg_all] = make_uint4(relu_pack2(v[0], v[1]),
                                    relu_pack2(v[2], v[3]),
                                    relu_pack2(v[4], v[5]),
                                    relu_pack2(v[6], v[7]));
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


int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return budgeted_sms(n);
}

// Tile shape per layer (output width, stride, channels): a strip of Q outputs
// per thread, TW | wo, and (TW/Q)*TH*NB*groups close to a multiple of 32 <= 256.
struct DwPlan {
  int q, tw, th, nb, cb;
  bool ok;
};

DwPlan dw_plan(int ho, int wo, int c, int stride) {
  const int cb = std::min(c, 64);
  DwPlan p{0, 0, 0, 1, cb, false};
  auto set = [&](int q, int tw, int th, int nb) {
    const int items = (tw / q) * th * nb * (cb / 8);  // one per thread
    if (wo % tw == 0 && tw % q == 0 && items <= kDwMaxThreads) p = DwPlan{q, tw, th, nb, cb, true};
  };
  if (stride == 1) {
    if (wo % 16 == 0 && wo >= 64) set(4, 16, cb >= 64 ? 8 : 16, 1);  // 112x112
    else if (wo % 8 == 0 && wo >= 48) set(4, 8, 14, 1);              // 56x56
    else if (wo % 4 == 0 && wo >= 20) set(4, wo, 4, 1);              // 28x28
    else if (wo % 7 == 0 && wo >= 14) set(7, wo, std::min(ho, 14), 1);  // 14x14
    else if (wo == 7) set(7, 7, 7, 4);                                // 7x7
  } else {
    if (wo % 8 == 0 && wo >= 48) set(2, 8, 8, 1);                     // 112 -> 56
    else if (wo % 14 == 0) set(2, 14, 4, 1);                          // 56 -> 28, 28 -> 14
    else if (wo == 7) set(7, 7, 7, 2);                                // 14 -> 7
  }
  return p;
}

DwKernelArgs make_args(const DwPlan& p, int n, int h, int w, int c, int stride) {
  DwKernelArgs a{};
  a.n = n;
  a.c = c;
  a.ho = (h - 1) / stride + 1;
  a.wo = (w - 1) / stride + 1;
  a.tw = p.tw;
  a.th = p.th;
  a.nb = p.nb;
  int glog2 = 0;
  while ((8 << glog2) < p.cb) ++glog2;
  a.glog2 = glog2;
  a.iw = (p.tw - 1) * stride + 3;
  a.ih = (p.th - 1) * stride + 3;
  a.tiles_x = a.wo / p.tw;
  a.tiles_y = (a.ho + p.th - 1) / p.th;
  a.tiles_n = (n + p.nb - 1) / p.nb;
  a.cblocks = c / p.cb;
  a.tiles = a.tiles_x * a.tiles_y * a.tiles_n * a.cblocks;
  a.div_tx = make_fastdiv(static_cast<uint32_t>(a.tiles_x));
  a.div_ty = make_fastdiv(static_cast<uint32_t>(a.tiles_y));
  a.div_sp = make_fastdiv(static_cast<uint32_t>(a.tiles_x * a.tiles_y * a.tiles_n));
  a.box_bytes = static_cast<uint32_t>(a.iw * a.ih * p.nb * p.cb * 2);
  // 2-4 boxes in flight, <= ~72 KB per CTA so three CTAs share an SM (the
  // ring always fits the 200 KB dynamic shared memory set in launch_plan)
  constexpr int kBudget = 72 * 1024, kMaxStages = 4, kSmemCap = 200 * 1024;
  int st = std::max(2, std::min(kMaxStages, static_cast<int>(kBudget / a.box_bytes)));
  while (st > 2 && st * static_cast<int>(a.box_bytes) + 8 * st + 16 > kSmemCap) --st;
  a.stages = st;
  return a;
}

template <int S, int Q>
cudaError_t launch_plan(const CUtensorMap& map, DwKernelArgs a, const DwPlan& p,
                        cudaStream_t stream) {
  auto kernel = dw_tma_kernel<S, Q>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int items = ((p.tw / Q) * p.th * p.nb) * (p.cb / 8);
  const int threads = std::min(kDwMaxThreads, (items + 31) / 32 * 32);
  const size_t smem = static_cast<size_t>(a.stages) * a.box_bytes + 8 * a.stages + 16;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int grid = std::min(a.tiles, sm_count() * per_sm);
  return launch_pdl(kernel, dim3(grid), dim3(threads), smem, stream, map, a);
}

}  // namespace

bool dwconv_tma_supported(int c) {
  return c >= 8 && (c & (c - 1)) == 0;  // power-of-two channel count (>= one 16 B group)
}

bool dwconv_tma_plan_ok(int h, int w, int c, int stride) {
  if (!dwconv_tma_supported(c) || (stride != 1 && stride != 2)) return false;
  return dw_plan((h - 1) / stride + 1, (w - 1) / stride + 1, c, stride).ok;
}

cudaError_t launch_dwconv3x3_tma(const CUtensorMap& in_map, const __nv_bfloat16* w,
                                 const float* bias, __nv_bfloat16* y, int n, int h, int wd, int c,
                                 int stride, cudaStream_t stream) {
  if (!dwconv_tma_plan_ok(h, wd, c, stride)) return cudaErrorInvalidValue;
  const DwPlan p = dw_plan((h - 1) / stride + 1, (wd - 1) / stride + 1, c, stride);
  DwKernelArgs a = make_args(p, n, h, wd, c, stride);
  a.span = launch_span();
  a.w = w;
  a.bias = bias;
  a.y = reinterpret_cast<uint4*>(y);
  if (stride == 1) {
    if (p.q == 4) return launch_plan<1, 4>(in_map, a, p, stream);
    return launch_plan<1, 7>(in_map, a, p, stream);
  }
  if (p.q == 2) return launch_plan<2, 2>(in_map, a, p, stream);
  return launch_plan<2, 7>(in_map, a, p, stream);
}

bool dwconv_tma_input_map(CUtensorMap* map, const void* x, int max_n, int h, int w, int c,
                          int stride) {
  if (!dwconv_tma_plan_ok(h, w, c, stride)) return false;
  const DwPlan p = dw_plan((h - 1) / stride + 1, (w - 1) / stride + 1, c, stride);
  return encode_tmap_nhwc(map, x, max_n, h, w, c, p.cb, (p.tw - 1) * stride + 3,
                          (p.th - 1) * stride + 3, p.nb);
}

}  // namespace ds
