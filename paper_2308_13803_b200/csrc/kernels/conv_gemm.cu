// Implicit-GEMM convolution on the sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// This is the device compute that replaces the analytic stand-in
// `mean_batch_latency` / `mean_mt_latency` (reference perf_model.cpp:70-78)
// behind GpuSim::run_batch / run_mt_request (reference gpu_sim.cpp:13-24):
// every dense conv, 1x1 conv and FC layer of the served networks runs here.
//
// CTA = 6 warps, one 128 x BN output tile:
//   warps 0-3  A producers: gather the im2col rows of the tile straight from
//              the NHWC input with zero-filling cp.async (padding, K tail and
//              M tail become zeros), written in the 128 B-swizzled K-major
//              layout the UMMA descriptor expects; completion is signalled to
//              the stage's full barrier by cp.async.mbarrier.arrive.
//              For 1x1 stride-1 layers the A tile is a plain 2D box and the
//              TMA warp loads it instead (kTmaA).
//              After the main loop the same 4 warps are the epilogue: TMEM ->
//              registers (tcgen05.ld), + bias (+ residual), ReLU, bf16/fp32
//              stores into the (possibly channel-sliced) NHWC output.
//   warp 4     TMA producer for the weight tile (and A in kTmaA); owns TMEM.
//   warp 5     one elected thread issues tcgen05.mma (M=128, N=BN, K=16) into
//              an fp32 TMEM accumulator and commits stage releases.
#include "conv_gemm.cuh"
#include "sm100_ptx.cuh"

#include <cstdio>
#include <mutex>

namespace ds {

namespace {

constexpr int kABytes = kConvBM * kConvBK * 2;  // 16 KiB per stage

struct SmemLayout {
  uint32_t a_off, b_off, bar_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(int BN, int stages) {
  SmemLayout L;
  L.a_off = 0;
  L.b_off = static_cast<uint32_t>(stages) * kABytes;
  L.bar_off = L.b_off + static_cast<uint32_t>(stages) * BN * 128;
  // full[stages], empty[stages], tmem_full, tmem slot
  L.total = L.bar_off + (2 * stages + 2) * 8;
  return L;
}

template <int G>
__device__ __forceinline__ void gather_a_tiles(const ConvGemmArgs& a, uint8_t* smem,
                                               uint64_t* full, uint64_t* empty, int m0) {
  constexpr int GPR = 64 / G;        // granules per 128 B row
  constexpr int RPP = 128 / GPR;     // rows covered per pass of 128 threads
  constexpr int PASSES = 128 / RPP;  // passes per tile
  constexpr int GB = G * 2;          // granule bytes
  const int t = threadIdx.x;
  const int gi = t % GPR;
  const int r0 = t / GPR;
  const int HoWo = a.Ho * a.Wo;

  int pix[PASSES], hi0[PASSES], wi0[PASSES];
#pragma unroll
  for (int p = 0; p < PASSES; ++p) {
    const int m = m0 + r0 + p * RPP;
    if (m < a.M) {
      const int n = m / HoWo;
      const int rem = m - n * HoWo;
      const int ho = rem / a.Wo;
      const int wo = rem - ho * a.Wo;
      pix[p] = n * a.H * a.W;
      hi0[p] = ho * a.stride_h - a.pad_h;
      wi0[p] = wo * a.stride_w - a.pad_w;
    } else {
      pix[p] = 0;
      hi0[p] = -(1 << 28);  // never inside the image: whole row zero-filled
      wi0[p] = 0;
    }
  }

  const uint32_t smem_base = ptx::smem_u32(smem);
  const int col_bytes = gi * GB;
  for (int kb = 0; kb < a.num_kb; ++kb) {
    const int s = kb % a.stages;
    if (kb >= a.stages) ptx::mbar_wait(&empty[s], ((kb / a.stages) - 1) & 1);
    const int k = kb * kConvBK + gi * G;
    const int tap = k / a.C;
    const int c = k - tap * a.C;
    const int r = tap / a.S;
    const int sx = tap - r * a.S;
    const bool kvalid = tap < a.taps;
    const uint32_t sbase = smem_base + s * kABytes;
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      const int row = r0 + p * RPP;
      const int hi = hi0[p] + r;
      const int wi = wi0[p] + sx;
      const bool v = kvalid && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W;
      const __nv_bfloat16* src =
          v ? a.x + (static_cast<size_t>(pix[p] + hi * a.W + wi) * a.C + c) : a.x;
      const uint32_t off =
          row * 128 + ((((col_bytes >> 4) ^ (row & 7)) << 4) | (col_bytes & 15));
      if constexpr (GB == 16) {
        ptx::cp_async_16(sbase + off, src, v ? 16u : 0u);
      } else {
        ptx::cp_async_8(sbase + off, src, v ? 8u : 0u);
      }
    }
    ptx::cp_async_mbar_arrive_noinc(&full[s]);
  }
}

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void epilogue_chunk(const ConvGemmArgs& a, int m, int n,
                                               const uint32_t (&raw)[16]) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]);
  if (n + 16 <= a.Cout) {
    const float4* b4 = reinterpret_cast<const float4*>(a.bias + n);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 b = __ldg(b4 + q);
      v[4 * q + 0] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
    if (a.residual) {
      const uint4* rp =
          reinterpret_cast<const uint4*>(a.residual + static_cast<size_t>(m) * a.ld_res + n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint4 rr = __ldg(rp + q);
        const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[8 * q + 2 * e] += bf16_lo(w[e]);
          v[8 * q + 2 * e + 1] += bf16_hi(w[e]);
        }
      }
    }
    if (a.relu) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.0f);
    }
    if (a.out_f32) {
      float4* yp = reinterpret_cast<float4*>(static_cast<float*>(a.y) +
                                             static_cast<size_t>(m) * a.ldy + a.c_off + n);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        yp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      uint4* yp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) +
                                           static_cast<size_t>(m) * a.ldy + a.c_off + n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        yp[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                           pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                           pack_bf16(v[8 * q + 6], v[8 * q + 7]));
      }
    }
  } else {
    for (int j = 0; j < 16 && n + j < a.Cout; ++j) {
      float x = v[j] + a.bias[n + j];
      if (a.residual) x += __bfloat162float(a.residual[static_cast<size_t>(m) * a.ld_res + n + j]);
      if (a.relu) x = fmaxf(x, 0.0f);
      const size_t o = static_cast<size_t>(m) * a.ldy + a.c_off + n + j;
      if (a.out_f32)
        static_cast<float*>(a.y)[o] = x;
      else
        static_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(x);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_gemm_kernel(const __grid_constant__ ConvGemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128 B swizzle atoms must sit on 1 KiB boundaries.
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const SmemLayout L = smem_layout(args.BN, args.stages);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + args.stages;
  uint64_t* tmem_full = empty + args.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * args.BN;
  const int m0 = blockIdx.y * kConvBM;

  if (warp == 4) {
    if (lane == 0) {
      const uint32_t a_arrivals = (MODE == static_cast<int>(ConvLoadMode::kTmaA)) ? 0u : 128u;
      for (int s = 0; s < args.stages; ++s) {
        ptx::mbar_init(&full[s], a_arrivals + 1);
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(tmem_full, 1);
      ptx::fence_barrier_init();
      ptx::tma_prefetch_desc(&args.tmap_b);
      if (MODE == static_cast<int>(ConvLoadMode::kTmaA)) ptx::tma_prefetch_desc(&args.tmap_a);
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_slot, args.tmem_cols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;

  if (warp < 4) {
    if constexpr (MODE == static_cast<int>(ConvLoadMode::kGather16)) {
      gather_a_tiles<8>(args, smem + L.a_off, full, empty, m0);
    } else if constexpr (MODE == static_cast<int>(ConvLoadMode::kGather8)) {
      gather_a_tiles<4>(args, smem + L.a_off, full, empty, m0);
    }
    // Epilogue: this warp owns TMEM lanes [32*warp, 32*warp + 32).
    ptx::mbar_wait(tmem_full, 0);
    ptx::tc_fence_after();
    const int m = m0 + threadIdx.x;
    const uint32_t t_row = tmem_d + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c0 = 0; c0 < args.BN; c0 += 16) {
      uint32_t raw[16];
      ptx::tmem_ld_32x32b_x16(t_row + c0, raw);
      ptx::tmem_ld_wait();
      if (m < args.M && n0 + c0 < args.Cout) epilogue_chunk(args, m, n0 + c0, raw);
    }
  } else if (warp == 4) {
    if (lane == 0) {
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      const uint32_t tx = b_bytes + (MODE == static_cast<int>(ConvLoadMode::kTmaA) ? kABytes : 0);
      for (int kb = 0; kb < args.num_kb; ++kb) {
        const int s = kb % args.stages;
        if (kb >= args.stages) ptx::mbar_wait(&empty[s], ((kb / args.stages) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&full[s], tx);
        ptx::tma_load_2d(ptx::smem_u32(smem + L.b_off + s * b_bytes), &args.tmap_b, &full[s],
                         kb * kConvBK, n0);
        if constexpr (MODE == static_cast<int>(ConvLoadMode::kTmaA)) {
          ptx::tma_load_2d(ptx::smem_u32(smem + L.a_off + s * kABytes), &args.tmap_a, &full[s],
                           kb * kConvBK, m0);
        }
      }
    }
  } else {  // warp 5: MMA issuer
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(kConvBM, args.BN);
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      for (int kb = 0; kb < args.num_kb; ++kb) {
        const int s = kb % args.stages;
        ptx::mbar_wait(&full[s], (kb / args.stages) & 1);
        ptx::tc_fence_after();
        if constexpr (MODE != static_cast<int>(ConvLoadMode::kTmaA)) ptx::fence_proxy_async_smem();
        const uint64_t da = ptx::umma_desc_sw128_kmajor(ptx::smem_u32(smem + L.a_off + s * kABytes));
        const uint64_t db = ptx::umma_desc_sw128_kmajor(ptx::smem_u32(smem + L.b_off + s * b_bytes));
#pragma unroll
        for (int k = 0; k < kConvBK / 16; ++k) {
          // +32 B along K inside the swizzle row = +2 in the >>4 start field.
          ptx::umma_bf16(tmem_d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
        }
        ptx::umma_commit(&empty[s]);
      }
      ptx::umma_commit(tmem_full);
    }
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_d, args.tmem_cols);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

}  // namespace

bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint64_t row_stride_elems, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kConvBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t conv_gemm_smem_bytes(int BN, int stages) {
  return smem_layout(BN, stages).total + 1024;  // + alignment slack
}

cudaError_t conv_gemm_init() {
  // Opt every instantiation into the full 227 KiB of dynamic shared memory
  // once, outside any stream capture.
  static cudaError_t status = [] {
    const int cap = 227 * 1024;
    cudaError_t e = cudaFuncSetAttribute(conv_gemm_kernel<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(conv_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               cap);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(conv_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               cap);
    return e;
  }();
  return status;
}

cudaError_t launch_conv_gemm(const ConvGemmArgs& args, ConvLoadMode mode, cudaStream_t stream) {
  const size_t smem = conv_gemm_smem_bytes(args.BN, args.stages);
  const dim3 grid((args.Cout + args.BN - 1) / args.BN, (args.M + kConvBM - 1) / kConvBM);
  switch (mode) {
    case ConvLoadMode::kGather16:
      conv_gemm_kernel<0><<<grid, kConvThreads, smem, stream>>>(args);
      break;
    case ConvLoadMode::kGather8:
      conv_gemm_kernel<1><<<grid, kConvThreads, smem, stream>>>(args);
      break;
    case ConvLoadMode::kTmaA:
      conv_gemm_kernel<2><<<grid, kConvThreads, smem, stream>>>(args);
      break;
  }
  return cudaGetLastError();
}

}  // namespace ds
