// Standalone bring-up check for the tcgen05 implicit-GEMM conv kernel:
// random bf16 data, several conv geometries / load modes, compared against a
// double-precision CPU loop over the same bf16 values. Dev tool only; the
// parity gate proper lives in tests/ (through the C-ABI).
#include "../paper_2308_13803_b200/csrc/kernels/conv_gemm.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

using namespace ds;

static float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

struct Case {
  const char* name;
  int N, H, W, C, R, S, sh, sw, ph, pw, Cout, BN;
  ConvLoadMode mode;
  bool residual, f32, relu;
  int ldy_extra, c_off;
};

static int run(const Case& cs) {
  const int Ho = (cs.H + 2 * cs.ph - cs.R) / cs.sh + 1;
  const int Wo = (cs.W + 2 * cs.pw - cs.S) / cs.sw + 1;
  const int M = cs.N * Ho * Wo;
  const int K = cs.R * cs.S * cs.C;
  const int Kpad = (K + 63) / 64 * 64;
  const int ldy = cs.Cout + cs.ldy_extra;
  std::mt19937 rng(1234);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<__nv_bfloat16> hx((size_t)cs.N * cs.H * cs.W * cs.C), hw((size_t)cs.Cout * Kpad),
      hr((size_t)M * cs.Cout);
  std::vector<float> fx(hx.size()), fw(hw.size(), 0.f), fr(hr.size()), hb(cs.Cout);
  for (size_t i = 0; i < hx.size(); ++i) { fx[i] = bf(nd(rng)); hx[i] = __float2bfloat16_rn(fx[i]); }
  for (int n = 0; n < cs.Cout; ++n)
    for (int k = 0; k < Kpad; ++k) {
      float v = k < K ? bf(nd(rng) * 0.05f) : 0.f;
      fw[(size_t)n * Kpad + k] = v;
      hw[(size_t)n * Kpad + k] = __float2bfloat16_rn(v);
    }
  for (size_t i = 0; i < hr.size(); ++i) { fr[i] = bf(nd(rng)); hr[i] = __float2bfloat16_rn(fr[i]); }
  for (int n = 0; n < cs.Cout; ++n) hb[n] = nd(rng) * 0.1f;

  __nv_bfloat16 *dx, *dw, *dr;
  float* db;
  void* dy;
  const size_t ybytes = (size_t)M * ldy * (cs.f32 ? 4 : 2);
  cudaMalloc(&dx, hx.size() * 2 + 4096);
  cudaMalloc(&dw, hw.size() * 2);
  cudaMalloc(&dr, hr.size() * 2);
  cudaMalloc(&db, hb.size() * 4);
  cudaMalloc(&dy, ybytes);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, hr.data(), hr.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dy, 0xFF, ybytes);  // NaN-fill so unwritten outputs are caught

  ConvGemmArgs a{};
  a.cluster = 1;
  ConvLoadMode mode = cs.mode;
  Case cs_bn = cs;  // BN=<n> overrides the case's N tile (A/B experiments)
  if (getenv("BN")) cs_bn.BN = atoi(getenv("BN"));
  const Case& cs2 = cs_bn;
#define cs cs2
  if (getenv("I2C") && cs.mode == ConvLoadMode::kGather16 && cs.C % 64 == 0) mode = ConvLoadMode::kIm2col;
  if (getenv("PAIR") && mode == ConvLoadMode::kTmaA) {  // cta_group::2 pair MMAs
    mode = ConvLoadMode::kPairTmaA;
    a.cluster = 2;
  }
  if (getenv("PAIR") && mode == ConvLoadMode::kGather16) {
    mode = ConvLoadMode::kPairGather;
    a.cluster = 2;
  }
  if (getenv("PAIR") && mode == ConvLoadMode::kIm2col) {
    mode = ConvLoadMode::kPairIm2col;
    a.cluster = 2;
  }
  if ((mode == ConvLoadMode::kIm2col || mode == ConvLoadMode::kPairIm2col) &&
      !encode_tmap_im2col(&a.tmap_a, dx, cs.N, cs.H, cs.W, cs.C, cs.R, cs.S, cs.sh, cs.sw, cs.ph, cs.pw)) {
    printf("%s: im2col map encode failed\n", cs.name);
    return 1;
  }
  if (!encode_tmap_2d_bf16(&a.tmap_b, dw, cs.Cout, Kpad, Kpad,
                           cs.BN / a.cluster)) {
    printf("%s: tmap_b encode failed\n", cs.name);
    return 1;
  }
  if (cs.mode == ConvLoadMode::kTmaA &&
      !encode_tmap_2d_bf16(&a.tmap_a, dx, M, cs.C, cs.C, kConvBM)) {
    printf("%s: tmap_a encode failed\n", cs.name);
    return 1;
  }
  a.x = dx; a.H = cs.H; a.W = cs.W; a.C = cs.C; a.R = cs.R; a.S = cs.S;
  a.stride_h = cs.sh; a.stride_w = cs.sw; a.pad_h = cs.ph; a.pad_w = cs.pw;
  a.Ho = Ho; a.Wo = Wo; a.M = M; a.num_kb = Kpad / 64; a.taps = cs.R * cs.S;
  a.Cout = cs.Cout; a.BN = cs.BN;
  a.stages = conv_gemm_stages(cs.BN, cs.Cout);
  a.tmem_cols = conv_gemm_tmem_cols(cs.BN);
  a.y_tma = encode_tmap_out(&a.tmap_y, static_cast<uint8_t*>(dy) + cs.c_off * (cs.f32 ? 4 : 2), M,
                            cs.Cout, ldy, cs.f32) ? 1 : 0;
  if (getenv("WIN") && cs.sh == 1 && cs.sw == 1 && cs.R * cs.S > 1 && !cs.f32) {
    // kWindow as the engine sets it up (engine.cu): 16 x 8 pixel blocks, one
    // halo box per 64-channel K block, 4-D TMA-store epilogue
    mode = ConvLoadMode::kWindow;
    a.dw_th = 16; a.dw_tw = 8; a.dw_rw = 4;
    a.dw_tiles_y = (Ho + 15) / 16; a.dw_tiles_x = (Wo + 7) / 8;
    a.win_iw = 8 + cs.S - 1; a.win_ih = 16 + cs.R - 1;
    const int cb = cs.C < 64 ? cs.C : 64;
    a.win_box_bytes = static_cast<uint32_t>(a.win_iw * a.win_ih * cb * 2);
    a.win_direct = cs.C % 64 == 0 ? 1 : 0;
    if (!encode_tmap_nhwc(&a.tmap_a, dx, cs.N, cs.H, cs.W, cs.C, cb, a.win_iw, a.win_ih, 1,
                          a.win_direct != 0) ||
        !encode_tmap_out4d(&a.tmap_y, static_cast<uint8_t*>(dy) + cs.c_off * 2, cs.N, Ho, Wo, cs.Cout,
                           ldy, a.dw_tw, a.dw_rw)) {
      printf("%s: window maps failed\n", cs.name);
      return 1;
    }
    a.y_tma = 1;
  }
  if (getenv("NO_TMA_STORE")) a.y_tma = 0;
  if (getenv("STAGES")) a.stages = atoi(getenv("STAGES"));
  if (getenv("DEBUG_FLAGS")) a.debug_flags = atoi(getenv("DEBUG_FLAGS"));
  if (getenv("TMEM_COLS")) a.tmem_cols = atoi(getenv("TMEM_COLS"));  // 512 forces 1 CTA/SM
#undef cs
  a.bias = db; a.residual = cs.residual ? dr : nullptr; a.ld_res = cs.Cout;
  a.y = dy; a.ldy = ldy; a.c_off = cs.c_off; a.out_f32 = cs.f32; a.relu = cs.relu;
  // channels [c_off, c_off+Cout) of an ldy-wide buffer; keep Cout+c_off <= ldy
  conv_gemm_init();
  cudaError_t e = launch_conv_gemm(a, mode, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: CUDA error %s\n", cs.name, cudaGetErrorString(e));
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) launch_conv_gemm(a, mode, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  ms /= 20;

  if (getenv("TS")) {  // per-CTA timelines of launches 2 and 3 of 3 back to back (globaltimer)
    const int nct = 148 * 2;
    unsigned long long* dts[2];
    for (auto& d : dts) {
      cudaMalloc(&d, nct * 64 * 8);
      cudaMemset(d, 0, nct * 64 * 8);
    }
    launch_conv_gemm(a, mode, 0);
    for (int i = 0; i < 2; ++i) {
      a.ts = dts[i];
      launch_conv_gemm(a, mode, 0);
    }
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h[2];
    for (int i = 0; i < 2; ++i) {
      h[i].resize(nct * 64);
      cudaMemcpy(h[i].data(), dts[i], h[i].size() * 8, cudaMemcpyDeviceToHost);
      cudaFree(dts[i]);
    }
    a.ts = nullptr;
    unsigned long long t0 = ~0ull;  // earliest entry of launch 3
    for (int c = 0; c < nct; ++c)
      if (h[1][c * 64 + 4]) t0 = std::min(t0, h[1][c * 64 + 4]);
    auto stat = [&](int l, int k, const char* name) {
      std::vector<double> v;
      for (int c = 0; c < nct; ++c)
        if (h[l][c * 64 + k]) v.push_back((static_cast<double>(h[l][c * 64 + k]) - t0) * 1e-3);
      if (v.empty()) return;
      std::sort(v.begin(), v.end());
      printf("  %-26s n=%3zu  min %7.2f  med %7.2f  max %7.2f us\n", name, v.size(), v[0],
             v[v.size() / 2], v.back());
    };
    printf("  timeline (us from launch 3's first CTA entry)\n");
    stat(0, 2, "L2 MMA loop done");
    stat(0, 3, "L2 exit barrier");
    stat(1, 4, "entry");
    stat(1, 5, "prologue done");
    stat(1, 1, "pdl_wait done");
    for (int j = 0; j < 8; ++j) {
      char nm[64];
      snprintf(nm, sizeof nm, "tile%d TMA issue", j); stat(1, 40 + j, nm);
      snprintf(nm, sizeof nm, "tile%d MMA first", j); stat(1, 8 + j, nm);
      snprintf(nm, sizeof nm, "tile%d MMA commit", j); stat(1, 16 + j, nm);
      snprintf(nm, sizeof nm, "tile%d epi start", j); stat(1, 24 + j, nm);
      snprintf(nm, sizeof nm, "tile%d halo0 done", j); stat(1, 48 + j, nm);
      snprintf(nm, sizeof nm, "tile%d epi end", j); stat(1, 32 + j, nm);
    }
    stat(1, 2, "MMA loop done");
    stat(1, 3, "exit barrier");
  }

  if (getenv("NOCHECK")) {
    const double flops = 2.0 * M * cs.Cout * K;
    printf("%-28s M=%7d N=%5d K=%5d  mode %d  %.3f us  %.1f TFLOP/s (unchecked)\n", cs.name, M, cs.Cout, K,
           static_cast<int>(mode), ms * 1e3, flops / (ms * 1e-3) / 1e12);
    cudaFree(dx); cudaFree(dw); cudaFree(dr); cudaFree(db); cudaFree(dy);
    return 0;
  }
  std::vector<uint8_t> hy(ybytes);
  cudaMemcpy(hy.data(), dy, ybytes, cudaMemcpyDeviceToHost);
  double max_err = 0, max_ref = 0;
  long bad = 0;
  for (int m = 0; m < M; ++m) {
    const int n_img = m / (Ho * Wo), rem = m % (Ho * Wo), ho = rem / Wo, wo = rem % Wo;
    for (int co = 0; co < cs.Cout; ++co) {
      double acc = hb[co];
      for (int r = 0; r < cs.R; ++r)
        for (int s = 0; s < cs.S; ++s) {
          const int hi = ho * cs.sh - cs.ph + r, wi = wo * cs.sw - cs.pw + s;
          if (hi < 0 || hi >= cs.H || wi < 0 || wi >= cs.W) continue;
          const float* xp = &fx[(((size_t)n_img * cs.H + hi) * cs.W + wi) * cs.C];
          const float* wp = &fw[(size_t)co * Kpad + (r * cs.S + s) * cs.C];
          for (int c = 0; c < cs.C; ++c) acc += (double)xp[c] * wp[c];
        }
      if (cs.residual) acc += fr[(size_t)m * cs.Cout + co];
      if (cs.relu && acc < 0) acc = 0;
      const size_t o = (size_t)m * ldy + cs.c_off + co;
      double got = cs.f32 ? ((float*)hy.data())[o]
                          : __bfloat162float(((__nv_bfloat16*)hy.data())[o]);
      double err = std::fabs(got - acc);
      if (!(err <= 0.02 + 0.01 * std::fabs(acc))) ++bad;
      if (!(err <= max_err)) max_err = err;
      if (std::fabs(acc) > max_ref) max_ref = std::fabs(acc);
    }
  }
  const double flops = 2.0 * M * cs.Cout * K;
  printf("%-28s M=%7d N=%5d K=%5d  max_err=%.4g (max|ref| %.3g) bad=%ld  %.3f us  %.1f TFLOP/s\n",
         cs.name, M, cs.Cout, K, max_err, max_ref, bad, ms * 1e3, flops / (ms * 1e-3) / 1e12);
  cudaFree(dx); cudaFree(dw); cudaFree(dr); cudaFree(db); cudaFree(dy);
  return bad ? 1 : 0;
}

int main(int argc, char** argv) {
  const Case cases[] = {
      {"tiny 1x1 (fixed cost)", 1, 8, 16, 64, 1, 1, 1, 1, 0, 0, 64, 64, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"1x1 s1 tmaA", 2, 14, 14, 256, 1, 1, 1, 1, 0, 0, 512, 128, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"1x1 s1 gather", 2, 14, 14, 256, 1, 1, 1, 1, 0, 0, 512, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"3x3 s1 p1", 1, 28, 28, 128, 3, 3, 1, 1, 1, 1, 128, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"3x3 s2 p1 N96", 2, 28, 28, 64, 3, 3, 2, 2, 1, 1, 96, 96, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"1x7 p(0,3) N160", 2, 17, 17, 128, 1, 7, 1, 1, 0, 3, 160, 160, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"fc 2048->1000 f32", 3, 1, 1, 2048, 1, 1, 1, 1, 0, 0, 1000, 256, ConvLoadMode::kTmaA, false, true, false, 0, 0},
      {"1x1 residual+slice", 2, 7, 7, 512, 1, 1, 1, 1, 0, 0, 256, 128, ConvLoadMode::kTmaA, true, false, true, 64, 32},
      {"3x3 C80 N192", 1, 20, 20, 80, 3, 3, 1, 1, 0, 0, 192, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"1x1 7x7 2048 Mtail", 1, 7, 7, 512, 1, 1, 1, 1, 0, 0, 2048, 256, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"fc 10 classes", 5, 1, 1, 128, 1, 1, 1, 1, 0, 0, 10, 16, ConvLoadMode::kTmaA, false, true, false, 0, 0},
      {"big 1x1 s1", 64, 56, 56, 64, 1, 1, 1, 1, 0, 0, 256, 256, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"big 3x3 256", 32, 14, 14, 256, 3, 3, 1, 1, 1, 1, 256, 256, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"mbv1 pw1 bs128", 128, 112, 112, 32, 1, 1, 1, 1, 0, 0, 64, 64, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"mbv1 pw1g bs128", 128, 112, 112, 32, 1, 1, 1, 1, 0, 0, 64, 64, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"tmaA C32 small", 3, 5, 7, 32, 1, 1, 1, 1, 0, 0, 48, 48, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"mbv1 pw2 bs128", 128, 56, 56, 64, 1, 1, 1, 1, 0, 0, 128, 128, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"mbv1 pw7 bs128", 128, 14, 14, 512, 1, 1, 1, 1, 0, 0, 512, 256, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"mbv1 pw5 bs128", 128, 28, 28, 256, 1, 1, 1, 1, 0, 0, 256, 256, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"mbv1 fc bs128", 128, 1, 1, 1024, 1, 1, 1, 1, 0, 0, 1000, 64, ConvLoadMode::kTmaA, false, true, false, 0, 0},
      {"rn 28 3x3 bs256", 256, 28, 28, 128, 3, 3, 1, 1, 1, 1, 128, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"rn 14 3x3 bs256", 256, 14, 14, 256, 3, 3, 1, 1, 1, 1, 256, 256, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"rn 7 3x3 bs256", 256, 7, 7, 512, 3, 3, 1, 1, 1, 1, 512, 256, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"rn 56 1x1s2 bs256", 256, 56, 56, 256, 1, 1, 2, 2, 0, 0, 128, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 17 1x7 c128 bs128", 128, 17, 17, 128, 1, 7, 1, 1, 0, 3, 128, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 17 7x1 c192 bs128", 128, 17, 17, 192, 7, 1, 1, 1, 3, 0, 192, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 8 3x3 c448 bs128", 128, 8, 8, 448, 3, 3, 1, 1, 1, 1, 384, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 8 1x3 c384 bs128", 128, 8, 8, 384, 1, 3, 1, 1, 0, 1, 384, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 35 5x5 c48 bs128", 128, 35, 35, 48, 5, 5, 1, 1, 2, 2, 64, 64, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 35 3x3 c96 bs128", 128, 35, 35, 96, 3, 3, 1, 1, 1, 1, 96, 96, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 35 3x3 c64 bs128", 128, 35, 35, 64, 3, 3, 1, 1, 1, 1, 96, 96, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"in 35 3x3 c64 n64 bs128", 128, 35, 35, 64, 3, 3, 1, 1, 1, 1, 64, 64, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"rn 56 3x3 bs256", 256, 56, 56, 64, 3, 3, 1, 1, 1, 1, 64, 64, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"rn 56 1x1 64-320 bs256", 256, 56, 56, 64, 1, 1, 1, 1, 0, 0, 320, 192, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"rn 56 1x1 64-256 res bs256", 256, 56, 56, 64, 1, 1, 1, 1, 0, 0, 256, 256, ConvLoadMode::kTmaA, true, false, true, 0, 0},
      {"rn 28 1x1 128-512 res bs256", 256, 28, 28, 128, 1, 1, 1, 1, 0, 0, 512, 256, ConvLoadMode::kTmaA, true, false, true, 0, 0},
      {"rn 14 1x1 256-1024 res bs256", 256, 14, 14, 256, 1, 1, 1, 1, 0, 0, 1024, 256, ConvLoadMode::kTmaA, true, false, true, 0, 0},
      {"rn 7 1x1 512-2048 res bs256", 256, 7, 7, 512, 1, 1, 1, 1, 0, 0, 2048, 256, ConvLoadMode::kTmaA, true, false, true, 0, 0},
      {"rn 28 1x1 512-128 bs256", 256, 28, 28, 512, 1, 1, 1, 1, 0, 0, 128, 128, ConvLoadMode::kTmaA, false, false, true, 0, 0},
      {"small 5x5 c48 chk", 2, 11, 9, 48, 5, 5, 1, 1, 2, 2, 64, 64, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"small 3x3 c128 chk", 3, 10, 12, 128, 3, 3, 1, 1, 1, 1, 128, 128, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"small 3x3s2 c64 chk", 3, 15, 13, 64, 3, 3, 2, 2, 1, 1, 192, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"small 1x7 c192 chk", 2, 17, 17, 192, 1, 7, 1, 1, 0, 3, 192, 192, ConvLoadMode::kGather16, false, false, true, 0, 0},
      {"mbv1 pw4 bs128", 128, 28, 28, 128, 1, 1, 1, 1, 0, 0, 256, 256, ConvLoadMode::kTmaA, false, false, true, 0, 0},
  };
  // Optional filter: substring of the case name; "--no-check" skips the CPU reference.
  const char* only = argc > 1 ? argv[1] : nullptr;
  int fails = 0;
  for (const auto& c : cases)
    if (!only || std::strstr(c.name, only)) fails += run(c);
  printf("%s (%d failing cases)\n", fails ? "FAIL" : "PASS", fails);
  return fails ? 1 : 0;
}
