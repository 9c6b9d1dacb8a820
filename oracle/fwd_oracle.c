/*
 * FP32 CPU forward-pass oracle — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * leg may load this library, and only as the checker / CPU baseline. The
 * product path (paper_2308_13803_b200/) never links or calls it.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference repository has no forward
 * pass at all — its "GPU" returns a + b*bs milliseconds (reference
 * proj/core/src/perf_model.cpp:70-86) — so no reference test, fixture or
 * golden vector pins any logit. This file is an independent restatement of
 * the canonical architectures (MobileNet-v1 1.0/224, ResNet-50 v1 (stride on
 * the first 1x1), Inception-v3/299 without aux head, and the synthetic CNN of
 * config 1), written without reading the product code, and is cross-checked
 * against torch.nn.functional on CPU by tests/golden/make_golden.py.
 *
 * What IS pinned to the reference: the generator. Weights and images come
 * from the reference's RandomStream / mix_seed (proj/core/include/dnnscaler/
 * random.hpp:10-47: mt19937_64, (x>>11)*2^-53 uniform, Box-Muller with a
 * cached spare), restated here in C including mt19937_64 itself.
 *
 * Conventions:
 *   layer l (emission order below) draws from RandomStream(mix_seed(42, 1000+l));
 *   conv/fc weights drawn co-major then (r, s, c) over real input channels,
 *   w = bf16_rne((float)(z * sd * gain)); then one bias per channel
 *   (float)(0.1 z) (FC: bias 0, no draws); sd = sqrt(2/fan_in) (FC sqrt(1/fan_in));
 *   depthwise: per channel 9 taps, sd = sqrt(2/9).
 *   image i: RandomStream(mix_seed(seed, 1000000+i)); a textured image (img_one:
 *   base colour + three triangle gratings + per-pixel noise, integer math);
 *   x = bf16_rne((p - 127.5f) / 63.75f).
 *
 * bf16_storage = 1 rounds every stored activation to bf16 exactly where the
 * device stores bf16 (all layer outputs and the pooled features); 0 keeps
 * everything fp32 after the bf16 input/weights.
 */
#include <math.h>
#include <stdio.h>
#include <pthread.h>
#include <unistd.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ----------------------------------------------------------- mt19937_64 */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* reference random.hpp:10-15 */
static uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

typedef struct {
  mt64 g;
  int has_spare;
  double spare;
} rstream;

static void rs_init(rstream* r, uint64_t seed) {
  mt64_seed(&r->g, seed);
  r->has_spare = 0;
  r->spare = 0.0;
}

/* reference random.hpp:22 */
static double rs_uniform(rstream* r) { return (double)(mt64_next(&r->g) >> 11) * 0x1.0p-53; }

/* reference random.hpp:26-38 */
static double rs_gaussian(rstream* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = rs_uniform(r);
  while (u1 <= 0.0) u1 = rs_uniform(r);
  double u2 = rs_uniform(r);
  double rad = sqrt(-2.0 * log(u1));
  const double pi = 3.14159265358979323846;
  r->spare = rad * sin(2.0 * pi * u2);
  r->has_spare = 1;
  return rad * cos(2.0 * pi * u2);
}

static uint16_t bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return 0x7FC0;
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

static float bf16_round(float f) {
  uint32_t u = (uint32_t)bf16_bits(f) << 16;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

/* ----------------------------------------------------------- threads */
typedef void (*range_fn)(void* ctx, int i);
typedef struct {
  range_fn fn;
  void* ctx;
  int count;
  int next; /* guarded by mu */
  pthread_mutex_t mu;
} pf_job;

static void* pf_worker(void* arg) {
  pf_job* j = (pf_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->count) return NULL;
    j->fn(j->ctx, i);
  }
}

static int g_threads = 0; /* 0: all online cores */

void oracle_set_threads(int n) { g_threads = n; }

int oracle_get_threads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* Dynamic parallel-for over [0, count) on oracle_get_threads() threads. */
static void parallel_for(int count, range_fn fn, void* ctx) {
  int nt = oracle_get_threads();
  if (nt > count) nt = count;
  if (nt <= 1) {
    for (int i = 0; i < count; ++i) fn(ctx, i);
    return;
  }
  pf_job j;
  j.fn = fn;
  j.ctx = ctx;
  j.count = count;
  j.next = 0;
  pthread_mutex_init(&j.mu, NULL);
  pthread_t th[256];
  if (nt > 256) nt = 256;
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, pf_worker, &j);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&j.mu);
}

/* ----------------------------------------------------------- model IR */
enum { K_CONV, K_DW, K_MAXPOOL, K_AVGPOOL, K_GAP, K_FC };

typedef struct {
  int h, w, c;
} shape;

typedef struct {
  int kind;
  int in, out, c_off, res;
  int kh, kw, sh, sw, ph, pw, relu;
  int cin, cout; /* conv: real input channels, output channels */
  float gain;
  float* wt; /* conv/fc: [kh*kw*cin][cout]; dw: [9][c] */
  float* bias;
} op;

typedef struct {
  const char* id;
  int in_h, in_w, classes;
  int nb, nops;
  shape buf[160];
  op ops[160];
  int logits;
} net;

static int nbuf(net* n, int h, int w, int c) {
  n->buf[n->nb].h = h;
  n->buf[n->nb].w = w;
  n->buf[n->nb].c = c;
  return n->nb++;
}

static op* nop(net* n, int kind) {
  op* o = &n->ops[n->nops++];
  memset(o, 0, sizeof(*o));
  o->kind = kind;
  o->res = -1;
  o->relu = 1;
  o->gain = 1.0f;
  return o;
}

/* conv with explicit geometry; out < 0 allocates; returns output buffer */
static int cv(net* n, int in, int cout, int kh, int kw, int sh, int sw, int ph, int pw, int out,
              int c_off) {
  shape s = n->buf[in];
  int ho = (s.h + 2 * ph - kh) / sh + 1, wo = (s.w + 2 * pw - kw) / sw + 1;
  if (out < 0) out = nbuf(n, ho, wo, cout);
  op* o = nop(n, K_CONV);
  o->in = in;
  o->out = out;
  o->c_off = c_off;
  o->kh = kh;
  o->kw = kw;
  o->sh = sh;
  o->sw = sw;
  o->ph = ph;
  o->pw = pw;
  o->cin = s.c;
  o->cout = cout;
  return out;
}

static int cvs(net* n, int in, int cout, int k, int st, int pad) {
  return cv(n, in, cout, k, k, st, st, pad, pad, -1, 0);
}

static int pool(net* n, int in, int is_max, int st, int pad, int out, int c_off) {
  shape s = n->buf[in];
  int ho = (s.h + 2 * pad - 3) / st + 1, wo = (s.w + 2 * pad - 3) / st + 1;
  if (out < 0) out = nbuf(n, ho, wo, s.c);
  op* o = nop(n, is_max ? K_MAXPOOL : K_AVGPOOL);
  o->in = in;
  o->out = out;
  o->c_off = c_off;
  o->sh = o->sw = st;
  o->ph = o->pw = pad;
  o->relu = 0;
  return out;
}

static void head(net* n, int x, int classes) {
  shape s = n->buf[x];
  int g = nbuf(n, 1, 1, s.c);
  op* o = nop(n, K_GAP);
  o->in = x;
  o->out = g;
  o->relu = 0;
  int lg = nbuf(n, 1, 1, classes);
  o = nop(n, K_FC);
  o->in = g;
  o->out = lg;
  o->cin = s.c;
  o->cout = classes;
  o->kh = o->kw = 1;
  o->relu = 0;
  n->logits = lg;
  n->classes = classes;
}

static void build_synthetic(net* n) {
  n->in_h = n->in_w = 32;
  int x = nbuf(n, 32, 32, 3);
  x = cvs(n, x, 32, 3, 1, 1);
  x = cvs(n, x, 64, 3, 2, 1);
  x = cvs(n, x, 128, 3, 2, 1);
  head(n, x, 10);
}

static void build_mobilenet(net* n) {
  static const int pw_ch[13] = {64, 128, 128, 256, 256, 512, 512, 512, 512, 512, 512, 1024, 1024};
  static const int dw_st[13] = {1, 2, 1, 2, 1, 2, 1, 1, 1, 1, 1, 2, 1};
  n->in_h = n->in_w = 224;
  int x = nbuf(n, 224, 224, 3);
  x = cvs(n, x, 32, 3, 2, 1);
  for (int i = 0; i < 13; ++i) {
    shape s = n->buf[x];
    int ho = (s.h - 1) / dw_st[i] + 1, wo = (s.w - 1) / dw_st[i] + 1;
    int y = nbuf(n, ho, wo, s.c);
    op* o = nop(n, K_DW);
    o->in = x;
    o->out = y;
    o->sh = o->sw = dw_st[i];
    o->ph = o->pw = 1;
    o->kh = o->kw = 3;
    o->cin = 1;
    o->cout = s.c;
    x = cvs(n, y, pw_ch[i], 1, 1, 0);
  }
  head(n, x, 1000);
}

static void build_resnet50(net* n) {
  static const int nblk[4] = {3, 4, 6, 3}, width[4] = {64, 128, 256, 512};
  n->in_h = n->in_w = 224;
  int x = nbuf(n, 224, 224, 3);
  x = cvs(n, x, 64, 7, 2, 3);
  x = pool(n, x, 1, 2, 1, -1, 0);
  for (int st = 0; st < 4; ++st) {
    for (int b = 0; b < nblk[st]; ++b) {
      int stride = (b == 0 && st > 0) ? 2 : 1, w = width[st];
      int in = x;
      int y = cv(n, in, w, 1, 1, stride, stride, 0, 0, -1, 0); /* v1: stride on 1x1 */
      y = cvs(n, y, w, 3, 1, 1);
      int sc = in;
      if (b == 0) {
        sc = cv(n, in, 4 * w, 1, 1, stride, stride, 0, 0, -1, 0);
        n->ops[n->nops - 1].relu = 0;
      }
      x = cv(n, y, 4 * w, 1, 1, 1, 1, 0, 0, -1, 0);
      n->ops[n->nops - 1].res = sc;
      n->ops[n->nops - 1].gain = 0.5f;
    }
  }
  head(n, x, 1000);
}

static int inc_a(net* n, int x, int pf) {
  shape s = n->buf[x];
  int out = nbuf(n, s.h, s.w, 224 + pf);
  cv(n, x, 64, 1, 1, 1, 1, 0, 0, out, 0);
  int t = cvs(n, x, 48, 1, 1, 0);
  cv(n, t, 64, 5, 5, 1, 1, 2, 2, out, 64);
  t = cvs(n, x, 64, 1, 1, 0);
  t = cvs(n, t, 96, 3, 1, 1);
  cv(n, t, 96, 3, 3, 1, 1, 1, 1, out, 128);
  t = pool(n, x, 0, 1, 1, -1, 0);
  cv(n, t, pf, 1, 1, 1, 1, 0, 0, out, 224);
  return out;
}

static int inc_b(net* n, int x) {
  shape s = n->buf[x];
  int out = nbuf(n, (s.h - 3) / 2 + 1, (s.w - 3) / 2 + 1, 480 + s.c);
  cv(n, x, 384, 3, 3, 2, 2, 0, 0, out, 0);
  int t = cvs(n, x, 64, 1, 1, 0);
  t = cvs(n, t, 96, 3, 1, 1);
  cv(n, t, 96, 3, 3, 2, 2, 0, 0, out, 384);
  pool(n, x, 1, 2, 0, out, 480);
  return out;
}

static int inc_c(net* n, int x, int c7) {
  shape s = n->buf[x];
  int out = nbuf(n, s.h, s.w, 768);
  cv(n, x, 192, 1, 1, 1, 1, 0, 0, out, 0);
  int t = cvs(n, x, c7, 1, 1, 0);
  t = cv(n, t, c7, 1, 7, 1, 1, 0, 3, -1, 0);
  cv(n, t, 192, 7, 1, 1, 1, 3, 0, out, 192);
  t = cvs(n, x, c7, 1, 1, 0);
  t = cv(n, t, c7, 7, 1, 1, 1, 3, 0, -1, 0);
  t = cv(n, t, c7, 1, 7, 1, 1, 0, 3, -1, 0);
  t = cv(n, t, c7, 7, 1, 1, 1, 3, 0, -1, 0);
  cv(n, t, 192, 1, 7, 1, 1, 0, 3, out, 384);
  t = pool(n, x, 0, 1, 1, -1, 0);
  cv(n, t, 192, 1, 1, 1, 1, 0, 0, out, 576);
  return out;
}

static int inc_d(net* n, int x) {
  shape s = n->buf[x];
  int out = nbuf(n, (s.h - 3) / 2 + 1, (s.w - 3) / 2 + 1, 512 + s.c);
  int t = cvs(n, x, 192, 1, 1, 0);
  cv(n, t, 320, 3, 3, 2, 2, 0, 0, out, 0);
  t = cvs(n, x, 192, 1, 1, 0);
  t = cv(n, t, 192, 1, 7, 1, 1, 0, 3, -1, 0);
  t = cv(n, t, 192, 7, 1, 1, 1, 3, 0, -1, 0);
  cv(n, t, 192, 3, 3, 2, 2, 0, 0, out, 320);
  pool(n, x, 1, 2, 0, out, 512);
  return out;
}

static int inc_e(net* n, int x) {
  shape s = n->buf[x];
  int out = nbuf(n, s.h, s.w, 2048);
  cv(n, x, 320, 1, 1, 1, 1, 0, 0, out, 0);
  int t = cvs(n, x, 384, 1, 1, 0);
  cv(n, t, 384, 1, 3, 1, 1, 0, 1, out, 320);
  cv(n, t, 384, 3, 1, 1, 1, 1, 0, out, 704);
  t = cvs(n, x, 448, 1, 1, 0);
  t = cvs(n, t, 384, 3, 1, 1);
  cv(n, t, 384, 1, 3, 1, 1, 0, 1, out, 1088);
  cv(n, t, 384, 3, 1, 1, 1, 1, 0, out, 1472);
  t = pool(n, x, 0, 1, 1, -1, 0);
  cv(n, t, 192, 1, 1, 1, 1, 0, 0, out, 1856);
  return out;
}

static void build_inception(net* n) {
  n->in_h = n->in_w = 299;
  int x = nbuf(n, 299, 299, 3);
  x = cvs(n, x, 32, 3, 2, 0);
  x = cvs(n, x, 32, 3, 1, 0);
  x = cvs(n, x, 64, 3, 1, 1);
  x = pool(n, x, 1, 2, 0, -1, 0);
  x = cvs(n, x, 80, 1, 1, 0);
  x = cvs(n, x, 192, 3, 1, 0);
  x = pool(n, x, 1, 2, 0, -1, 0);
  x = inc_a(n, x, 32);
  x = inc_a(n, x, 64);
  x = inc_a(n, x, 64);
  x = inc_b(n, x);
  x = inc_c(n, x, 128);
  x = inc_c(n, x, 160);
  x = inc_c(n, x, 160);
  x = inc_c(n, x, 192);
  x = inc_d(n, x);
  x = inc_e(n, x);
  x = inc_e(n, x);
  head(n, x, 1000);
}

static int has_params(const op* o) { return o->kind == K_CONV || o->kind == K_DW || o->kind == K_FC; }

/* Calibrated classifier head (product synth.hpp HeadCalib):
 * <head_dir>/<id>.head = "DSHEAD1\0", int32 C, int32 k, f64 mu[C],
 * f64 scale[k], f64 v[k][C]. W[co][c] = bf16(sum_j (R[co][j] scale[j]) v[j][c])
 * with R drawn co-major from the FC layer's stream, b = -sum_c W mu. The
 * file is model data shared with the product (like trained weights); absent
 * file = plain random head. */
static char g_head_dir[1024] = "";

void oracle_set_head_dir(const char* dir) {
  strncpy(g_head_dir, dir ? dir : "", sizeof(g_head_dir) - 1);
}

static int gen_head(net* n, op* o, rstream* rs) {
  if (!g_head_dir[0]) return 0;
  char path[1200];
  snprintf(path, sizeof(path), "%s/%s.head", g_head_dir, n->id);
  FILE* f = fopen(path, "rb");
  if (!f) return 0;
  char magic[8];
  int32_t dims[2];
  if (fread(magic, 1, 8, f) != 8 || memcmp(magic, "DSHEAD1", 8) != 0 || fread(dims, 4, 2, f) != 2 ||
      dims[0] != o->cin || dims[1] <= 0 || dims[1] > dims[0]) {
    fclose(f);
    abort(); /* corrupt or mismatched calibration: never silently fall back */
  }
  const int C = dims[0], k = dims[1];
  double* mu = (double*)malloc(sizeof(double) * C);
  double* scale = (double*)malloc(sizeof(double) * k);
  double* v = (double*)malloc(sizeof(double) * (size_t)k * C);
  if (fread(mu, 8, C, f) != (size_t)C || fread(scale, 8, k, f) != (size_t)k ||
      fread(v, 8, (size_t)k * C, f) != (size_t)k * C)
    abort();
  fclose(f);
  double* r = (double*)malloc(sizeof(double) * (size_t)o->cout * k);
  for (size_t q = 0; q < (size_t)o->cout * k; ++q) r[q] = rs_gaussian(rs);
  o->wt = (float*)malloc(sizeof(float) * (size_t)C * o->cout);
  o->bias = (float*)malloc(sizeof(float) * o->cout);
  for (int co = 0; co < o->cout; ++co) {
    double bacc = 0.0;
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += (r[(size_t)co * k + j] * scale[j]) * v[(size_t)j * C + c];
      const float wv = bf16_round((float)acc);
      o->wt[(size_t)c * o->cout + co] = wv;
      bacc += (double)wv * mu[c];
    }
    o->bias[co] = (float)(-bacc);
  }
  free(mu); free(scale); free(v); free(r);
  return 1;
}

static void gen_weights(net* n) {
  int layer = 0;
  for (int i = 0; i < n->nops; ++i) {
    op* o = &n->ops[i];
    if (!has_params(o)) continue;
    rstream rs;
    rs_init(&rs, mix_seed(42, 1000 + (uint64_t)layer));
    ++layer;
    if (o->kind == K_DW) {
      int c = o->cout;
      o->wt = (float*)malloc(sizeof(float) * 9 * c);
      o->bias = (float*)malloc(sizeof(float) * c);
      double sd = sqrt(2.0 / 9.0);
      for (int ch = 0; ch < c; ++ch)
        for (int t = 0; t < 9; ++t) o->wt[t * c + ch] = bf16_round((float)(rs_gaussian(&rs) * sd));
      for (int ch = 0; ch < c; ++ch) o->bias[ch] = (float)(0.1 * rs_gaussian(&rs));
      continue;
    }
    int kk = o->kh * o->kw * o->cin;
    int fc = o->kind == K_FC;
    if (fc && gen_head(n, o, &rs)) continue;
    double sd = (fc ? sqrt(1.0 / kk) : sqrt(2.0 / kk)) * (double)o->gain;
    o->wt = (float*)malloc(sizeof(float) * (size_t)kk * o->cout);
    o->bias = (float*)malloc(sizeof(float) * o->cout);
    for (int co = 0; co < o->cout; ++co)
      for (int k = 0; k < kk; ++k) o->wt[(size_t)k * o->cout + co] = bf16_round((float)(rs_gaussian(&rs) * sd));
    for (int co = 0; co < o->cout; ++co) o->bias[co] = fc ? 0.0f : (float)(0.1 * rs_gaussian(&rs));
  }
}

static net* g_nets[4];
static const char* g_ids[4] = {"synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3"};

static net* get_net(const char* id) {
  int k = -1;
  for (int i = 0; i < 4; ++i)
    if (strcmp(id, g_ids[i]) == 0) k = i;
  if (k < 0) return NULL;
  if (!g_nets[k]) {
    net* n = (net*)calloc(1, sizeof(net));
    n->id = g_ids[k];
    if (k == 0) build_synthetic(n);
    if (k == 1) build_mobilenet(n);
    if (k == 2) build_resnet50(n);
    if (k == 3) build_inception(n);
    gen_weights(n);
    g_nets[k] = n;
  }
  return g_nets[k];
}

/* ----------------------------------------------------------- forward */
static void run_conv(const net* n, const op* o, float** B, int st) {
  shape si = n->buf[o->in], so = n->buf[o->out];
  const float* x = B[o->in];
  float* y = B[o->out];
  const int cout = o->cout, cin = o->cin;
  enum { T = 8 };
  float acc[T][2048];
  const int npix = so.h * so.w;
  for (int p0 = 0; p0 < npix; p0 += T) {
    int np = npix - p0 < T ? npix - p0 : T;
    for (int t = 0; t < np; ++t) memcpy(acc[t], o->bias, sizeof(float) * cout);
    for (int r = 0; r < o->kh; ++r)
      for (int s = 0; s < o->kw; ++s)
        for (int t = 0; t < np; ++t) {
          int p = p0 + t, oy = p / so.w, ox = p % so.w;
          int iy = oy * o->sh - o->ph + r, ix = ox * o->sw - o->pw + s;
          if (iy < 0 || iy >= si.h || ix < 0 || ix >= si.w) continue;
          const float* xp = x + ((size_t)iy * si.w + ix) * si.c;
          const float* wrow = o->wt + (size_t)((r * o->kw + s) * cin) * cout;
          float* a = acc[t];
          for (int c = 0; c < cin; ++c) {
            const float xv = xp[c];
            const float* wr = wrow + (size_t)c * cout;
            for (int co = 0; co < cout; ++co) a[co] += xv * wr[co];
          }
        }
    for (int t = 0; t < np; ++t) {
      float* a = acc[t];
      const size_t pix = (size_t)(p0 + t);
      if (o->res >= 0) {
        const float* rp = B[o->res] + pix * cout;
        for (int co = 0; co < cout; ++co) a[co] += rp[co];
      }
      float* yp = y + pix * so.c + o->c_off;
      for (int co = 0; co < cout; ++co) {
        float v = a[co];
        if (o->relu && v < 0.0f) v = 0.0f;
        yp[co] = st ? bf16_round(v) : v;
      }
    }
  }
}

static void run_dw(const net* n, const op* o, float** B, int st) {
  shape si = n->buf[o->in], so = n->buf[o->out];
  const int c = si.c;
  for (int oy = 0; oy < so.h; ++oy)
    for (int ox = 0; ox < so.w; ++ox) {
      float* yp = B[o->out] + ((size_t)oy * so.w + ox) * c;
      for (int ch = 0; ch < c; ++ch) {
        float a = o->bias[ch];
        for (int r = 0; r < 3; ++r)
          for (int s = 0; s < 3; ++s) {
            int iy = oy * o->sh - 1 + r, ix = ox * o->sw - 1 + s;
            if (iy < 0 || iy >= si.h || ix < 0 || ix >= si.w) continue;
            a += B[o->in][((size_t)iy * si.w + ix) * c + ch] * o->wt[(r * 3 + s) * c + ch];
          }
        if (a < 0.0f) a = 0.0f;
        yp[ch] = st ? bf16_round(a) : a;
      }
    }
}

static void run_pool(const net* n, const op* o, float** B, int st) {
  shape si = n->buf[o->in], so = n->buf[o->out];
  const int c = si.c, is_max = o->kind == K_MAXPOOL;
  for (int oy = 0; oy < so.h; ++oy)
    for (int ox = 0; ox < so.w; ++ox) {
      float* yp = B[o->out] + ((size_t)oy * so.w + ox) * so.c + o->c_off;
      for (int ch = 0; ch < c; ++ch) {
        float a = is_max ? -INFINITY : 0.0f;
        for (int r = 0; r < 3; ++r)
          for (int s = 0; s < 3; ++s) {
            int iy = oy * o->sh - o->ph + r, ix = ox * o->sw - o->pw + s;
            if (iy < 0 || iy >= si.h || ix < 0 || ix >= si.w) continue;
            float v = B[o->in][((size_t)iy * si.w + ix) * c + ch];
            a = is_max ? (v > a ? v : a) : a + v;
          }
        if (!is_max) a = a / 9.0f; /* count_include_pad */
        yp[ch] = st ? bf16_round(a) : a;
      }
    }
}

static float* g_feat_out = NULL; /* debug: pooled features of a single-image call */
void oracle_debug_features(float* out) { g_feat_out = out; }
static int g_dbg_buf = -1;       /* debug: capture this activation buffer ... */
static float* g_dbg_out = NULL;  /* ... into this array (single-image calls only) */

static void forward_one(const net* n, const uint8_t* img, int st, float* logits) {
  float* B[160];
  for (int b = 0; b < n->nb; ++b)
    B[b] = (float*)calloc((size_t)n->buf[b].h * n->buf[b].w * n->buf[b].c, sizeof(float));
  const size_t npx = (size_t)n->in_h * n->in_w * 3;
  for (size_t q = 0; q < npx; ++q) B[0][q] = bf16_round(((float)img[q] - 127.5f) / 63.75f);
  for (int i = 0; i < n->nops; ++i) {
    const op* o = &n->ops[i];
    switch (o->kind) {
      case K_CONV:
        run_conv(n, o, B, st);
        break;
      case K_DW:
        run_dw(n, o, B, st);
        break;
      case K_MAXPOOL:
      case K_AVGPOOL:
        run_pool(n, o, B, st);
        break;
      case K_GAP: {
        shape si = n->buf[o->in];
        const int hw = si.h * si.w;
        for (int ch = 0; ch < si.c; ++ch) {
          float a = 0.0f;
          for (int q = 0; q < hw; ++q) a += B[o->in][(size_t)q * si.c + ch];
          a = a / (float)hw;
          B[o->out][ch] = st ? bf16_round(a) : a;
        }
        break;
      }
      case K_FC: {
        const float* x = B[o->in];
        for (int co = 0; co < o->cout; ++co) {
          float a = o->bias[co];
          for (int c = 0; c < o->cin; ++c) a += x[c] * o->wt[(size_t)c * o->cout + co];
          B[o->out][co] = a;
        }
        break;
      }
    }
  }
  memcpy(logits, B[n->logits], sizeof(float) * n->classes);
  if (g_feat_out) memcpy(g_feat_out, B[n->ops[n->nops - 1].in], sizeof(float) * n->ops[n->nops - 1].cin);
  if (g_dbg_out && g_dbg_buf >= 0 && g_dbg_buf < n->nb)
    memcpy(g_dbg_out, B[g_dbg_buf],
           sizeof(float) * n->buf[g_dbg_buf].h * n->buf[g_dbg_buf].w * n->buf[g_dbg_buf].c);
  for (int b = 0; b < n->nb; ++b) free(B[b]);
}

/* ----------------------------------------------------------- C API */
/* Debug: one image through the net, activation buffer `buf` (NHWC fp32) out;
 * returns its element count, or -1. Buffer ids follow emission order. */
long oracle_debug_buffer(const char* id, const uint8_t* img, int bf16_storage, int buf,
                         float* out) {
  net* n = get_net(id);
  if (!n || buf < 0 || buf >= n->nb) return -1;
  long count = (long)n->buf[buf].h * n->buf[buf].w * n->buf[buf].c;
  if (out) {
    float* logits = (float*)malloc(sizeof(float) * n->classes);
    g_dbg_buf = buf;
    g_dbg_out = out;
    forward_one(n, img, bf16_storage, logits);
    g_dbg_out = NULL;
    g_dbg_buf = -1;
    free(logits);
  }
  return count;
}
int oracle_model_info(const char* id, int* in_h, int* in_w, int* classes, int* n_params,
                      double* macs) {
  net* n = get_net(id);
  if (!n) return 1;
  int np = 0;
  double m = 0.0;
  for (int i = 0; i < n->nops; ++i) {
    const op* o = &n->ops[i];
    if (has_params(o)) ++np;
    shape so = n->buf[o->out];
    if (o->kind == K_CONV) m += (double)so.h * so.w * o->cout * o->kh * o->kw * o->cin;
    if (o->kind == K_DW) m += (double)so.h * so.w * so.c * 9;
    if (o->kind == K_FC) m += (double)o->cout * o->cin;
  }
  if (in_h) *in_h = n->in_h;
  if (in_w) *in_w = n->in_w;
  if (classes) *classes = n->classes;
  if (n_params) *n_params = np;
  if (macs) *macs = m;
  return 0;
}

typedef struct {
  int h, w;
  uint64_t seed;
  int64_t first;
  uint8_t* out;
} img_ctx;

static void img_one(void* c, int i) {
  img_ctx* x = (img_ctx*)c;
  const size_t per = (size_t)x->h * x->w * 3;
  rstream rs;
  rs_init(&rs, mix_seed(x->seed, 1000000ULL + (uint64_t)(x->first + i)));
  uint8_t* o = x->out + per * (size_t)i;
  /* Textured image: a base colour,
   * three triangle-wave gratings with per-channel amplitude, and per-pixel
   * noise, all in integer arithmetic. Draw order: base[3]; per grating fx, fy,
   * phase, amp[3]; then one noise draw per (h, w, c). */
  int base[3], fx[3], fy[3], ph[3], amp[3][3];
  for (int c = 0; c < 3; ++c) base[c] = 64 + (int)(mt64_next(&rs.g) >> 57);
  for (int g = 0; g < 3; ++g) {
    fx[g] = (int)(mt64_next(&rs.g) >> 59) - 16;
    fy[g] = (int)(mt64_next(&rs.g) >> 59) - 16;
    ph[g] = (int)(mt64_next(&rs.g) >> 56);
    for (int c = 0; c < 3; ++c) amp[g][c] = (int)(mt64_next(&rs.g) >> 58);
  }
  for (int y = 0; y < x->h; ++y) {
    const int py = y * 256 / x->h;
    for (int xx = 0; xx < x->w; ++xx) {
      const int px = xx * 256 / x->w;
      int tri[3];
      for (int g = 0; g < 3; ++g) {
        const unsigned p = (unsigned)(fx[g] * px + fy[g] * py + ph[g]) & 255u;
        tri[g] = abs((int)p - 128) - 64;
      }
      for (int c = 0; c < 3; ++c) {
        int v = base[c] + (int)(mt64_next(&rs.g) >> 58) - 32;
        for (int g = 0; g < 3; ++g) v += (tri[g] * amp[g][c] + 4096) / 64 - 64; /* floor(t*a/64) */
        *o++ = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
      }
    }
  }
}

void oracle_generate_images(int h, int w, uint64_t seed, int64_t first, int count, uint8_t* out) {
  img_ctx c = {h, w, seed, first, out};
  parallel_for(count, img_one, &c);
}

typedef struct {
  const net* n;
  const uint8_t* images;
  int st;
  float* logits;
} fwd_ctx;

static void fwd_one(void* c, int i) {
  fwd_ctx* x = (fwd_ctx*)c;
  const size_t per = (size_t)x->n->in_h * x->n->in_w * 3;
  forward_one(x->n, x->images + per * (size_t)i, x->st, x->logits + (size_t)i * x->n->classes);
}

/* images: u8 NHWC [count][h][w][3]; logits: [count][classes] */
int oracle_forward(const char* id, const uint8_t* images, int count, int bf16_storage,
                   float* logits) {
  net* n = get_net(id);
  if (!n) return 1;
  fwd_ctx c = {n, images, bf16_storage, logits};
  parallel_for(count, fwd_one, &c);
  return 0;
}

/* Exports parameter layer `layer` in the device layout: conv/fc
 * bf16 [cout][kpad] with k = (r*S+s)*cin_stored + c (cin_stored = 4 for a
 * stem reading the 3-channel input), dw bf16 [9][C]; fp32 bias. */
int oracle_param_device_layout(const char* id, int layer, uint16_t* w, size_t w_cap, size_t* w_len,
                               float* b, int* kpad_out) {
  net* n = get_net(id);
  if (!n) return 1;
  int l = -1;
  for (int i = 0; i < n->nops; ++i) {
    op* o = &n->ops[i];
    if (!has_params(o)) continue;
    if (++l != layer) continue;
    if (o->kind == K_DW) {
      size_t len = (size_t)9 * o->cout;
      *w_len = len;
      *kpad_out = 9;
      if (w && w_cap >= len)
        for (size_t q = 0; q < len; ++q) w[q] = bf16_bits(o->wt[q]);
      if (b) memcpy(b, o->bias, sizeof(float) * o->cout);
      return 0;
    }
    int cs = (o->in == 0) ? 4 : o->cin;
    int kpad = (o->kh * o->kw * cs + 63) / 64 * 64;
    size_t len = (size_t)o->cout * kpad;
    *w_len = len;
    *kpad_out = kpad;
    if (w && w_cap >= len) {
      memset(w, 0, len * sizeof(uint16_t));
      for (int co = 0; co < o->cout; ++co)
        for (int r = 0; r < o->kh; ++r)
          for (int s = 0; s < o->kw; ++s)
            for (int c = 0; c < o->cin; ++c)
              w[(size_t)co * kpad + (r * o->kw + s) * cs + c] =
                  bf16_bits(o->wt[(size_t)((r * o->kw + s) * o->cin + c) * o->cout + co]);
    }
    if (b) memcpy(b, o->bias, sizeof(float) * o->cout);
    return 0;
  }
  return 2;
}

/* ---- IR export for the independent torch cross-check (tests/golden) ---- */
int oracle_num_ops(const char* id) {
  net* n = get_net(id);
  return n ? n->nops : -1;
}

int oracle_num_buffers(const char* id) {
  net* n = get_net(id);
  return n ? n->nb : -1;
}

int oracle_buffer_shape(const char* id, int b, int* h, int* w, int* c) {
  net* n = get_net(id);
  if (!n || b < 0 || b >= n->nb) return 1;
  *h = n->buf[b].h;
  *w = n->buf[b].w;
  *c = n->buf[b].c;
  return 0;
}

/* f[14] = kind, in, out, c_off, res, kh, kw, sh, sw, ph, pw, relu, cin, cout */
int oracle_op(const char* id, int i, int* f) {
  net* n = get_net(id);
  if (!n || i < 0 || i >= n->nops) return 1;
  const op* o = &n->ops[i];
  int v[14] = {o->kind, o->in, o->out, o->c_off, o->res, o->kh, o->kw,
               o->sh,   o->sw, o->ph,  o->pw,    o->relu, o->cin, o->cout};
  memcpy(f, v, sizeof(v));
  return 0;
}

/* Canonical fp32 (bf16-valued) weights of op i: conv/fc [cout][kh][kw][cin],
 * depthwise [9][C]; bias [cout]. Returns the weight count, or -1. */
long oracle_op_params(const char* id, int i, float* w, float* b) {
  net* n = get_net(id);
  if (!n || i < 0 || i >= n->nops) return -1;
  const op* o = &n->ops[i];
  if (!has_params(o)) return 0;
  if (o->kind == K_DW) {
    if (w) memcpy(w, o->wt, sizeof(float) * 9 * o->cout);
    if (b) memcpy(b, o->bias, sizeof(float) * o->cout);
    return 9L * o->cout;
  }
  const long kk = (long)o->kh * o->kw * o->cin;
  if (w)
    for (int co = 0; co < o->cout; ++co)
      for (long k = 0; k < kk; ++k) w[(long)co * kk + k] = o->wt[k * o->cout + co];
  if (b) memcpy(b, o->bias, sizeof(float) * o->cout);
  return kk * o->cout;
}

/* The oracle's restated generator, same contract as ref_random(). */
void oracle_random(uint64_t seed, int n, uint64_t* u64_out, double* gauss_out, uint64_t* mix_out) {
  rstream a, b;
  rs_init(&a, seed);
  rs_init(&b, seed);
  for (int i = 0; i < n; ++i) {
    u64_out[i] = mt64_next(&a.g);
    gauss_out[i] = rs_gaussian(&b);
    mix_out[i] = mix_seed(seed, (uint64_t)i);
  }
}
