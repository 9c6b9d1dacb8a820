// Architecture definitions (see model.hpp). Parameter layers are numbered in
// the order the builder emits them; that index seeds each layer's weights
// (mix_seed(42, 1000 + index), reference random.hpp:10-15), so the order here
// is part of the model definition and is restated independently in
// oracle/fwd_oracle.c.
#include "model.hpp"

#include "../kernels/conv_gemm.cuh"

#include <cstdlib>
#include <stdexcept>

namespace ds {

namespace {

class Builder {
 public:
  explicit Builder(ModelSpec& m) : m_(m) {}

  int buffer(int h, int w, int c, bool f32 = false) {
    m_.buffers.push_back(BufferSpec{h, w, c, f32});
    return static_cast<int>(m_.buffers.size()) - 1;
  }

  const BufferSpec& buf(int id) const { return m_.buffers.at(id); }

  // Dense conv; writes channels [c_off, c_off + cout) of `out` (a new buffer
  // when out < 0). Returns the output buffer.
  int conv(int in, int cout, int r, int s, int sh, int sw, int ph, int pw, int out = -1,
           int c_off = 0, int residual = -1, bool relu = true, float gain = 1.0f) {
    const BufferSpec ib = buf(in);
    const int ho = (ib.h + 2 * ph - r) / sh + 1;
    const int wo = (ib.w + 2 * pw - s) / sw + 1;
    if (out < 0) out = buffer(ho, wo, cout);
    const BufferSpec ob = buf(out);
    if (ob.h != ho || ob.w != wo || c_off + cout > ob.c)
      throw std::logic_error("conv output shape mismatch in " + m_.id);
    ParamSpec p;
    p.kind = OpKind::kConv;
    p.cout = cout;
    p.r = r;
    p.s = s;
    p.cin_stored = ib.c;
    p.cin = (in == 0) ? 3 : ib.c;
    p.gain = gain;
    m_.params.push_back(p);
    OpSpec op;
    op.kind = OpKind::kConv;
    op.in = in;
    op.out = out;
    op.c_off = c_off;
    op.residual = residual;
    op.r = r;
    op.s = s;
    op.sh = sh;
    op.sw = sw;
    op.ph = ph;
    op.pw = pw;
    op.relu = relu;
    op.param = static_cast<int>(m_.params.size()) - 1;
    m_.ops.push_back(op);
    m_.macs_per_image += static_cast<double>(ho) * wo * cout * r * s * p.cin;
    return out;
  }

  int conv_sq(int in, int cout, int k, int stride, int pad, int out = -1, int c_off = 0) {
    return conv(in, cout, k, k, stride, stride, pad, pad, out, c_off);
  }

  int dw(int in, int stride) {
    const BufferSpec ib = buf(in);
    const int ho = (ib.h + 2 - 3) / stride + 1, wo = (ib.w + 2 - 3) / stride + 1;
    const int out = buffer(ho, wo, ib.c);
    ParamSpec p;
    p.kind = OpKind::kDwConv;
    p.cout = ib.c;
    p.r = p.s = 3;
    p.cin = p.cin_stored = 1;
    m_.params.push_back(p);
    OpSpec op;
    op.kind = OpKind::kDwConv;
    op.in = in;
    op.out = out;
    op.r = op.s = 3;
    op.sh = op.sw = stride;
    op.ph = op.pw = 1;
    op.param = static_cast<int>(m_.params.size()) - 1;
    m_.ops.push_back(op);
    m_.macs_per_image += static_cast<double>(ho) * wo * ib.c * 9;
    return out;
  }

  int pool(int in, bool is_max, int stride, int pad, int out = -1, int c_off = 0) {
    const BufferSpec ib = buf(in);
    const int ho = (ib.h + 2 * pad - 3) / stride + 1, wo = (ib.w + 2 * pad - 3) / stride + 1;
    if (out < 0) out = buffer(ho, wo, ib.c);
    const BufferSpec ob = buf(out);
    if (ob.h != ho || ob.w != wo || c_off + ib.c > ob.c)
      throw std::logic_error("pool output shape mismatch in " + m_.id);
    OpSpec op;
    op.kind = is_max ? OpKind::kMaxPool : OpKind::kAvgPool;
    op.in = in;
    op.out = out;
    op.c_off = c_off;
    op.r = op.s = 3;
    op.sh = op.sw = stride;
    op.ph = op.pw = pad;
    op.relu = false;
    m_.ops.push_back(op);
    return out;
  }

  int gap(int in) {
    const BufferSpec ib = buf(in);
    const int out = buffer(1, 1, ib.c);
    OpSpec op;
    op.kind = OpKind::kGlobalAvgPool;
    op.in = in;
    op.out = out;
    op.relu = false;
    m_.ops.push_back(op);
    return out;
  }

  int fc(int in, int classes) {
    const BufferSpec ib = buf(in);
    const int out = buffer(1, 1, classes, true);
    ParamSpec p;
    p.kind = OpKind::kFc;
    p.cout = classes;
    p.cin = p.cin_stored = ib.c;
    p.fc = true;
    m_.params.push_back(p);
    OpSpec op;
    op.kind = OpKind::kFc;
    op.in = in;
    op.out = out;
    op.relu = false;
    op.param = static_cast<int>(m_.params.size()) - 1;
    m_.ops.push_back(op);
    m_.macs_per_image += static_cast<double>(classes) * ib.c;
    m_.logits = out;
    m_.classes = classes;
    return out;
  }

 private:
  ModelSpec& m_;
};

ModelSpec synthetic_cnn() {
  // Config 1: 3x32x32 -> conv3x3 32 -> conv3x3 s2 64 -> conv3x3 s2 128 -> GAP -> FC 10.
  ModelSpec m;
  m.id = "synthetic_cnn";
  m.in_h = m.in_w = 32;
  Builder b(m);
  int x = b.buffer(32, 32, 4);
  x = b.conv_sq(x, 32, 3, 1, 1);
  x = b.conv_sq(x, 64, 3, 2, 1);
  x = b.conv_sq(x, 128, 3, 2, 1);
  b.fc(b.gap(x), 10);
  return m;
}

ModelSpec mobilenet_v1() {
  // Howard et al. 2017, width 1.0, 224x224 (Table 1): stem + 13 dw/pw pairs.
  ModelSpec m;
  m.id = "mobilenet_v1";
  m.in_h = m.in_w = 224;
  Builder b(m);
  int x = b.buffer(224, 224, 4);
  x = b.conv_sq(x, 32, 3, 2, 1);
  const int cfg[13][2] = {{64, 1},  {128, 2}, {128, 1}, {256, 2}, {256, 1},
                          {512, 2}, {512, 1}, {512, 1}, {512, 1}, {512, 1},
                          {512, 1}, {1024, 2}, {1024, 1}};
  for (const auto& c : cfg) {
    x = b.dw(x, c[1]);
    x = b.conv_sq(x, c[0], 1, 1, 0);
  }
  b.fc(b.gap(x), 1000);
  return m;
}

ModelSpec resnet50_v1() {
  // He et al. 2016, original v1: the stride of a down-sampling bottleneck
  // sits on its first 1x1 conv (and on the projection shortcut).
  ModelSpec m;
  m.id = "resnet50_v1";
  m.in_h = m.in_w = 224;
  Builder b(m);
  int x = b.buffer(224, 224, 4);
  x = b.conv_sq(x, 64, 7, 2, 3);
  x = b.pool(x, true, 2, 1);
  const int blocks[4] = {3, 4, 6, 3};
  const int width[4] = {64, 128, 256, 512};
  for (int st = 0; st < 4; ++st) {
    for (int i = 0; i < blocks[st]; ++i) {
      const int stride = (i == 0 && st > 0) ? 2 : 1;
      const int w = width[st];
      const int in = x;
      int y = b.conv(in, w, 1, 1, stride, stride, 0, 0);
      y = b.conv_sq(y, w, 3, 1, 1);
      int shortcut = in;
      if (i == 0) shortcut = b.conv(in, 4 * w, 1, 1, stride, stride, 0, 0, -1, 0, -1, false);
      x = b.conv(y, 4 * w, 1, 1, 1, 1, 0, 0, -1, 0, shortcut, true, 0.5f);
    }
  }
  b.fc(b.gap(x), 1000);
  return m;
}

// Inception-v3 (Szegedy et al. 2016), torchvision layout without the aux head.
int inception_a(Builder& b, int x, int pool_features) {
  const auto in = b.buf(x);
  const int out = b.buffer(in.h, in.w, 64 + 64 + 96 + pool_features);
  b.conv_sq(x, 64, 1, 1, 0, out, 0);
  int t = b.conv_sq(x, 48, 1, 1, 0);
  b.conv_sq(t, 64, 5, 1, 2, out, 64);
  t = b.conv_sq(x, 64, 1, 1, 0);
  t = b.conv_sq(t, 96, 3, 1, 1);
  b.conv_sq(t, 96, 3, 1, 1, out, 128);
  t = b.pool(x, false, 1, 1);
  b.conv_sq(t, pool_features, 1, 1, 0, out, 224);
  return out;
}

int inception_b(Builder& b, int x) {
  const auto in = b.buf(x);
  const int ho = (in.h - 3) / 2 + 1, wo = (in.w - 3) / 2 + 1;
  const int out = b.buffer(ho, wo, 384 + 96 + in.c);
  b.conv_sq(x, 384, 3, 2, 0, out, 0);
  int t = b.conv_sq(x, 64, 1, 1, 0);
  t = b.conv_sq(t, 96, 3, 1, 1);
  b.conv_sq(t, 96, 3, 2, 0, out, 384);
  b.pool(x, true, 2, 0, out, 480);
  return out;
}

int inception_c(Builder& b, int x, int c7) {
  const auto in = b.buf(x);
  const int out = b.buffer(in.h, in.w, 768);
  b.conv_sq(x, 192, 1, 1, 0, out, 0);
  int t = b.conv_sq(x, c7, 1, 1, 0);
  t = b.conv(t, c7, 1, 7, 1, 1, 0, 3);
  b.conv(t, 192, 7, 1, 1, 1, 3, 0, out, 192);
  t = b.conv_sq(x, c7, 1, 1, 0);
  t = b.conv(t, c7, 7, 1, 1, 1, 3, 0);
  t = b.conv(t, c7, 1, 7, 1, 1, 0, 3);
  t = b.conv(t, c7, 7, 1, 1, 1, 3, 0);
  b.conv(t, 192, 1, 7, 1, 1, 0, 3, out, 384);
  t = b.pool(x, false, 1, 1);
  b.conv_sq(t, 192, 1, 1, 0, out, 576);
  return out;
}

int inception_d(Builder& b, int x) {
  const auto in = b.buf(x);
  const int ho = (in.h - 3) / 2 + 1, wo = (in.w - 3) / 2 + 1;
  const int out = b.buffer(ho, wo, 320 + 192 + in.c);
  int t = b.conv_sq(x, 192, 1, 1, 0);
  b.conv_sq(t, 320, 3, 2, 0, out, 0);
  t = b.conv_sq(x, 192, 1, 1, 0);
  t = b.conv(t, 192, 1, 7, 1, 1, 0, 3);
  t = b.conv(t, 192, 7, 1, 1, 1, 3, 0);
  b.conv_sq(t, 192, 3, 2, 0, out, 320);
  b.pool(x, true, 2, 0, out, 512);
  return out;
}

int inception_e(Builder& b, int x) {
  const auto in = b.buf(x);
  const int out = b.buffer(in.h, in.w, 2048);
  b.conv_sq(x, 320, 1, 1, 0, out, 0);
  int t = b.conv_sq(x, 384, 1, 1, 0);
  b.conv(t, 384, 1, 3, 1, 1, 0, 1, out, 320);
  b.conv(t, 384, 3, 1, 1, 1, 1, 0, out, 704);
  t = b.conv_sq(x, 448, 1, 1, 0);
  t = b.conv_sq(t, 384, 3, 1, 1);
  b.conv(t, 384, 1, 3, 1, 1, 0, 1, out, 1088);
  b.conv(t, 384, 3, 1, 1, 1, 1, 0, out, 1472);
  t = b.pool(x, false, 1, 1);
  b.conv_sq(t, 192, 1, 1, 0, out, 1856);
  return out;
}

ModelSpec inception_v3() {
  ModelSpec m;
  m.id = "inception_v3";
  m.in_h = m.in_w = 299;
  Builder b(m);
  int x = b.buffer(299, 299, 4);
  x = b.conv_sq(x, 32, 3, 2, 0);
  x = b.conv_sq(x, 32, 3, 1, 0);
  x = b.conv_sq(x, 64, 3, 1, 1);
  x = b.pool(x, true, 2, 0);
  x = b.conv_sq(x, 80, 1, 1, 0);
  x = b.conv_sq(x, 192, 3, 1, 0);
  x = b.pool(x, true, 2, 0);
  x = inception_a(b, x, 32);
  x = inception_a(b, x, 64);
  x = inception_a(b, x, 64);
  x = inception_b(b, x);
  x = inception_c(b, x, 128);
  x = inception_c(b, x, 160);
  x = inception_c(b, x, 160);
  x = inception_c(b, x, 192);
  x = inception_d(b, x);
  x = inception_e(b, x);
  x = inception_e(b, x);
  b.fc(b.gap(x), 1000);
  return m;
}

}  // namespace

namespace {
// The op that reads the staged input (buffer 0), when it is a conv and its only reader.
int stem_op(const ModelSpec& m) {
  int stem = -1;
  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    if (op.in != 0 && op.residual != 0) continue;
    if (stem >= 0 || op.kind != OpKind::kConv || op.residual == 0 || m.buffers[0].c != 4) return -1;
    stem = static_cast<int>(i);
  }
  return stem;
}
}  // namespace

S2dPlan stem_s2d(const ModelSpec& m) {
  S2dPlan p;
  const int stem = stem_op(m);
  if (stem < 0) return p;
  const OpSpec& op = m.ops[stem];
  const BufferSpec& out = m.buffers[op.out];
  const int cout = m.params[op.param].cout;
  if (op.sh != 2 || op.sw != 2 || op.ph != op.pw || op.r > 8 || op.s > 8 || cout > 256) return p;
  p.dr = (op.r + 1) / 2;
  p.ds = (op.s + 1) / 2;
  p.kpad = (p.dr * p.ds * 16 + 63) / 64 * 64;
  if (p.kpad / 64 * ((cout + 15) / 16 * 16) * 128 > 64 * 1024) return p;  // weights stay resident
  p.op = stem;
  p.hs = out.h + p.dr - 1;
  p.ws = out.w + p.ds - 1;
  p.pad = op.ph;
  return p;
}

int fused_stem(const ModelSpec& m) {
  if (stem_s2d(m).op >= 0) return -1;  // the space-to-depth stem wins where it applies
  int stem = -1;
  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    if (op.in != 0 && op.residual != 0) continue;
    if (stem >= 0 || op.kind != OpKind::kConv || op.residual == 0 || m.buffers[0].c != 4) return -1;
    stem = static_cast<int>(i);
  }
  if (stem >= 0) {
    const OpSpec& op = m.ops[stem];
    const BufferSpec& in = m.buffers[0];
    (void)in;
    if (!conv_gemm_stem_fits(op.r, op.s, m.params[op.param].cout)) return -1;
  }
  return stem;
}

std::vector<KernelCost> kernel_costs(const ModelSpec& m) {
  const int stem = fused_stem(m);
  const S2dPlan s2d = stem_s2d(m);
  std::vector<KernelCost> out;
  const double px = static_cast<double>(m.in_h) * m.in_w;
  const double s2d_bytes = static_cast<double>(s2d.hs) * s2d.ws * 32;
  if (s2d.op >= 0) out.push_back({KernelKind::kStage, 0.0, px * 3 + s2d_bytes, 0.0});
  for (const auto& op : m.ops) {
    const BufferSpec& in = m.buffers[op.in];
    const BufferSpec& out_b = m.buffers[op.out];
    const double in_elems = static_cast<double>(in.h) * in.w * in.c;
    const double hw_out = static_cast<double>(out_b.h) * out_b.w;
    KernelCost k{KernelKind::kPool, 0.0, 0.0, 0.0};
    switch (op.kind) {
      case OpKind::kConv:
      case OpKind::kFc: {
        const ParamSpec& p = m.params[op.param];
        const double out_elems = hw_out * p.cout;
        k.kind = KernelKind::kConvGemm;
        k.flops_per_image = 2.0 * out_elems * p.r * p.s * p.cin;
        // the fused stem reads the u8 image (3 B per pixel); the s2d stem its
        // space-to-depth tensor
        const int oi = static_cast<int>(&op - m.ops.data());
        const double in_bytes = oi == stem ? px * 3 : oi == s2d.op ? s2d_bytes : in_elems * 2;
        k.bytes_per_image = in_bytes + out_elems * (out_b.f32 ? 4 : 2) +
                            (op.residual >= 0 ? out_elems * 2 : 0.0);
        k.fixed_bytes = static_cast<double>(p.cout) * p.r * p.s * p.cin * 2 + p.cout * 4.0;
        for (const auto& f : op.fused) {  // siblings: the input is read once
          const ParamSpec& q = m.params[f.param];
          const double oe = hw_out * q.cout;
          k.flops_per_image += 2.0 * oe * q.cin;
          k.bytes_per_image += oe * 2;
          k.fixed_bytes += static_cast<double>(q.cout) * q.cin * 2 + q.cout * 4.0;
        }
        break;
      }
      case OpKind::kDwConv: {
        k.kind = KernelKind::kDwConv;
        k.flops_per_image = 2.0 * hw_out * in.c * 9;
        k.bytes_per_image = in_elems * 2 + hw_out * in.c * 2;
        k.fixed_bytes = in.c * 9.0 * 2 + in.c * 4.0;
        break;
      }
      case OpKind::kMaxPool:
      case OpKind::kAvgPool:
        k.kind = KernelKind::kPool;
        k.bytes_per_image = in_elems * 2 + hw_out * in.c * 2;
        break;
      case OpKind::kGlobalAvgPool:
        k.kind = KernelKind::kGap;
        k.bytes_per_image = in_elems * 2 + in.c * 2.0;
        break;
    }
    out.push_back(k);
  }
  out.push_back({KernelKind::kSoftmax, 0.0, m.classes * 8.0, 0.0});
  return out;
}

std::vector<std::string> model_ids() {
  return {"synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3"};
}

void swap_avgpool_1x1(ModelSpec& m) {
  for (size_t i = 0; i < m.ops.size(); ++i) {
    OpSpec& pool = m.ops[i];
    if (pool.kind != OpKind::kAvgPool || pool.sh != 1 || pool.sw != 1 || pool.ph != 1 || pool.pw != 1 ||
        pool.c_off != 0 || pool.post_bias >= 0)
      continue;
    const int t = pool.out;
    int consumer = -1, uses = 0;
    for (size_t j = 0; j < m.ops.size(); ++j) {
      const OpSpec& o = m.ops[j];
      if (o.in == t || o.residual == t) {
        ++uses;
        consumer = static_cast<int>(j);
      }
      if (j != i && o.out == t) uses = 99;  // (t written elsewhere)
    }
    if (uses != 1 || consumer <= static_cast<int>(i)) continue;
    OpSpec conv = m.ops[consumer];
    if (conv.kind != OpKind::kConv || conv.r != 1 || conv.s != 1 || conv.sh != 1 || conv.sw != 1 ||
        conv.ph != 0 || conv.pw != 0 || conv.residual >= 0 || !conv.fused.empty() || conv.no_bias ||
        m.buffers[conv.out].f32)
      continue;
    const BufferSpec x = m.buffers[pool.in];
    const int cout = m.params[conv.param].cout;
    if (cout % 8 != 0) continue;
    m.buffers.push_back(BufferSpec{x.h, x.w, cout, false});
    const int z = static_cast<int>(m.buffers.size()) - 1;
    OpSpec c2 = conv;  // W x, no bias, no ReLU
    c2.in = pool.in;
    c2.out = z;
    c2.c_off = 0;
    c2.relu = false;
    c2.no_bias = true;
    OpSpec p2 = pool;  // pool the conv output, + b, ReLU, into the conv's slice
    p2.in = z;
    p2.out = conv.out;
    p2.c_off = conv.c_off;
    p2.post_bias = conv.param;
    p2.relu = conv.relu;
    m.ops[i] = c2;
    m.ops[consumer] = p2;
  }
}

void fuse_sibling_1x1(ModelSpec& m) {
  auto is_1x1 = [&](const OpSpec& o) {
    return o.kind == OpKind::kConv && o.r == 1 && o.s == 1 && o.ph == 0 && o.pw == 0 &&
           o.residual < 0 && o.fused.empty() && !m.buffers[o.out].f32 && o.in != 0;
  };
  std::vector<OpSpec> out;
  std::vector<char> taken(m.ops.size(), 0);
  for (size_t i = 0; i < m.ops.size(); ++i) {
    if (taken[i]) continue;
    OpSpec op = m.ops[i];
    if (is_1x1(op)) {
      for (size_t j = i + 1; j < m.ops.size() && op.fused.size() < 3; ++j) {
        const OpSpec& o = m.ops[j];
        if (taken[j] || !is_1x1(o) || o.in != op.in || o.sh != op.sh || o.sw != op.sw) continue;
        // moving op j up to i: nothing in between may read its output or
        // write the buffer it reads
        bool safe = true;
        for (size_t k = i + 1; k < j && safe; ++k) {
          const OpSpec& b = m.ops[k];
          if (b.in == o.out || b.residual == o.out || b.out == o.in) safe = false;
          for (const auto& f : b.fused)
            if (f.out == o.in) safe = false;
        }
        if (!safe) continue;
        op.fused.push_back(ConvSeg{o.param, o.out, o.c_off, o.relu, o.no_bias});
        taken[j] = 1;
      }
    }
    out.push_back(op);
  }
  m.ops = std::move(out);
}

ModelSpec build_model(const std::string& id) {
  ModelSpec m;
  if (id == "synthetic_cnn") m = synthetic_cnn();
  else if (id == "mobilenet_v1") m = mobilenet_v1();
  else if (id == "resnet50_v1") m = resnet50_v1();
  else if (id == "inception_v3") m = inception_v3();
  else throw std::invalid_argument("unknown model: " + id);
  const char* sw = std::getenv("DS_POOL_SWAP");
  if (!(sw && sw[0] == '0')) swap_avgpool_1x1(m);
  const char* e = std::getenv("DS_FUSE_1X1");
  if (!(e && e[0] == '0')) fuse_sibling_1x1(m);
  return m;
}

}  // namespace ds
