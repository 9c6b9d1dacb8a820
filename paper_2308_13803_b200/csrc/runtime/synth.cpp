#include "synth.hpp"

#include <dlfcn.h>

#include <stdexcept>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>

namespace ds {

uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return 0x7FC0;  // NaN
  const uint32_t rounding = 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>((u + rounding) >> 16);
}

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Fills one layer. Draw order: weights output-channel-major, then (r, s, c)
// over the real input channels; then one bias per output channel (none for FC).
void fill_layer(const ParamSpec& p, int l, uint64_t seed, int kpad, uint16_t* w, float* b,
                const HeadCalib* head) {
  RandomStream rs(mix_seed(seed, kWeightSalt + static_cast<uint64_t>(l)));
  if (p.kind == OpKind::kDwConv) {
    const double sd = std::sqrt(2.0 / 9.0) * static_cast<double>(p.gain);
    for (int co = 0; co < p.cout; ++co)
      for (int tap = 0; tap < 9; ++tap)
        w[static_cast<size_t>(tap) * p.cout + co] =
            f32_to_bf16_rne(static_cast<float>(rs.gaussian() * sd));
    for (int co = 0; co < p.cout; ++co) b[co] = static_cast<float>(0.1 * rs.gaussian());
    return;
  }
  if (p.fc && head) {
    // Calibrated head (synth.hpp HeadCalib): W = bf16(R diag(scale) V),
    // b = -W mu, R[co][j] drawn co-major from this layer's stream.
    const int k = head->k, C = head->c;
    std::vector<double> r(static_cast<size_t>(p.cout) * k);
    for (auto& x : r) x = rs.gaussian();
    for (int co = 0; co < p.cout; ++co) {
      uint16_t* row = w + static_cast<size_t>(co) * kpad;
      double bacc = 0.0;
      for (int c = 0; c < C; ++c) {
        double acc = 0.0;
        for (int j = 0; j < k; ++j)
          acc += (r[static_cast<size_t>(co) * k + j] * head->scale[j]) * head->v[static_cast<size_t>(j) * C + c];
        row[c] = f32_to_bf16_rne(static_cast<float>(acc));
        uint32_t u = static_cast<uint32_t>(row[c]) << 16;
        float wf;
        std::memcpy(&wf, &u, 4);
        bacc += static_cast<double>(wf) * head->mu[c];
      }
      b[co] = static_cast<float>(-bacc);
    }
    return;
  }
  const int fan_in = p.r * p.s * p.cin;
  const double sd = (p.fc ? std::sqrt(1.0 / fan_in) : std::sqrt(2.0 / fan_in)) *
                    static_cast<double>(p.gain);
  for (int co = 0; co < p.cout; ++co) {
    uint16_t* row = w + static_cast<size_t>(co) * kpad;
    for (int r = 0; r < p.r; ++r)
      for (int s = 0; s < p.s; ++s)
        for (int c = 0; c < p.cin; ++c)
          row[(r * p.s + s) * p.cin_stored + c] =
              f32_to_bf16_rne(static_cast<float>(rs.gaussian() * sd));
  }
  for (int co = 0; co < p.cout; ++co) b[co] = p.fc ? 0.0f : static_cast<float>(0.1 * rs.gaussian());
}

}  // namespace

std::string head_dir() {
  if (const char* e = std::getenv("DS_HEAD_DIR")) return e;
  Dl_info info{};
  if (dladdr(reinterpret_cast<void*>(&head_dir), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t slash = p.rfind('/');
    return (slash == std::string::npos ? std::string(".") : p.substr(0, slash)) + "/data/heads";
  }
  return "data/heads";
}

HeadCalib load_head(const std::string& model_id) {
  HeadCalib h;
  const std::string path = head_dir() + "/" + model_id + ".head";
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return h;  // uncalibrated: plain random head
  char magic[8];
  int32_t dims[2];
  bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "DSHEAD1", 8) == 0 &&
            std::fread(dims, 4, 2, f) == 2 && dims[0] > 0 && dims[1] > 0 && dims[1] <= dims[0];
  if (ok) {
    h.c = dims[0];
    h.k = dims[1];
    h.mu.resize(h.c);
    h.scale.resize(h.k);
    h.v.resize(static_cast<size_t>(h.k) * h.c);
    ok = std::fread(h.mu.data(), 8, h.c, f) == static_cast<size_t>(h.c) &&
         std::fread(h.scale.data(), 8, h.k, f) == static_cast<size_t>(h.k) &&
         std::fread(h.v.data(), 8, h.v.size(), f) == h.v.size();
  }
  std::fclose(f);
  if (!ok) throw std::runtime_error("corrupt head calibration file " + path);
  return h;
}

HostParams generate_params(const ModelSpec& m, uint64_t seed) {
  HostParams hp;
  size_t wn = 0, bn = 0;
  for (const auto& p : m.params) {
    int kpad;
    size_t welems;
    if (p.kind == OpKind::kDwConv) {
      kpad = 9;
      welems = static_cast<size_t>(9) * p.cout;
    } else {
      kpad = (p.r * p.s * p.cin_stored + 63) / 64 * 64;
      welems = static_cast<size_t>(p.cout) * kpad;
    }
    hp.kpad.push_back(kpad);
    hp.w_off.push_back(wn);
    hp.b_off.push_back(bn);
    wn = align_up(wn + welems, 64);
    bn = align_up(bn + p.cout, 32);
  }
  hp.head = load_head(m.id);
  if (hp.head.k > 0 && hp.head.c != m.params.back().cin)
    throw std::runtime_error("head calibration " + m.id + ": feature width mismatch");
  hp.w.assign(wn, 0);
  hp.b.assign(bn, 0.0f);
  const int nl = static_cast<int>(m.params.size());
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      for (int l = static_cast<int>(t); l < nl; l += static_cast<int>(nt))
        fill_layer(m.params[l], l, seed, hp.kpad[l], hp.w.data() + hp.w_off[l],
                   hp.b.data() + hp.b_off[l], hp.head.k > 0 ? &hp.head : nullptr);
    });
  }
  for (auto& th : pool) th.join();
  return hp;
}

const HostParams& params_for(const ModelSpec& m) {
  static std::mutex mu;
  static std::map<std::string, HostParams> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(m.id);
  if (it == cache.end()) it = cache.emplace(m.id, generate_params(m)).first;
  return it->second;
}

void generate_images(int h, int w, uint64_t seed, int64_t first, int count, uint8_t* out) {
  const size_t per = static_cast<size_t>(h) * w * 3;
  // Textured image: base colour, three triangle-wave gratings with
  // per-channel amplitude, per-pixel noise; integer arithmetic only, so the
  // bytes are identical on every host (same draws as oracle img_one).
  auto one = [&](int i) {
    RandomStream rs(mix_seed(seed, kImageSalt + static_cast<uint64_t>(first + i)));
    uint8_t* o = out + per * i;
    int base[3], fx[3], fy[3], ph[3], amp[3][3];
    for (int c = 0; c < 3; ++c) base[c] = 64 + static_cast<int>(rs.next_u64() >> 57);
    for (int g = 0; g < 3; ++g) {
      fx[g] = static_cast<int>(rs.next_u64() >> 59) - 16;
      fy[g] = static_cast<int>(rs.next_u64() >> 59) - 16;
      ph[g] = static_cast<int>(rs.next_u64() >> 56);
      for (int c = 0; c < 3; ++c) amp[g][c] = static_cast<int>(rs.next_u64() >> 58);
    }
    for (int y = 0; y < h; ++y) {
      const int py = y * 256 / h;
      for (int x = 0; x < w; ++x) {
        const int px = x * 256 / w;
        int tri[3];
        for (int g = 0; g < 3; ++g) {
          const unsigned p = static_cast<unsigned>(fx[g] * px + fy[g] * py + ph[g]) & 255u;
          tri[g] = std::abs(static_cast<int>(p) - 128) - 64;
        }
        for (int c = 0; c < 3; ++c) {
          int v = base[c] + static_cast<int>(rs.next_u64() >> 58) - 32;
          for (int g = 0; g < 3; ++g) v += (tri[g] * amp[g][c] + 4096) / 64 - 64;
          *o++ = static_cast<uint8_t>(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
      }
    }
  };
  if (count < 4) {
    for (int i = 0; i < count; ++i) one(i);
    return;
  }
  const int nt = std::max(1, std::min(16, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (int i = t; i < count; i += nt) one(i);
    });
  for (auto& th : pool) th.join();
}

}  // namespace ds
