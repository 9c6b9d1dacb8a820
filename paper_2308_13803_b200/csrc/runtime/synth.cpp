#include "synth.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
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
void fill_layer(const ParamSpec& p, int l, uint64_t seed, int kpad, uint16_t* w, float* b) {
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
  hp.w.assign(wn, 0);
  hp.b.assign(bn, 0.0f);
  const int nl = static_cast<int>(m.params.size());
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      for (int l = static_cast<int>(t); l < nl; l += static_cast<int>(nt))
        fill_layer(m.params[l], l, seed, hp.kpad[l], hp.w.data() + hp.w_off[l],
                   hp.b.data() + hp.b_off[l]);
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
  auto one = [&](int i) {
    RandomStream rs(mix_seed(seed, kImageSalt + static_cast<uint64_t>(first + i)));
    uint8_t* o = out + per * i;
    for (size_t q = 0; q < per; ++q) o[q] = static_cast<uint8_t>(rs.next_u64() >> 56);
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
