// extern "C" boundary over ds::Backend (include/dnnscaler_b200.h).
#include "../../../include/dnnscaler_b200.h"

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "abi_internal.hpp"

namespace {

thread_local std::string g_last_error;

}  // namespace

void ds_internal_set_error(const std::string& msg) { g_last_error = msg; }

namespace {

template <typename F>
ds_status guard(F&& f) {
  try {
    f();
    return DS_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return DS_EINVAL;
  } catch (const ds::CudaError& e) {
    g_last_error = e.what();
    return DS_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return DS_ERUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return DS_ERUNTIME;
  }
}

ds_status null_handle() {
  g_last_error = "null handle";
  return DS_EINVAL;
}

}  // namespace

extern "C" {

const char* ds_last_error(void) { return g_last_error.c_str(); }

ds_status ds_backend_create(const char* model_id, ds_config config, uint64_t seed, int device,
                            ds_backend** out) {
  if (!out || !model_id) return null_handle();
  *out = nullptr;
  return guard([&] {
    ds::BackendConfig cfg{config.abs_max_bs, config.max_mtl};
    auto* impl = new ds::Backend(model_id, cfg, seed, device);
    *out = new ds_backend{impl};
  });
}

void ds_backend_destroy(ds_backend* b) {
  if (!b) return;
  delete b->impl;
  delete b;
}

ds_status ds_run_batch(ds_backend* b, int bs, double* latency_ms) {
  if (!b) return null_handle();
  return guard([&] {
    const double lat = b->impl->run_batch(bs);
    if (latency_ms) *latency_ms = lat;
  });
}

ds_status ds_run_mt_request(ds_backend* b, double* latency_ms) {
  if (!b) return null_handle();
  return guard([&] {
    const double lat = b->impl->run_mt_request();
    if (latency_ms) *latency_ms = lat;
  });
}

ds_status ds_apply_instance_change(ds_backend* b, int delta, double* delay_ms) {
  if (!b) return null_handle();
  return guard([&] {
    const double d = b->impl->apply_instance_change(delta);
    if (delay_ms) *delay_ms = d;
  });
}

ds_status ds_set_mtl(ds_backend* b, int target, double* total_delay_ms) {
  if (!b) return null_handle();
  return guard([&] {
    const double d = b->impl->set_mtl(target);
    if (total_delay_ms) *total_delay_ms = d;
  });
}

int ds_mtl(const ds_backend* b) { return b ? b->impl->mtl() : 0; }

double ds_clock_ms(const ds_backend* b) { return b ? b->impl->clock_ms() : 0.0; }

ds_config ds_get_config(const ds_backend* b) {
  ds_config c{0, 0};
  if (b) {
    c.abs_max_bs = b->impl->config().abs_max_bs;
    c.max_mtl = b->impl->config().max_mtl;
  }
  return c;
}

ds_status ds_run_batches(ds_backend* b, int bs, int count, double* latencies_ms) {
  if (!b) return null_handle();
  if (count < 0 || (count > 0 && !latencies_ms)) {
    g_last_error = "invalid window";
    return DS_EINVAL;
  }
  return guard([&] { b->impl->run_batches(bs, count, latencies_ms); });
}

ds_status ds_run_mt_requests(ds_backend* b, int count, double* latencies_ms) {
  if (!b) return null_handle();
  if (count < 0 || (count > 0 && !latencies_ms)) {
    g_last_error = "invalid window";
    return DS_EINVAL;
  }
  return guard([&] { b->impl->run_mt_requests(count, latencies_ms); });
}

ds_status ds_run_combo_requests(ds_backend* b, int bs, int mtl, int count, double* latencies_ms) {
  if (!b) return null_handle();
  if (count < 0 || (count > 0 && !latencies_ms)) {
    g_last_error = "invalid window";
    return DS_EINVAL;
  }
  return guard([&] { b->impl->run_combo_requests(bs, mtl, count, latencies_ms); });
}

ds_status ds_forward(ds_backend* b, const uint8_t* images, int bs, float* logits, float* probs) {
  if (!b) return null_handle();
  if (!images) {
    g_last_error = "null images";
    return DS_EINVAL;
  }
  return guard([&] { b->impl->forward(images, bs, logits, probs); });
}

ds_status ds_set_host_io(ds_backend* b, int enabled) {
  if (!b) return null_handle();
  return guard([&] { b->impl->set_host_io(enabled != 0); });
}

ds_status ds_last_output(ds_backend* b, int instance, float* logits, size_t cap,
                         int64_t* first_image, int* bs) {
  if (!b || !bs) return null_handle();
  return guard([&] {
    const int n = b->impl->last_output(instance, nullptr, nullptr);
    const size_t need = static_cast<size_t>(n) * b->impl->model().classes;
    if (logits && cap < need) throw std::invalid_argument("output buffer too small");
    *bs = b->impl->last_output(instance, logits, first_image);
  });
}

ds_status ds_set_mt_mode(ds_backend* b, int mode) {
  if (!b) return null_handle();
  return guard([&] { b->impl->set_mt_mode(mode); });
}

int ds_get_mt_mode(const ds_backend* b) { return b ? b->impl->mt_mode() : -1; }

ds_status ds_kernel_spans(ds_backend* b, int instance, int reset, double* ms_out, int cap,
                          int64_t* forwards) {
  if (!b) return null_handle();
  return guard([&] {
    if (reset) {
      b->impl->reset_spans(instance);
      if (forwards) *forwards = 0;
      return;
    }
    std::vector<double> ms;
    const int64_t n = b->impl->read_spans(instance, &ms);
    if (n < 0) throw std::runtime_error("live kernel timing slots disagree");
    if (forwards) *forwards = n;
    if (ms_out)
      for (int i = 0; i < cap && i < static_cast<int>(ms.size()); ++i) ms_out[i] = ms[i];
  });
}

ds_status ds_drain(ds_backend* b) {
  if (!b) return null_handle();
  return guard([&] { b->impl->drain(); });
}

void ds_nvtx_push(const char* name) { nvtxRangePushA(name ? name : ""); }

void ds_nvtx_pop(void) { nvtxRangePop(); }

ds_status ds_timer_start(ds_backend* b) {
  if (!b) return null_handle();
  return guard([&] { b->impl->timer_start(); });
}

ds_status ds_timer_stop(ds_backend* b, double* elapsed_ms) {
  if (!b || !elapsed_ms) return null_handle();
  return guard([&] { *elapsed_ms = b->impl->timer_stop(); });
}

ds_status ds_model_info_get(const char* model_id, ds_model_info* out) {
  if (!model_id || !out) return null_handle();
  return guard([&] {
    const ds::ModelSpec m = ds::build_model(model_id);
    std::memset(out, 0, sizeof(*out));
    out->in_h = m.in_h;
    out->in_w = m.in_w;
    out->classes = m.classes;
    out->n_ops = static_cast<int>(m.ops.size());
    out->n_params = static_cast<int>(m.params.size());
    out->macs_per_image = m.macs_per_image;
    double wc = 0.0;
    for (const auto& p : m.params) {
      if (p.kind == ds::OpKind::kDwConv)
        wc += 9.0 * p.cout + p.cout;
      else
        wc += static_cast<double>(p.cout) * p.r * p.s * p.cin + p.cout;
    }
    out->weight_count = wc;
    double act = 0.0;
    for (const auto& b : m.buffers) act += static_cast<double>(b.h) * b.w * b.c * (b.f32 ? 4 : 2);
    out->act_bytes_per_image = act;
    out->feature_buffer = m.ops.back().in;
    out->feature_channels = m.params.back().cin;
    out->head_k = ds::params_for(m).head.k;
  });
}

ds_status ds_backend_stats_get(const ds_backend* b, ds_backend_stats* out) {
  if (!b || !out) return null_handle();
  return guard([&] {
    out->kernel_launches = b->impl->kernel_launches();
    out->h2d_bytes = b->impl->h2d_bytes();
    out->d2h_bytes = b->impl->d2h_bytes();
    out->instances_created = b->impl->instances_created();
    out->kernels_per_forward = b->impl->kernels_per_forward();
    out->device_bytes = static_cast<double>(b->impl->device_bytes());
  });
}

ds_status ds_model_kernels(const char* model_id, ds_kernel_cost* out, int cap, int* n) {
  if (!model_id || !n) return null_handle();
  return guard([&] {
    const auto costs = ds::kernel_costs(ds::build_model(model_id));
    *n = static_cast<int>(costs.size());
    for (int i = 0; out && i < cap && i < *n; ++i)
      out[i] = ds_kernel_cost{static_cast<int>(costs[i].kind), costs[i].flops_per_image,
                              costs[i].bytes_per_image, costs[i].fixed_bytes};
  });
}

ds_status ds_profile_kernels(ds_backend* b, int bs, int reps, double* ms_out, int cap) {
  if (!b || !ms_out) return null_handle();
  return guard([&] {
    const auto ms = b->impl->profile_kernels(bs, reps < 1 ? 1 : reps);
    if (static_cast<int>(ms.size()) > cap) throw std::invalid_argument("output too small");
    for (size_t i = 0; i < ms.size(); ++i) ms_out[i] = ms[i];
  });
}

ds_status ds_debug_read_buffer(ds_backend* b, int buffer, int bs, void* out, size_t cap,
                               size_t* out_len) {
  if (!b || !out_len) return null_handle();
  return guard([&] {
    const ds::ModelSpec& m = b->impl->model();
    if (buffer < 0 || buffer >= static_cast<int>(m.buffers.size()))
      throw std::invalid_argument("invalid buffer");
    if (bs < 1 || bs > b->impl->config().abs_max_bs) throw std::invalid_argument("invalid batch size");
    const ds::BufferSpec& s = m.buffers[buffer];
    *out_len = static_cast<size_t>(bs) * s.h * s.w * s.c * (s.f32 ? 4 : 2);
    if (out && cap >= *out_len) b->impl->read_buffer(buffer, bs, out);
  });
}

ds_status ds_generate_images(int h, int w, uint64_t seed, int64_t first, int count,
                             uint8_t* out) {
  if (!out || h < 1 || w < 1 || count < 0) {
    g_last_error = "invalid image request";
    return DS_EINVAL;
  }
  return guard([&] { ds::generate_images(h, w, seed, first, count, out); });
}

ds_status ds_model_param(const char* model_id, int layer, uint16_t* w, size_t w_cap,
                         size_t* w_len, float* b, size_t b_cap, size_t* b_len, int* kpad) {
  if (!model_id) return null_handle();
  return guard([&] {
    static thread_local ds::ModelSpec m;
    if (m.id != model_id) m = ds::build_model(model_id);
    if (layer < 0 || layer >= static_cast<int>(m.params.size()))
      throw std::invalid_argument("invalid layer");
    const ds::HostParams& hp = ds::params_for(m);
    const ds::ParamSpec& p = m.params[layer];
    const size_t wl = p.kind == ds::OpKind::kDwConv ? static_cast<size_t>(9) * p.cout
                                                     : static_cast<size_t>(p.cout) * hp.kpad[layer];
    if (w_len) *w_len = wl;
    if (b_len) *b_len = static_cast<size_t>(p.cout);
    if (kpad) *kpad = hp.kpad[layer];
    if (w && w_cap >= wl) std::memcpy(w, hp.w.data() + hp.w_off[layer], wl * sizeof(uint16_t));
    if (b && b_cap >= static_cast<size_t>(p.cout))
      std::memcpy(b, hp.b.data() + hp.b_off[layer], p.cout * sizeof(float));
  });
}

}  // extern "C"
