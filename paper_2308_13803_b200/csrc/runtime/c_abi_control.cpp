// extern "C" boundary over the control plane (include/dnnscaler_b200.h,
// "Control plane" section).
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>

#include "../../../include/dnnscaler_b200.h"
#include "../../../include/dnnscaler_b200/control.hpp"
#include "abi_internal.hpp"
#include "device_seam.hpp"

struct ds_job_result {
  ds::JobTrace trace;
};

struct ds_job_session {
  ds::Scenario scenario;
  ds::JobSpec job;
  std::vector<ds::DnnProfile> catalog;
  std::unique_ptr<ds::JobSession> session;
};

namespace {

template <typename F>
ds_status guard(F&& f) {
  try {
    f();
    return DS_OK;
  } catch (const std::invalid_argument& e) {
    ds_internal_set_error(e.what());
    return DS_EINVAL;
  } catch (const ds::CudaError& e) {
    ds_internal_set_error(e.what());
    return DS_ECUDA;
  } catch (const std::exception& e) {
    ds_internal_set_error(e.what());
    return DS_ERUNTIME;
  }
}

ds_status invalid(const char* msg) {
  ds_internal_set_error(msg);
  return DS_EINVAL;
}

ds::Knob to_knob(ds_knob k) {
  return ds::Knob{k.kind == 1 ? ds::KnobKind::kMultiTenancy : ds::KnobKind::kBatching, k.value};
}

ds_knob from_knob(const ds::Knob& k) {
  return ds_knob{k.kind == ds::KnobKind::kMultiTenancy ? 1 : 0, k.value};
}

ds::Scenario to_scenario(const ds_scenario& s, const ds::JobSpec& job) {
  ds::Scenario sc;
  sc.jobs = {job};
  sc.controller = s.controller == 1   ? ds::ControllerKind::kClipper
                  : s.controller == 2 ? ds::ControllerKind::kStaticKnob
                                      : ds::ControllerKind::kDnnScaler;
  sc.static_knob = to_knob(s.static_knob);
  sc.seed = s.seed;
  sc.alpha = s.alpha;
  sc.m = s.m;
  sc.n = s.n;
  sc.abs_max_bs = s.abs_max_bs;
  sc.max_mtl = s.max_mtl;
  if (s.window < 1) throw std::invalid_argument("scenario: window must be positive");
  sc.window = static_cast<size_t>(s.window);
  sc.sigma = s.sigma;
  return sc;
}

ds::JobSpec to_job(const ds_job_spec& j) {
  ds::JobSpec job;
  job.job_id = j.job_id;
  job.dnn_id = j.dnn_id ? j.dnn_id : "";
  job.slo_ms = j.slo_ms;
  job.duration_s = j.duration_s;
  for (int i = 0; i < j.n_slo_steps; ++i)
    job.slo_schedule.push_back(ds::SloStep{j.slo_steps[i].at_s, j.slo_steps[i].slo_ms});
  return job;
}

std::vector<ds::DnnProfile> to_catalog(const ds_dnn_profile* c, int n) {
  std::vector<ds::DnnProfile> out;
  for (int i = 0; i < n; ++i) {
    ds::DnnProfile p;
    p.id = c[i].id ? c[i].id : "";
    for (int k = 0; k < c[i].n_batching; ++k)
      p.batching_points.emplace_back(c[i].batching_x[k], c[i].batching_tput[k]);
    for (int k = 0; k < c[i].n_mt; ++k) p.mt_points.emplace_back(c[i].mt_x[k], c[i].mt_tput[k]);
    if (c[i].has_sigma) p.sigma = c[i].sigma;
    if (c[i].has_u1) p.u1 = c[i].u1;
    out.push_back(std::move(p));
  }
  return out;
}

ds::SeamFactory make_factory(const ds_seam_spec& spec) {
  switch (spec.kind) {
    case DS_SEAM_ANALYTIC:
      return ds::analytic_seam_factory();
    case DS_SEAM_REPLAY: {
      std::vector<double> tape(spec.tape, spec.tape + spec.tape_len);
      std::vector<double> energy;
      if (spec.energy_tape) energy.assign(spec.energy_tape, spec.energy_tape + spec.energy_tape_len);
      return [tape, energy](const ds::Scenario& sc, const ds::JobSpec&, const ds::BatchingModel&,
                            const ds::MtModel&) {
        auto r = std::make_unique<ds::ReplaySeam>(tape, ds::Seam::Config{sc.abs_max_bs, sc.max_mtl});
        r->set_energy_tape(energy);
        return r;
      };
    }
    case DS_SEAM_DEVICE: {
      ds::Backend* shared = spec.backend ? spec.backend->impl : nullptr;
      const int device = spec.device;
      const bool host_io = spec.host_io != 0;
      return [shared, device, host_io](const ds::Scenario& sc, const ds::JobSpec& job,
                                       const ds::BatchingModel&,
                                       const ds::MtModel&) -> std::unique_ptr<ds::Seam> {
        if (shared) {
          if (shared->model().id != job.dnn_id)
            throw std::invalid_argument("backend serves " + shared->model().id + ", job wants " +
                                        job.dnn_id);
          if (shared->config().abs_max_bs < sc.abs_max_bs || shared->config().max_mtl < sc.max_mtl)
            throw std::invalid_argument("backend limits below scenario limits");
          return std::make_unique<ds::DeviceSeam>(*shared);
        }
        auto b = std::make_unique<ds::Backend>(
            job.dnn_id, ds::BackendConfig{sc.abs_max_bs, sc.max_mtl},
            ds::mix_seed_u64(sc.seed, static_cast<uint64_t>(job.job_id)), device);
        if (host_io) b->set_host_io(true);
        return std::make_unique<ds::DeviceSeam>(std::move(b));
      };
    }
  }
  throw std::invalid_argument("unknown seam kind");
}

}  // namespace

extern "C" {

ds_status ds_job_run(const ds_scenario* scenario, const ds_job_spec* job,
                     const ds_dnn_profile* catalog, int n_catalog, const ds_seam_spec* seam,
                     ds_job_result** out) {
  if (!scenario || !job || !seam || !out || (n_catalog > 0 && !catalog))
    return invalid("null argument");
  *out = nullptr;
  return guard([&] {
    const ds::JobSpec js = to_job(*job);
    const ds::Scenario sc = to_scenario(*scenario, js);
    const auto cat = to_catalog(catalog, n_catalog);
    const auto factory = make_factory(*seam);
    auto traces = ds::run_scenario(sc, cat, factory);
    *out = new ds_job_result{std::move(traces.front())};
  });
}

ds_status ds_job_start(const ds_scenario* scenario, const ds_job_spec* job,
                       const ds_dnn_profile* catalog, int n_catalog, const ds_seam_spec* seam,
                       ds_job_session** out) {
  if (!scenario || !job || !seam || !out || (n_catalog > 0 && !catalog))
    return invalid("null argument");
  *out = nullptr;
  return guard([&] {
    auto s = std::make_unique<ds_job_session>();
    s->job = to_job(*job);
    s->scenario = to_scenario(*scenario, s->job);
    s->catalog = to_catalog(catalog, n_catalog);
    ds::validate_scenario(s->scenario);
    s->session = std::make_unique<ds::JobSession>(s->scenario, s->scenario.jobs.front(),
                                                  s->catalog, make_factory(*seam));
    s->session->start();
    *out = s.release();
  });
}

ds_status ds_job_step(ds_job_session* s, ds_metrics_record* record, int* done) {
  if (!s) return invalid("null session");
  return guard([&] {
    const ds::MetricsRecord& r = s->session->step();
    if (record) {
      record->time_s = r.time_s;
      record->job_id = r.job_id;
      record->knob = from_knob(r.knob);
      record->p95_ms = r.p95_ms;
      record->mean_ms = r.mean_ms;
      record->throughput = r.throughput;
      record->power_w = r.power_w;
      record->slo_ms = r.slo_ms;
      record->violated = r.violated ? 1 : 0;
    }
    if (done) *done = s->session->done() ? 1 : 0;
  });
}

ds_status ds_job_knob(const ds_job_session* s, ds_knob* knob) {
  if (!s || !knob) return invalid("null argument");
  *knob = from_knob(s->session->knob());
  return DS_OK;
}

ds_status ds_job_finish(ds_job_session* s, ds_job_result** out) {
  if (!s || !out) return invalid("null argument");
  return guard([&] { *out = new ds_job_result{s->session->finish()}; });
}

void ds_job_session_free(ds_job_session* s) { delete s; }

size_t ds_job_result_records(const ds_job_result* r, ds_metrics_record* out, size_t cap) {
  if (!r) return 0;
  const auto& recs = r->trace.records;
  for (size_t i = 0; out && i < recs.size() && i < cap; ++i) {
    const auto& x = recs[i];
    out[i] = ds_metrics_record{x.time_s,  x.job_id,     from_knob(x.knob), x.p95_ms, x.mean_ms,
                               x.throughput, x.power_w, x.slo_ms,         x.violated ? 1 : 0};
  }
  return recs.size();
}

ds_status ds_job_result_summary(const ds_job_result* r, ds_job_summary* o) {
  if (!r || !o) return invalid("null argument");
  const ds::JobSummary& s = r->trace.summary;
  std::memset(o, 0, sizeof(*o));
  o->job_id = s.job_id;
  o->approach_kind = s.approach == "multi-tenancy" ? 1 : 0;
  o->profiled = s.profiled ? 1 : 0;
  o->ti_batching = s.ti_batching;
  o->ti_mt = s.ti_mt;
  o->profiling_cost_ms = s.profiling_cost_ms;
  o->steady_knob = from_knob(s.steady_knob);
  o->converged = s.converged ? 1 : 0;
  o->knob_changes = s.knob_changes;
  o->settle_period = s.settle_period;
  o->periods = s.periods;
  o->duration_s = s.duration_s;
  o->total_items = s.total_items;
  o->avg_throughput = s.avg_throughput;
  o->steady_throughput = s.steady_throughput;
  o->p95_overall_ms = s.p95_overall_ms;
  o->slo_compliance = s.slo_compliance;
  o->avg_power_w = s.avg_power_w;
  o->power_measured = s.power_measured ? 1 : 0;
  o->power_efficiency = s.power_efficiency;
  o->final_slo_ms = s.final_slo_ms;
  o->n_readaptations = static_cast<int>(s.readaptations.size());
  o->failed = s.error.empty() ? 0 : 1;
  return DS_OK;
}

namespace {
ds_profile_report to_report(const ds::ProfileReport& p) {
  return ds_profile_report{p.tput_base,         p.tput_batching,
                           p.tput_mt,           p.ti_batching,
                           p.ti_mt,             p.base_latency_ms,
                           p.probe_latency_batching_ms, p.probe_latency_mt_ms,
                           p.m,                 p.n,
                           p.batches_per_point, p.base_elapsed_ms,
                           p.batching_elapsed_ms, p.mt_elapsed_ms,
                           p.transition_ms,     p.profiling_cost_ms,
                           p.items_served};
}
}  // namespace

ds_status ds_profile_dnn(const ds_dnn_profile* catalog, int n_catalog, const char* dnn_id, int m,
                         int n, int batches, uint64_t seed, double sigma,
                         const ds_seam_spec* seam, ds_profile_report* out) {
  if (!dnn_id || !seam || !out || (n_catalog > 0 && !catalog)) return invalid("null argument");
  return guard([&] {
    const auto cat = to_catalog(catalog, n_catalog);
    const ds::DnnProfile& dnn = ds::find_dnn(cat, dnn_id);
    const double used_sigma = sigma >= 0.0 ? sigma : dnn.sigma.value_or(0.05);
    const auto bm = ds::calibrate_batching(dnn.batching_points, used_sigma);
    const auto mm = ds::calibrate_mt(dnn.mt_points, used_sigma);
    std::unique_ptr<ds::Seam> gpu;
    if (seam->kind == DS_SEAM_ANALYTIC) {
      // GpuSim(bm, mm, pm, GpuSim::Config{}, seed): the raw seed, default limits
      gpu = std::make_unique<ds::AnalyticSeam>(bm, mm, ds::Seam::Config{}, seed);
    } else {
      ds::Scenario sc;
      sc.seed = seed;
      sc.max_mtl = std::max(sc.max_mtl, n);
      sc.abs_max_bs = std::max(sc.abs_max_bs, m);
      ds::JobSpec job;
      job.dnn_id = dnn_id;
      gpu = make_factory(*seam)(sc, job, bm, mm);
    }
    *out = to_report(ds::profile(*gpu, m, n, batches));
  });
}

ds_status ds_combination_sweep(const ds_dnn_profile* catalog, int n_catalog, const char* dnn_id,
                               const int* bs_list, int n_bs, const int* mtl_list, int n_mtl,
                               int samples, uint64_t seed, double sigma, double* cells) {
  if (!dnn_id || !cells || n_bs < 0 || n_mtl < 0 || (n_bs > 0 && !bs_list) ||
      (n_mtl > 0 && !mtl_list) || (n_catalog > 0 && !catalog))
    return invalid("null argument");
  return guard([&] {
    const auto cat = to_catalog(catalog, n_catalog);
    const ds::DnnProfile& dnn = ds::find_dnn(cat, dnn_id);
    const double used_sigma = sigma >= 0.0 ? sigma : 0.0;
    const auto out = ds::combination_sweep(ds::calibrate_batching(dnn.batching_points, used_sigma),
                                           ds::calibrate_mt(dnn.mt_points, used_sigma),
                                           std::vector<int>(bs_list, bs_list + n_bs),
                                           std::vector<int>(mtl_list, mtl_list + n_mtl), samples, seed);
    for (size_t i = 0; i < out.size(); ++i) {
      double* c = cells + 5 * i;
      c[0] = out[i].bs;
      c[1] = out[i].mtl;
      c[2] = out[i].mean_ms;
      c[3] = out[i].p95_ms;
      c[4] = out[i].throughput;
    }
  });
}

ds_status ds_job_result_profile(const ds_job_result* r, ds_profile_report* o) {
  if (!r || !o) return invalid("null argument");
  *o = to_report(r->trace.report);
  return DS_OK;
}

size_t ds_job_result_tape(const ds_job_result* r, double* out, size_t cap) {
  if (!r) return 0;
  const auto& t = r->trace.tape;
  if (out) std::memcpy(out, t.data(), std::min(cap, t.size()) * sizeof(double));
  return t.size();
}

size_t ds_job_result_energy_tape(const ds_job_result* r, double* out, size_t cap) {
  if (!r) return 0;
  const auto& t = r->trace.energy_tape;
  if (out) std::memcpy(out, t.data(), std::min(cap, t.size()) * sizeof(double));
  return t.size();
}

size_t ds_job_result_latencies(const ds_job_result* r, double* out, size_t cap) {
  if (!r) return 0;
  const auto& t = r->trace.latencies;
  if (out) std::memcpy(out, t.data(), std::min(cap, t.size()) * sizeof(double));
  return t.size();
}

size_t ds_job_result_readaptations(const ds_job_result* r, double* at_s, int* periods,
                                   size_t cap) {
  if (!r) return 0;
  const auto& ra = r->trace.summary.readaptations;
  for (size_t i = 0; i < ra.size() && i < cap; ++i) {
    if (at_s) at_s[i] = ra[i].at_s;
    if (periods) periods[i] = ra[i].periods;
  }
  return ra.size();
}

const char* ds_job_result_error(const ds_job_result* r) {
  return r ? r->trace.summary.error.c_str() : "";
}

void ds_job_result_free(ds_job_result* r) { delete r; }

ds_status ds_percentile(const double* samples, size_t n, double q, double* out) {
  if (!out || (n > 0 && !samples)) return invalid("null argument");
  return guard([&] { *out = ds::percentile(std::vector<double>(samples, samples + n), q); });
}

ds_status ds_band_verdict(double p95_ms, double slo_ms, double alpha, int* verdict) {
  if (!verdict) return invalid("null argument");
  return guard([&] { *verdict = static_cast<int>(ds::band_verdict(p95_ms, slo_ms, alpha)); });
}

ds_status ds_batch_step(ds_batch_scaler* st, double p95_ms, double slo_ms, double alpha,
                        int* changed) {
  if (!st) return invalid("null argument");
  return guard([&] {
    ds::BatchScalerState s;
    s.min_bs = st->min_bs;
    s.max_bs = st->max_bs;
    s.current_bs = st->current_bs;
    s.abs_max_bs = st->abs_max_bs;
    s.infeasible = st->infeasible != 0;
    const auto d = ds::batch_step(s, p95_ms, slo_ms, alpha);
    *st = ds_batch_scaler{s.min_bs, s.max_bs, s.current_bs, s.abs_max_bs, s.infeasible ? 1 : 0};
    if (changed) *changed = d.changed ? 1 : 0;
  });
}

ds_status ds_mt_step(ds_mt_scaler* st, double p95_ms, double slo_ms, double alpha, int* action,
                     int* infeasible) {
  if (!st) return invalid("null argument");
  return guard([&] {
    ds::MtScalerState s;
    s.mtl = st->mtl;
    s.max_mtl = st->max_mtl;
    s.last_action = static_cast<ds::MtAction>(st->last_action);
    s.damped = st->damped != 0;
    const auto d = ds::mt_step(s, p95_ms, slo_ms, alpha);
    *st = ds_mt_scaler{s.mtl, s.max_mtl, static_cast<int>(s.last_action), s.damped ? 1 : 0};
    if (action) *action = static_cast<int>(d.action);
    if (infeasible) *infeasible = d.infeasible ? 1 : 0;
  });
}

ds_status ds_mt_init(double lat1_ms, double latn_ms, int n_probe, const double* rows, int n_rows,
                     int row_len, double slo_ms, int max_mtl, uint64_t seed, int* out) {
  if (!out || (n_rows > 0 && !rows)) return invalid("null argument");
  return guard([&] {
    std::vector<std::vector<double>> r;
    for (int i = 0; i < n_rows; ++i) r.emplace_back(rows + i * row_len, rows + (i + 1) * row_len);
    ds::CompletionOptions opts;
    opts.seed = seed;
    *out = ds::mt_init(lat1_ms, latn_ms, n_probe, r, slo_ms, max_mtl, opts);
  });
}

ds_status ds_estimate_row(const double* rows, int n_rows, int row_len, const int* levels,
                          const double* values, int n_obs, int width, uint64_t seed,
                          double* out) {
  if (!out || (n_rows > 0 && !rows)) return invalid("null argument");
  return guard([&] {
    std::vector<std::vector<double>> r;
    for (int i = 0; i < n_rows; ++i) r.emplace_back(rows + i * row_len, rows + (i + 1) * row_len);
    std::map<int, double> obs;
    for (int i = 0; i < n_obs; ++i) obs[levels[i]] = values[i];
    ds::CompletionOptions opts;
    opts.seed = seed;
    const auto est = ds::estimate_row(r, obs, width, opts);
    std::memcpy(out, est.data(), est.size() * sizeof(double));
  });
}

ds_status ds_decide(const ds_profile_report* r, double eps, int* approach) {
  if (!r || !approach) return invalid("null argument");
  return guard([&] {
    ds::ProfileReport p;
    p.ti_batching = r->ti_batching;
    p.ti_mt = r->ti_mt;
    p.probe_latency_batching_ms = r->probe_latency_batching_ms;
    p.probe_latency_mt_ms = r->probe_latency_mt_ms;
    *approach = ds::decide(p, eps) == ds::Approach::kMultiTenancy ? 1 : 0;
  });
}

ds_status ds_calibrate_batching(const int* x, const double* tput, int n, double* a_ms,
                                double* b_ms) {
  if (!x || !tput || !a_ms || !b_ms) return invalid("null argument");
  return guard([&] {
    std::vector<std::pair<int, double>> pts;
    for (int i = 0; i < n; ++i) pts.emplace_back(x[i], tput[i]);
    const auto m = ds::calibrate_batching(pts, 0.0);
    *a_ms = m.a_ms;
    *b_ms = m.b_ms;
  });
}

ds_status ds_calibrate_mt(const int* x, const double* tput, int n, double* l1_ms,
                          double* capacity) {
  if (!x || !tput || !l1_ms || !capacity) return invalid("null argument");
  return guard([&] {
    std::vector<std::pair<int, double>> pts;
    for (int i = 0; i < n; ++i) pts.emplace_back(x[i], tput[i]);
    const auto m = ds::calibrate_mt(pts, 0.0);
    *l1_ms = m.l1_ms;
    *capacity = m.capacity;
  });
}

}  // extern "C"
