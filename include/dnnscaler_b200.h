/*
 * dnnscaler_b200 — C ABI of the B200 serving backend.
 *
 * The reference has no FFI: its device seam is the concrete C++ class
 * dnnscaler::GpuSim (reference proj/core/include/dnnscaler/gpu_sim.hpp:13-50),
 * constructed by value inside JobRunner (harness.cpp:36-41) and taken by
 * reference by profile() (profiler.hpp:34). Each entry point below replaces
 * one GpuSim member, with the same argument meaning, error conditions and
 * messages; include/dnnscaler_b200/gpu_sim.hpp wraps them back into a
 * header-compatible `dnnscaler::GpuSim`.
 *
 * Errors: the reference throws std::invalid_argument with fixed messages;
 * here those return DS_EINVAL and the message is available from
 * ds_last_error() (thread-local). CUDA failures return DS_ECUDA.
 * A handle is single-owner: drive it from one host thread.
 */
#ifndef DNNSCALER_B200_H_
#define DNNSCALER_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ds_backend ds_backend;

typedef enum {
  DS_OK = 0,
  DS_EINVAL = 1,   /* std::invalid_argument in the reference */
  DS_ERUNTIME = 2, /* any other std::exception */
  DS_ECUDA = 3     /* CUDA driver/runtime failure */
} ds_status;

/* == GpuSim::Config (reference gpu_sim.hpp:15-18). */
typedef struct {
  int abs_max_bs;
  int max_mtl;
} ds_config;

/* Thread-local message of the last failing call on this thread. */
const char* ds_last_error(void);

/* GpuSim::GpuSim (gpu_sim.cpp:7-11). model_id: "synthetic_cnn",
 * "mobilenet_v1", "resnet50_v1", "inception_v3". seed picks the synthetic
 * image pool (weights are fixed per model). "invalid device
 * limits" when a limit is < 1. Starts at mtl = 1, clock 0. */
ds_status ds_backend_create(const char* model_id, ds_config config, uint64_t seed, int device,
                            ds_backend** out);
void ds_backend_destroy(ds_backend* b);

/* GpuSim::run_batch (gpu_sim.cpp:13-18): one forward of bs images on the
 * batching instance; latency = cudaEvent pair; clock += latency.
 * "invalid batch size" outside [1, abs_max_bs]. */
ds_status ds_run_batch(ds_backend* b, int bs, double* latency_ms);

/* GpuSim::run_mt_request (gpu_sim.cpp:20-24): one bs=1 request while all
 * mtl instances serve concurrently; clock += latency / mtl. */
ds_status ds_run_mt_request(ds_backend* b, double* latency_ms);

/* GpuSim::apply_instance_change (gpu_sim.cpp:26-37): launch (+1) or
 * terminate (-1) one instance; delay = measured launch/terminate time.
 * "instance changes are single steps", "cannot terminate last instance",
 * "instance limit exceeded". */
ds_status ds_apply_instance_change(ds_backend* b, int delta, double* delay_ms);

/* GpuSim::set_mtl (gpu_sim.cpp:39-46). */
ds_status ds_set_mtl(ds_backend* b, int target, double* total_delay_ms);

/* GpuSim::mtl / clock_ms / config (gpu_sim.hpp:35-40). */
int ds_mtl(const ds_backend* b);
double ds_clock_ms(const ds_backend* b);
ds_config ds_get_config(const ds_backend* b);

/* ---- extensions (no reference counterpart) ---- */

/* One control window at a fixed knob: `count` consecutive run_batch(bs) /
 * run_mt_request() calls, latencies in call order (identical semantics to
 * calling the single-shot functions count times). */
ds_status ds_run_batches(ds_backend* b, int bs, int count, double* latencies_ms);
ds_status ds_run_mt_requests(ds_backend* b, int count, double* latencies_ms);

/* B x MT combination (the device counterpart of the reference's analytic
 * combination_sweep cell, harness.cpp:356-386): `mtl` full-size instances on
 * their own streams, each serving batches of `bs` concurrently; `count`
 * completed-batch latencies, round robin over the instances; clock advances
 * by latency / mtl. Device-resident inputs only. */
ds_status ds_run_combo_requests(ds_backend* b, int bs, int mtl, int count, double* latencies_ms);

/* Parity path: u8 NHWC images [bs][h][w][3] (host memory) through the full
 * network; fp32 logits [bs][classes] and softmax probs (either may be NULL). */
ds_status ds_forward(ds_backend* b, const uint8_t* images, int bs, float* logits, float* probs);

/* End-to-end mode: each request copies its images from pinned host memory
 * and its logits back, inside the timed event pair. */
ds_status ds_set_host_io(ds_backend* b, int enabled);

/* Waits for all in-flight requests (the device is idle on return). */
ds_status ds_drain(ds_backend* b);

/* Live per-kernel timing inside the real graph-launched forwards (no event
 * nodes; CTA 0 of every kernel adds its %globaltimer after
 * griddepcontrol.wait into a slot): reset = 1 zeroes instance `instance`'s
 * slots; reset = 0 drains and writes each kernel's in-situ duration (ms,
 * ds_model_kernels() order, averaged over *forwards forwards since the reset)
 * to ms_out. Not in the reference. */
ds_status ds_kernel_spans(ds_backend* b, int instance, int reset, double* ms_out, int cap,
                          int64_t* forwards);

/* Multi-tenancy backing (not in the reference): 0 = every
 * co-located instance on its own stream over the whole device (default);
 * 1 = green-context SM partitions: at MT level k the SMs are split into k
 * equal groups and instance i runs on group i with grids sized to it.
 * DS_ERUNTIME when the driver has no green contexts. */
ds_status ds_set_mt_mode(ds_backend* b, int mode);
int ds_get_mt_mode(const ds_backend* b);

/* Parity aid: the output of the last request served by `instance`
 * (0 = batching instance, 1..max_mtl-1 = MT instances, max_mtl+k-1 =
 * B x MT combination instance k), after draining. logits: [bs][classes]
 * fp32 (cap elements; in host-I/O mode the copy the request itself read back
 * to pinned memory); first_image: pool index of its first image (images
 * first..first+bs-1 of ds_generate_images(seed)). Not in the reference. */
ds_status ds_last_output(ds_backend* b, int instance, float* logits, size_t cap,
                         int64_t* first_image, int* bs);

/* NVTX range markers (header-only NVTX v3; no-ops without a tool attached),
 * used to scope ncu captures to a bench's timed region. */
void ds_nvtx_push(const char* name);
void ds_nvtx_pop(void);

/* Device timer around a region of serving calls (drain + cudaEvent at both
 * ends, so every request issued in between on any instance is inside). */
ds_status ds_timer_start(ds_backend* b);
ds_status ds_timer_stop(ds_backend* b, double* elapsed_ms);

typedef struct {
  int in_h, in_w, classes;
  int n_ops, n_params;
  double macs_per_image;   /* algorithmic MACs (real input channels) */
  double weight_count;     /* parameters incl. biases */
  double act_bytes_per_image; /* bf16 bytes written by all layers (+input) */
  int feature_buffer;   /* pooled-feature buffer read by the FC (ds_debug_read_buffer id) */
  int feature_channels; /* its width (the FC's fan-in) */
  int head_k;           /* calibrated head: principal directions used (0: plain random head) */
} ds_model_info;

ds_status ds_model_info_get(const char* model_id, ds_model_info* out);

typedef struct {
  int64_t kernel_launches; /* kernels enqueued by this handle so far */
  int64_t h2d_bytes;       /* host-I/O mode copies so far */
  int64_t d2h_bytes;
  int instances_created;
  int kernels_per_forward;
  double device_bytes;
} ds_backend_stats;

ds_status ds_backend_stats_get(const ds_backend* b, ds_backend_stats* out);

/* Algorithmic cost of each kernel of one forward, launch order: input
 * staging, one per layer, softmax. kind: 0 staging, 1 conv/FC implicit GEMM,
 * 2 depthwise, 3 pool, 4 global-avg-pool, 5 softmax. A launch at batch B
 * moves B*bytes_per_image + fixed_bytes and computes B*flops_per_image. */
typedef struct {
  int kind;
  double flops_per_image;
  double bytes_per_image;
  double fixed_bytes;
} ds_kernel_cost;

ds_status ds_model_kernels(const char* model_id, ds_kernel_cost* out, int cap, int* n);

/* Device time (ms) of every kernel of one bs-forward, from cudaEvent nodes
 * captured between the kernels of a graph on the batching instance's
 * stream, averaged over reps launches. ms_out has ds_model_kernels() slots. */
ds_status ds_profile_kernels(ds_backend* b, int bs, int reps, double* ms_out, int cap);

/* Debug/parity aid: activation buffer `buffer` of the last forward on the
 * batching instance (first bs images; NHWC bf16 bits, or fp32 for logits).
 * Buffer ids follow the model IR (0 = staged input); out_len in bytes. */
ds_status ds_debug_read_buffer(ds_backend* b, int buffer, int bs, void* out, size_t cap,
                               size_t* out_len);

/* The synthetic inputs: image i = RandomStream(mix_seed(seed, 1000000 + i)),
 * one byte per (h, w, c) draw (next_u64() >> 56). */
ds_status ds_generate_images(int h, int w, uint64_t seed, int64_t first, int count,
                             uint8_t* out);

/* Device-layout weights of a model (bf16 bits / fp32 bias) for oracles:
 * copies parameter layer `layer` into w (elements as laid out on device:
 * conv/fc [cout][kpad], dw [9][C]) and b; returns sizes via out pointers. */
ds_status ds_model_param(const char* model_id, int layer, uint16_t* w, size_t w_cap,
                         size_t* w_len, float* b, size_t b_cap, size_t* b_len, int* kpad);

/* ======================================================================
 * Control plane (the reference's Profiler / Scaler / harness over a seam).
 * Replaces reference harness.hpp:54-80 (run_job / run_scenario),
 * profiler.hpp:34-38, scaler.hpp:13-70, matrix_completion.hpp:39-49.
 * ====================================================================== */

typedef struct {
  int kind; /* 0 batching, 1 multi-tenancy (reference KnobKind) */
  int value;
} ds_knob;

typedef struct {
  double at_s;
  double slo_ms;
} ds_slo_step;

/* == JobSpec (reference domain.hpp:41-48). */
typedef struct {
  int job_id;
  const char* dnn_id; /* catalog id; for the device seam also the model id */
  double slo_ms;
  double duration_s;
  int n_slo_steps;
  const ds_slo_step* slo_steps;
} ds_job_spec;

/* == DnnProfile (reference domain.hpp:26-34): (x, items/s) points. */
typedef struct {
  const char* id;
  int n_batching;
  const int* batching_x;
  const double* batching_tput;
  int n_mt;
  const int* mt_x;
  const double* mt_tput;
  int has_sigma;
  double sigma;
  int has_u1;
  double u1;
} ds_dnn_profile;

/* == Scenario (reference scenario.hpp:17-30), catalog passed separately. */
typedef struct {
  int controller; /* 0 dnnscaler, 1 clipper, 2 static */
  ds_knob static_knob;
  uint64_t seed;
  double alpha;
  int m, n, abs_max_bs, max_mtl, window;
  double sigma;
} ds_scenario;

typedef enum {
  DS_SEAM_ANALYTIC = 0, /* the reference's simulated GpuSim (perf model) */
  DS_SEAM_DEVICE = 1,   /* the B200 backend */
  DS_SEAM_REPLAY = 2    /* a recorded tape */
} ds_seam_kind;

typedef struct {
  int kind;
  ds_backend* backend; /* DEVICE: existing handle to serve on, or NULL to create one
                          per job (model = dnn_id, seed = mix_seed(seed, job_id)) */
  int device;          /* DEVICE with backend == NULL: CUDA ordinal */
  int host_io;         /* DEVICE with backend == NULL: end-to-end copies */
  const double* tape;  /* REPLAY */
  size_t tape_len;
  const double* energy_tape; /* REPLAY (optional): (mJ, wall ms, W) triples of a device run */
  size_t energy_tape_len;
} ds_seam_spec;

typedef struct {
  double time_s;
  int job_id;
  ds_knob knob;
  double p95_ms, mean_ms, throughput, power_w, slo_ms;
  int violated;
} ds_metrics_record;

/* == ProfileReport (reference profiler.hpp:11-29). */
typedef struct {
  double tput_base, tput_batching, tput_mt, ti_batching, ti_mt;
  double base_latency_ms, probe_latency_batching_ms, probe_latency_mt_ms;
  int m, n, batches_per_point;
  double base_elapsed_ms, batching_elapsed_ms, mt_elapsed_ms, transition_ms;
  double profiling_cost_ms, items_served;
} ds_profile_report;

/* == JobSummary (reference harness.hpp:19-43) minus strings. */
typedef struct {
  int job_id;
  int approach_kind; /* knob kind actually controlled */
  int profiled;
  double ti_batching, ti_mt, profiling_cost_ms;
  ds_knob steady_knob;
  int converged, knob_changes, settle_period, periods;
  double duration_s, total_items, avg_throughput, steady_throughput, p95_overall_ms;
  double slo_compliance, avg_power_w, power_efficiency, final_slo_ms;
  int n_readaptations;
  int failed; /* run_scenario semantics: error captured, see ds_job_result_error */
  int power_measured; /* 1: avg_power_w / power_efficiency / power_w from the board's
                         NVML energy counter (efficiency = inferences per joule),
                         0: the reference PowerModel */
} ds_job_summary;

typedef struct ds_job_result ds_job_result;

/* run_job (reference harness.cpp:329-333) on the given seam. A job that
 * throws yields a result with failed = 1 and its message (run_scenario
 * semantics, harness.cpp:341-351); the call itself returns DS_OK. */
ds_status ds_job_run(const ds_scenario* scenario, const ds_job_spec* job,
                     const ds_dnn_profile* catalog, int n_catalog, const ds_seam_spec* seam,
                     ds_job_result** out);

/* Incremental form: start (profile + seed the knob), then one control period
 * per ds_job_step, then ds_job_finish for the summary. */
typedef struct ds_job_session ds_job_session;
ds_status ds_job_start(const ds_scenario* scenario, const ds_job_spec* job,
                       const ds_dnn_profile* catalog, int n_catalog, const ds_seam_spec* seam,
                       ds_job_session** out);
ds_status ds_job_step(ds_job_session* s, ds_metrics_record* record, int* done);
ds_status ds_job_knob(const ds_job_session* s, ds_knob* knob);
ds_status ds_job_finish(ds_job_session* s, ds_job_result** out);
void ds_job_session_free(ds_job_session* s);

size_t ds_job_result_records(const ds_job_result* r, ds_metrics_record* out, size_t cap);
ds_status ds_job_result_summary(const ds_job_result* r, ds_job_summary* out);
ds_status ds_job_result_profile(const ds_job_result* r, ds_profile_report* out);
/* The B x MT grid on a catalog network's analytic model (reference
 * harness.cpp:356-386, CLI cmd_sweep at dnnscaler_main.cpp:186-199; sigma < 0
 * means 0, as the CLI does): n_bs * n_mtl cells, bs-major, each
 * (bs, mtl, mean_ms, p95_ms, throughput) written as 5 doubles to cells. */
ds_status ds_combination_sweep(const ds_dnn_profile* catalog, int n_catalog, const char* dnn_id,
                               const int* bs_list, int n_bs, const int* mtl_list, int n_mtl,
                               int samples, uint64_t seed, double sigma, double* cells);
/* The Profiler alone on one catalog network (reference tools/dnnscaler_main.cpp:88-99,
 * cmd_profile): sigma < 0 takes the catalog's sigma (else 0.05); the ANALYTIC
 * seam is GpuSim(bm, mm, pm, Config{}, seed) with the raw seed, as the
 * reference CLI builds it; DEVICE probes dnn_id on the B200. */
ds_status ds_profile_dnn(const ds_dnn_profile* catalog, int n_catalog, const char* dnn_id, int m,
                         int n, int batches, uint64_t seed, double sigma,
                         const ds_seam_spec* seam, ds_profile_report* out);
size_t ds_job_result_tape(const ds_job_result* r, double* out, size_t cap);
/* (mJ, wall ms, W) energy readings of a device run, for ds_seam_spec.energy_tape. */
size_t ds_job_result_energy_tape(const ds_job_result* r, double* out, size_t cap);
size_t ds_job_result_latencies(const ds_job_result* r, double* out, size_t cap);
size_t ds_job_result_readaptations(const ds_job_result* r, double* at_s, int* periods, size_t cap);
const char* ds_job_result_error(const ds_job_result* r);
void ds_job_result_free(ds_job_result* r);

/* Single controller steps, for unit parity with the reference goldens. */
ds_status ds_percentile(const double* samples, size_t n, double q, double* out);
ds_status ds_band_verdict(double p95_ms, double slo_ms, double alpha, int* verdict /*0 below,1 in,2 above*/);

typedef struct {
  int min_bs, max_bs, current_bs, abs_max_bs, infeasible;
} ds_batch_scaler;
ds_status ds_batch_step(ds_batch_scaler* st, double p95_ms, double slo_ms, double alpha,
                        int* changed);

typedef struct {
  int mtl, max_mtl, last_action /*0 hold,1 add,2 remove*/, damped;
} ds_mt_scaler;
ds_status ds_mt_step(ds_mt_scaler* st, double p95_ms, double slo_ms, double alpha, int* action,
                     int* infeasible);

ds_status ds_mt_init(double lat1_ms, double latn_ms, int n_probe, const double* rows,
                     int n_rows, int row_len, double slo_ms, int max_mtl, uint64_t seed,
                     int* out);
ds_status ds_estimate_row(const double* rows, int n_rows, int row_len, const int* levels,
                          const double* values, int n_obs, int width, uint64_t seed,
                          double* out);
ds_status ds_decide(const ds_profile_report* r, double eps, int* approach /*0 B, 1 MT*/);
ds_status ds_calibrate_batching(const int* x, const double* tput, int n, double* a_ms,
                                double* b_ms);
ds_status ds_calibrate_mt(const int* x, const double* tput, int n, double* l1_ms,
                          double* capacity);

#ifdef __cplusplus
}
#endif

#endif /* DNNSCALER_B200_H_ */
