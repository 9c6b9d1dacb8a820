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

/* Parity path: u8 NHWC images [bs][h][w][3] (host memory) through the full
 * network; fp32 logits [bs][classes] and softmax probs (either may be NULL). */
ds_status ds_forward(ds_backend* b, const uint8_t* images, int bs, float* logits, float* probs);

/* End-to-end mode: each request copies its images from pinned host memory
 * and its logits back, inside the timed event pair. */
ds_status ds_set_host_io(ds_backend* b, int enabled);

/* Waits for all in-flight requests (the device is idle on return). */
ds_status ds_drain(ds_backend* b);

typedef struct {
  int in_h, in_w, classes;
  int n_ops, n_params;
  double macs_per_image;   /* algorithmic MACs (real input channels) */
  double weight_count;     /* parameters incl. biases */
  double act_bytes_per_image; /* bf16 bytes written by all layers (+input) */
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

/* The synthetic inputs: image i = RandomStream(mix_seed(seed, 1000000 + i)),
 * one byte per (h, w, c) draw (next_u64() >> 56). */
ds_status ds_generate_images(int h, int w, uint64_t seed, int64_t first, int count,
                             uint8_t* out);

/* Device-layout weights of a model (bf16 bits / fp32 bias) for oracles:
 * copies parameter layer `layer` into w (elements as laid out on device:
 * conv/fc [cout][kpad], dw [9][C]) and b; returns sizes via out pointers. */
ds_status ds_model_param(const char* model_id, int layer, uint16_t* w, size_t w_cap,
                         size_t* w_len, float* b, size_t b_cap, size_t* b_len, int* kpad);

#ifdef __cplusplus
}
#endif

#endif /* DNNSCALER_B200_H_ */
