// The B200 serving backend: the device-side replacement of the reference's
// `GpuSim` (reference gpu_sim.hpp:13-50, gpu_sim.cpp:7-46).
//
//   Instance  one co-located model replica: its own weights, activation
//             workspace, stream, and a CUDA graph per batch size.
//   Backend   GpuSim's method set over real forward passes. run_batch serves
//             one batch on instance 0; run_mt_request serves one bs=1 request
//             while every active instance keeps requests in flight on its own
//             stream; latencies are cudaEvent pairs around each request. The
//             virtual clock keeps the reference's arithmetic (clock += lat,
//             += lat/mtl, += instance-change delay) so a recorded tape replays
//             bit-exactly through the reference control plane.
#pragma once

#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels/conv_gemm.cuh"
#include "green.hpp"
#include "model.hpp"
#include "synth.hpp"

namespace ds {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char* what);

class Instance {
 public:
  Instance(const ModelSpec& m, int max_bs, int device);
  ~Instance();
  Instance(const Instance&) = delete;
  Instance& operator=(const Instance&) = delete;

  // Enqueues one forward over the first bs images of input slot `slot`
  // (graph per (bs, slot)). Two slots let the next request's H2D copy (on
  // copy_stream()) overlap the current forward.
  void enqueue_forward(int bs, int slot = 0);
  // The same forward on another stream (a green-context lane) with the
  // persistent kernels' grids sized to `sms` (0: whole device); lane_key
  // separates its graphs from the default-stream ones.
  void enqueue_forward_on(int bs, int slot, cudaStream_t s, int sms, int lane_key);
  // Same sequence without a graph (used for capture and first launch). When
  // `marks` is given (kernels_per_forward()+1 events), an externally visible
  // event is recorded before the first and after every kernel.
  void enqueue_layers(int bs, const std::vector<cudaEvent_t>* marks = nullptr, int slot = 0);
  // Device time of every kernel of one forward (staging, ops..., softmax),
  // averaged over `reps` launches of a graph with event nodes between kernels.
  std::vector<double> profile_kernels(int bs, int reps);

  cudaStream_t stream() const { return stream_; }
  // Debug: copies activation buffer `id` (first bs images) to host, raw bytes.
  void read_buffer(int id, int bs, void* host) const;
  uint8_t* images(int slot = 0) const { return d_images_[slot]; }
  cudaStream_t copy_stream() const { return copy_stream_; }
  cudaEvent_t slot_free(int slot) const { return slot_free_[slot]; }
  cudaEvent_t h2d_done(int slot) const { return h2d_done_[slot]; }
  float* logits() const { return d_logits_; }
  cudaStream_t out_stream() const { return out_stream_; }
  float* out(int slot) const { return d_out_[slot]; }
  cudaEvent_t out_ready(int slot) const { return out_ready_[slot]; }
  cudaEvent_t out_read(int slot) const { return out_read_[slot]; }
  float* probs() const { return d_probs_; }
  int max_bs() const { return max_bs_; }
  // Live per-kernel timing (pdl.cuh span_mark): zero the slots; then the
  // in-situ duration of each kernel of the forward averaged over the forwards
  // run since (returns that count, or -1 when the slots disagree).
  void reset_spans();
  int64_t read_spans(std::vector<double>* ms) const;
  int kernels_per_forward() const { return kernels_per_forward_; }
  size_t device_bytes() const { return device_bytes_; }

 private:
  struct ConvPlan {
    ConvGemmArgs args;
    ConvLoadMode mode;
    int ho, wo;
  };
  const ModelSpec& m_;
  int max_bs_;
  int device_;
  cudaStream_t stream_ = nullptr;
  cudaStream_t cur_stream_ = nullptr;  // stream enqueue_layers launches on
  void* d_arena_ = nullptr;
  size_t device_bytes_ = 0;
  uint16_t* d_w_ = nullptr;
  float* d_b_ = nullptr;
  uint8_t* d_images_[2] = {nullptr, nullptr};
  cudaStream_t copy_stream_ = nullptr;
  cudaEvent_t slot_free_[2] = {nullptr, nullptr};  // forward done reading a slot
  cudaEvent_t h2d_done_[2] = {nullptr, nullptr};   // a slot's images have landed
  cudaStream_t out_stream_ = nullptr;               // logits D2H (end-to-end mode)
  float* d_out_[2] = {nullptr, nullptr};            // per-slot logits copies
  cudaEvent_t out_ready_[2] = {nullptr, nullptr};   // a slot's logits copy written
  cudaEvent_t out_read_[2] = {nullptr, nullptr};    // ... and read back to the host
  float* d_logits_ = nullptr;
  float* d_probs_ = nullptr;
  std::vector<void*> bufs_;
  std::vector<ConvPlan> plans_;  // indexed by op (conv/fc only)
  int stem_ = -1;                // stride-1 stem conv reading the u8 images (kStemU8), or -1
  S2dPlan s2d_;                  // stride-2 stem over the space-to-depth input (kS2D)
  __nv_bfloat16* d_s2d_ = nullptr;     // [max_bs][hs][ws][16]
  __nv_bfloat16* d_stem_w_ = nullptr;  // stem weights re-laid for the s2d taps [cout][kpad]
  std::vector<CUtensorMap> dw_maps_;  // TMA halo maps of depthwise inputs (by op)
  std::vector<CUtensorMap> pool_maps_;  // TMA halo maps of pool inputs (by op)
  std::vector<bool> pool_tma_;          // pool op uses the TMA kernel (DS_POOL_TMA=0: off)
  std::map<int64_t, cudaGraphExec_t> graphs_;
  unsigned long long* d_spans_ = nullptr;  // [kernels + 1] x {sum of start times, count}
  size_t spans_bytes_ = 0;
  int kernels_per_forward_ = 0;
};

struct BackendConfig {
  int abs_max_bs = 128;  // reference gpu_sim.hpp:16
  int max_mtl = 10;      // reference gpu_sim.hpp:17
};

class Backend {
 public:
  Backend(const std::string& model_id, BackendConfig cfg, uint64_t seed, int device);
  ~Backend();
  Backend(const Backend&) = delete;
  Backend& operator=(const Backend&) = delete;

  // --- reference GpuSim method set (gpu_sim.hpp:23-40) ---
  double run_batch(int bs);
  double run_mt_request();
  double apply_instance_change(int delta);
  double set_mtl(int target);
  int mtl() const { return mtl_; }
  int device() const { return device_; }
  double clock_ms() const { return clock_ms_; }
  const BackendConfig& config() const { return cfg_; }

  // --- extensions ---
  // One control window: `count` consecutive seam calls at a fixed knob.
  void run_batches(int bs, int count, double* lat_out);
  void run_mt_requests(int count, double* lat_out);
  // B x MT combination: mtl full-size instances each serving bs-batches
  // concurrently (reference combination_sweep).
  void run_combo_requests(int bs, int mtl, int count, double* lat_out);
  // Parity path: host u8 NHWC images in, fp32 logits (and probs) out.
  void forward(const uint8_t* host_images, int bs, float* host_logits, float* host_probs);
  // End-to-end mode: every request copies its images from a pinned host pool
  // and reads its logits back inside the timed event pair.
  void set_host_io(bool enabled);
  // Output of the last request served by instance i (0: batching; 1..max_mtl-1:
  // MT; max_mtl + k - 1: combination instance k), after draining: its logits
  // (host-I/O mode: the copy that request read back) and the pool index of its
  // first image (images first .. first + bs - 1). Returns bs.
  int last_output(int i, float* host_logits, int64_t* first_image);
  // Multi-tenancy backing: 0 = concurrent streams over the whole device,
  // 1 = green-context SM partitions (green.hpp), one per active instance.
  void set_mt_mode(int mode);
  int mt_mode() const { return mt_mode_; }
  bool host_io() const { return host_io_; }
  // Drains every in-flight request (device idle on return).
  void drain();
  // Device timer over a region of serving calls: both ends drain all
  // in-flight work and record a cudaEvent, so the elapsed time covers every
  // request issued in between on every instance stream.
  void timer_start();
  double timer_stop();
  // Per-kernel device time of one bs-forward on the batching instance.
  std::vector<double> profile_kernels(int bs, int reps) {
    drain();
    return instance(0).profile_kernels(bs, reps);
  }
  // Live per-kernel timing of instance i (see Instance::read_spans).
  void reset_spans(int i) {
    drain();
    instance(i).reset_spans();
  }
  int64_t read_spans(int i, std::vector<double>* ms) {
    drain();
    return instance(i).read_spans(ms);
  }

  const ModelSpec& model() const { return model_; }
  void read_buffer(int id, int bs, void* host) { instance(0).read_buffer(id, bs, host); }
  int64_t kernel_launches() const { return kernel_launches_; }
  int kernels_per_forward() const { return inst_[0]->kernels_per_forward(); }
  int64_t h2d_bytes() const { return h2d_bytes_; }
  int64_t d2h_bytes() const { return d2h_bytes_; }
  int instances_created() const;
  size_t device_bytes() const;
  cudaStream_t batch_stream() const;

 private:
  struct Inflight {
    cudaEvent_t start, end;
    int bs;
  };
  Instance& instance(int i);
  void enqueue_request(int i, int bs);
  double complete_oldest(int i);
  cudaEvent_t take_event();

  ModelSpec model_;
  BackendConfig cfg_;
  uint64_t seed_;
  int device_;
  std::vector<std::unique_ptr<Instance>> inst_;
  std::vector<std::deque<Inflight>> inflight_;
  std::vector<cudaEvent_t> free_events_;
  std::vector<cudaEvent_t> all_events_;
  std::vector<uint8_t> host_images_;  // synthetic image pool (pageable master copy)
  uint8_t* pinned_images_ = nullptr;  // pinned copy for host-I/O mode
  std::vector<float*> pinned_logits_;
  std::vector<int64_t> io_cursor_;
  std::vector<uint64_t> io_seq_;
  std::vector<int64_t> last_first_;  // per instance: first image of the last request
  std::vector<int> last_bs_;         // ... and its batch size (0: none yet)  // per-instance request count (input slot parity)
  int pool_images_ = 0;
  bool host_io_ = false;
  int batch_bs_ = 0;  // bs of batches in flight on instance 0 (0: none)
  bool mt_active_ = false;
  int rr_ = 0;
  int mtl_ = 1;
  int mt_mode_ = 0;
  std::unique_ptr<GreenPartitions> green_;
  double clock_ms_ = 0.0;
  int64_t kernel_launches_ = 0;
  int64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
  cudaEvent_t timer_[2] = {nullptr, nullptr};
  static constexpr int kDepth = 2;  // requests kept in flight per stream
};

}  // namespace ds
