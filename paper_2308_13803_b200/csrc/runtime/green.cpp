#include "green.hpp"

#include <mutex>
#include <stdexcept>
#include <string>

namespace ds {

namespace {

// Driver entry points through the runtime (no -lcuda link).
struct GreenApi {
  CUresult (*device_get)(CUdevice*, int) = nullptr;
  CUresult (*get_dev_resource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split_by_count)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*,
                             unsigned, unsigned) = nullptr;
  CUresult (*generate_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*ctx_create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*ctx_destroy)(CUgreenCtx) = nullptr;
  CUresult (*stream_create)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const GreenApi& api() {
  static GreenApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    a.ok = entry("cuDeviceGet", &a.device_get) &&
           entry("cuDeviceGetDevResource", &a.get_dev_resource) &&
           entry("cuDevSmResourceSplitByCount", &a.split_by_count) &&
           entry("cuDevResourceGenerateDesc", &a.generate_desc) &&
           entry("cuGreenCtxCreate", &a.ctx_create) &&
           entry("cuGreenCtxDestroy", &a.ctx_destroy) &&
           entry("cuGreenCtxStreamCreate", &a.stream_create);
  });
  return a;
}

void check_cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS)
    throw std::runtime_error(std::string("green context: ") + what + " failed (CUresult " +
                             std::to_string(static_cast<int>(r)) + ")");
}

}  // namespace

bool green_contexts_supported() { return api().ok; }

GreenPartitions::GreenPartitions(int device) : device_(device) {
  if (!api().ok) throw std::runtime_error("green contexts: driver entry points unavailable");
  cudaDeviceGetAttribute(&device_sms_, cudaDevAttrMultiProcessorCount, device_);
}

GreenPartitions::~GreenPartitions() {
  cudaSetDevice(device_);
  for (auto& kv : levels_)
    for (auto& l : kv.second) {
      if (l.stream) {
        cudaStreamSynchronize(l.stream);
        cudaStreamDestroy(l.stream);
      }
      if (l.ctx) api().ctx_destroy(l.ctx);
    }
}

const std::vector<GreenLane>& GreenPartitions::level(int k) {
  if (k < 1) throw std::invalid_argument("green partition level must be positive");
  auto it = levels_.find(k);
  if (it != levels_.end()) return it->second;
  const GreenApi& a = api();
  CUdevice dev;
  check_cu(a.device_get(&dev, device_), "cuDeviceGet");
  CUdevResource all{};
  check_cu(a.get_dev_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  const unsigned per = static_cast<unsigned>(all.sm.smCount) / static_cast<unsigned>(k);
  std::vector<CUdevResource> groups(k);
  unsigned n = static_cast<unsigned>(k);
  CUdevResource rest{};
  check_cu(a.split_by_count(groups.data(), &n, &all, &rest, 0, per > 0 ? per : 1),
           "cuDevSmResourceSplitByCount");
  if (n == 0) throw std::runtime_error("green contexts: SM split produced no groups");
  std::vector<GreenLane> lanes;
  for (unsigned g = 0; g < n; ++g) {
    CUdevResourceDesc desc;
    check_cu(a.generate_desc(&desc, &groups[g], 1), "cuDevResourceGenerateDesc");
    GreenLane l;
    check_cu(a.ctx_create(&l.ctx, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    CUstream s;
    check_cu(a.stream_create(&s, l.ctx, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
    l.stream = reinterpret_cast<cudaStream_t>(s);
    l.sms = static_cast<int>(groups[g].sm.smCount);
    lanes.push_back(l);
  }
  return levels_.emplace(k, std::move(lanes)).first->second;
}

}  // namespace ds
