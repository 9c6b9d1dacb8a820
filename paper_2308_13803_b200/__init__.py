"""DNNScaler on B200: a device backend for the reference's GpuSim seam
(hand-written sm_100a kernels behind a C ABI) plus the host control plane
(Profiler / Scaler / harness) restated in C++. See DESIGN.md."""
from .backend import Config, GpuBackend, MODELS, generate_images, model_info  # noqa: F401
