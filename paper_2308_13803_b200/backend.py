"""Python mirror of the reference device seam `dnnscaler::GpuSim`
(reference proj/core/include/dnnscaler/gpu_sim.hpp:13-50) over the B200
backend's C ABI. Same method names, argument meaning and error behaviour:
the reference's std::invalid_argument surfaces as ValueError with the same
message; CUDA failures raise DsError.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

MODELS = ("synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3")


@dataclass(frozen=True)
class Config:
    """== GpuSim::Config (gpu_sim.hpp:15-18)."""

    abs_max_bs: int = 128
    max_mtl: int = 10


@dataclass(frozen=True)
class ModelInfo:
    in_h: int
    in_w: int
    classes: int
    n_ops: int
    n_params: int
    macs_per_image: float
    weight_count: float
    act_bytes_per_image: float
    feature_buffer: int
    feature_channels: int
    head_k: int


def model_info(model_id: str) -> ModelInfo:
    lib = _lib.load()
    mi = _lib.DsModelInfo()
    _lib.check(lib.ds_model_info_get(model_id.encode(), ctypes.byref(mi)))
    return ModelInfo(mi.in_h, mi.in_w, mi.classes, mi.n_ops, mi.n_params, mi.macs_per_image,
                     mi.weight_count, mi.act_bytes_per_image, mi.feature_buffer,
                     mi.feature_channels, mi.head_k)


KERNEL_KINDS = ("stage", "conv_gemm", "dwconv", "pool", "gap", "softmax")


def kernel_costs(model_id: str) -> list:
    """Per-kernel algorithmic cost of one forward (launch order)."""
    lib = _lib.load()
    n = ctypes.c_int()
    _lib.check(lib.ds_model_kernels(model_id.encode(), None, 0, ctypes.byref(n)))
    arr = (_lib.DsKernelCost * n.value)()
    _lib.check(lib.ds_model_kernels(model_id.encode(), arr, n.value, ctypes.byref(n)))
    return [dict(kind=KERNEL_KINDS[c.kind], flops_per_image=c.flops_per_image,
                 bytes_per_image=c.bytes_per_image, fixed_bytes=c.fixed_bytes) for c in arr]


def generate_images(model_id: str, first: int, count: int, seed: int = 42) -> np.ndarray:
    """The synthetic inputs of DESIGN.md: u8 NHWC [count, h, w, 3]."""
    info = model_info(model_id)
    out = np.empty((count, info.in_h, info.in_w, 3), dtype=np.uint8)
    _lib.check(_lib.load().ds_generate_images(info.in_h, info.in_w, seed, first, count,
                                              out.ctypes.data))
    return out


class GpuBackend:
    """One serving backend on one GPU (single-owner, not thread-safe)."""

    def __init__(self, model_id: str, config: Config = Config(), seed: int = 42, device: int = 0):
        lib = _lib.load()
        self._lib = lib
        self._h = ctypes.c_void_p()
        _lib.check(lib.ds_backend_create(model_id.encode(),
                                         _lib.DsConfig(config.abs_max_bs, config.max_mtl),
                                         seed, device, ctypes.byref(self._h)))
        self.model_id = model_id
        self.info = model_info(model_id)
        self._config = config

    # ---- reference GpuSim method set -------------------------------------
    def run_batch(self, bs: int) -> float:
        lat = ctypes.c_double()
        _lib.check(self._lib.ds_run_batch(self._h, bs, ctypes.byref(lat)))
        return lat.value

    def run_mt_request(self) -> float:
        lat = ctypes.c_double()
        _lib.check(self._lib.ds_run_mt_request(self._h, ctypes.byref(lat)))
        return lat.value

    def apply_instance_change(self, delta: int) -> float:
        d = ctypes.c_double()
        _lib.check(self._lib.ds_apply_instance_change(self._h, delta, ctypes.byref(d)))
        return d.value

    def set_mtl(self, target: int) -> float:
        d = ctypes.c_double()
        _lib.check(self._lib.ds_set_mtl(self._h, target, ctypes.byref(d)))
        return d.value

    def mtl(self) -> int:
        return self._lib.ds_mtl(self._h)

    def clock_ms(self) -> float:
        return self._lib.ds_clock_ms(self._h)

    def config(self) -> Config:
        c = self._lib.ds_get_config(self._h)
        return Config(c.abs_max_bs, c.max_mtl)

    # ---- extensions --------------------------------------------------------
    def run_batches(self, bs: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        _lib.check(self._lib.ds_run_batches(self._h, bs, count, out.ctypes.data))
        return out

    def run_mt_requests(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        _lib.check(self._lib.ds_run_mt_requests(self._h, count, out.ctypes.data))
        return out

    def run_combo_requests(self, bs: int, mtl: int, count: int) -> np.ndarray:
        """B x MT: mtl instances each serving bs-batches concurrently."""
        out = np.empty(count, dtype=np.float64)
        _lib.check(self._lib.ds_run_combo_requests(self._h, bs, mtl, count, out.ctypes.data))
        return out

    def combination_sweep(self, bs_list, mtl_list, samples_per_cell: int = 50) -> list:
        """Device counterpart of the reference combination_sweep
        (harness.cpp:356-386): per (bs, mtl) cell the mean and nearest-rank p95
        of the per-instance batch latency and throughput = bs * mtl * 1000 /
        mean (the reference's formula), plus the throughput measured on the
        device clock over the cell."""
        from . import control as C
        if not bs_list or not mtl_list:
            raise ValueError("empty sweep grid")
        if samples_per_cell < 1:
            raise ValueError("samples_per_cell must be positive")
        cells = []
        for bs in bs_list:
            for mtl in mtl_list:
                self.run_combo_requests(bs, mtl, 2 * mtl)  # warm-up (instances, graphs)
                self.timer_start()
                lat = self.run_combo_requests(bs, mtl, samples_per_cell)
                ms = self.timer_stop()
                mean = float(lat.mean())
                cells.append({"bs": bs, "mtl": mtl, "mean_ms": mean,
                              "p95_ms": C.percentile(lat, 0.95),
                              "throughput": bs * mtl * 1000.0 / mean,
                              "measured_throughput": bs * samples_per_cell * 1000.0 / ms})
        return cells

    def forward(self, images: np.ndarray, probs: bool = False):
        images = np.ascontiguousarray(images, dtype=np.uint8)
        bs = images.shape[0]
        logits = np.empty((bs, self.info.classes), dtype=np.float32)
        p = np.empty_like(logits) if probs else None
        _lib.check(self._lib.ds_forward(self._h, images.ctypes.data, bs, logits.ctypes.data,
                                        p.ctypes.data if probs else None))
        return (logits, p) if probs else logits

    def set_host_io(self, enabled: bool) -> None:
        _lib.check(self._lib.ds_set_host_io(self._h, 1 if enabled else 0))

    def last_output(self, instance: int = 0):
        """(logits [bs, classes], first_image) of the last request the
        instance served (0 batching, 1..max_mtl-1 MT, max_mtl+k-1 combo k)."""
        cap = self._config.abs_max_bs * self.info.classes
        buf = np.empty(cap, dtype=np.float32)
        first, bs = ctypes.c_int64(), ctypes.c_int()
        _lib.check(self._lib.ds_last_output(self._h, instance, buf.ctypes.data, cap,
                                            ctypes.byref(first), ctypes.byref(bs)))
        return buf[:bs.value * self.info.classes].reshape(bs.value, self.info.classes).copy(), first.value

    def set_mt_mode(self, mode: str) -> None:
        """'streams' (default) or 'green' (green-context SM partitions)."""
        _lib.check(self._lib.ds_set_mt_mode(self._h, {"streams": 0, "green": 1}[mode]))

    def mt_mode(self) -> str:
        return ("streams", "green")[self._lib.ds_get_mt_mode(self._h)]

    def drain(self) -> None:
        _lib.check(self._lib.ds_drain(self._h))

    def timer_start(self) -> None:
        _lib.check(self._lib.ds_timer_start(self._h))

    def timer_stop(self) -> float:
        ms = ctypes.c_double()
        _lib.check(self._lib.ds_timer_stop(self._h, ctypes.byref(ms)))
        return ms.value

    def profile_kernels(self, bs: int, reps: int = 10) -> np.ndarray:
        """Device ms of every kernel of one bs-forward (event nodes in a graph)."""
        n = len(kernel_costs(self.model_id))
        out = np.empty(n, dtype=np.float64)
        _lib.check(self._lib.ds_profile_kernels(self._h, bs, reps, out.ctypes.data, n))
        return out

    def reset_kernel_spans(self, instance: int = 0) -> None:
        """Zero the live per-kernel timing slots of an instance."""
        n = ctypes.c_int64()
        _lib.check(self._lib.ds_kernel_spans(self._h, instance, 1, None, 0, ctypes.byref(n)))

    def kernel_spans(self, instance: int = 0):
        """(ms per kernel of the forward, forwards) measured live since the
        last reset, inside the real graph launches (ds_kernel_spans)."""
        k = len(kernel_costs(self.model_id))
        out = np.zeros(k, dtype=np.float64)
        n = ctypes.c_int64()
        _lib.check(self._lib.ds_kernel_spans(self._h, instance, 0, out.ctypes.data, k,
                                             ctypes.byref(n)))
        return out, n.value

    def stats(self) -> dict:
        s = _lib.DsBackendStats()
        _lib.check(self._lib.ds_backend_stats_get(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_}

    def close(self) -> None:
        if self._h:
            self._lib.ds_backend_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
