"""Python mirror of the reference control plane API (scenario.hpp, domain.hpp,
harness.hpp, profiler.hpp, scaler.hpp, matrix_completion.hpp) over the C
ABI. The logic itself runs in C++ inside libdnnscaler_b200.so.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .backend import GpuBackend

# ---------------------------------------------------------------- C structs


class _Knob(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("value", ctypes.c_int)]


class _SloStep(ctypes.Structure):
    _fields_ = [("at_s", ctypes.c_double), ("slo_ms", ctypes.c_double)]


class _JobSpec(ctypes.Structure):
    _fields_ = [("job_id", ctypes.c_int), ("dnn_id", ctypes.c_char_p), ("slo_ms", ctypes.c_double),
                ("duration_s", ctypes.c_double), ("n_slo_steps", ctypes.c_int),
                ("slo_steps", ctypes.POINTER(_SloStep))]


class _DnnProfile(ctypes.Structure):
    _fields_ = [("id", ctypes.c_char_p), ("n_batching", ctypes.c_int),
                ("batching_x", ctypes.POINTER(ctypes.c_int)),
                ("batching_tput", ctypes.POINTER(ctypes.c_double)), ("n_mt", ctypes.c_int),
                ("mt_x", ctypes.POINTER(ctypes.c_int)), ("mt_tput", ctypes.POINTER(ctypes.c_double)),
                ("has_sigma", ctypes.c_int), ("sigma", ctypes.c_double), ("has_u1", ctypes.c_int),
                ("u1", ctypes.c_double)]


class _Scenario(ctypes.Structure):
    _fields_ = [("controller", ctypes.c_int), ("static_knob", _Knob), ("seed", ctypes.c_uint64),
                ("alpha", ctypes.c_double), ("m", ctypes.c_int), ("n", ctypes.c_int),
                ("abs_max_bs", ctypes.c_int), ("max_mtl", ctypes.c_int), ("window", ctypes.c_int),
                ("sigma", ctypes.c_double)]


class _SeamSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("backend", ctypes.c_void_p), ("device", ctypes.c_int),
                ("host_io", ctypes.c_int), ("tape", ctypes.POINTER(ctypes.c_double)),
                ("tape_len", ctypes.c_size_t), ("energy_tape", ctypes.POINTER(ctypes.c_double)),
                ("energy_tape_len", ctypes.c_size_t)]


class _Record(ctypes.Structure):
    _fields_ = [("time_s", ctypes.c_double), ("job_id", ctypes.c_int), ("knob", _Knob),
                ("p95_ms", ctypes.c_double), ("mean_ms", ctypes.c_double),
                ("throughput", ctypes.c_double), ("power_w", ctypes.c_double),
                ("slo_ms", ctypes.c_double), ("violated", ctypes.c_int)]


class _Report(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "tput_base", "tput_batching", "tput_mt", "ti_batching", "ti_mt", "base_latency_ms",
        "probe_latency_batching_ms", "probe_latency_mt_ms")] + [
        ("m", ctypes.c_int), ("n", ctypes.c_int), ("batches_per_point", ctypes.c_int)] + [
        (n, ctypes.c_double) for n in ("base_elapsed_ms", "batching_elapsed_ms", "mt_elapsed_ms",
                                       "transition_ms", "profiling_cost_ms", "items_served")]


class _Summary(ctypes.Structure):
    _fields_ = [("job_id", ctypes.c_int), ("approach_kind", ctypes.c_int), ("profiled", ctypes.c_int),
                ("ti_batching", ctypes.c_double), ("ti_mt", ctypes.c_double),
                ("profiling_cost_ms", ctypes.c_double), ("steady_knob", _Knob),
                ("converged", ctypes.c_int), ("knob_changes", ctypes.c_int),
                ("settle_period", ctypes.c_int), ("periods", ctypes.c_int)] + [
        (n, ctypes.c_double) for n in (
            "duration_s", "total_items", "avg_throughput", "steady_throughput", "p95_overall_ms",
            "slo_compliance", "avg_power_w", "power_efficiency", "final_slo_ms")] + [
        ("n_readaptations", ctypes.c_int), ("failed", ctypes.c_int),
        ("power_measured", ctypes.c_int)]


class _BatchScaler(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("min_bs", "max_bs", "current_bs", "abs_max_bs",
                                            "infeasible")]


class _MtScaler(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("mtl", "max_mtl", "last_action", "damped")]


_P = ctypes.POINTER
_vp = ctypes.c_void_p
_SIGS = {
    "ds_job_run": (ctypes.c_int, [_P(_Scenario), _P(_JobSpec), _P(_DnnProfile), ctypes.c_int,
                                  _P(_SeamSpec), _P(_vp)]),
    "ds_job_start": (ctypes.c_int, [_P(_Scenario), _P(_JobSpec), _P(_DnnProfile), ctypes.c_int,
                                    _P(_SeamSpec), _P(_vp)]),
    "ds_job_step": (ctypes.c_int, [_vp, _P(_Record), _P(ctypes.c_int)]),
    "ds_job_knob": (ctypes.c_int, [_vp, _P(_Knob)]),
    "ds_job_finish": (ctypes.c_int, [_vp, _P(_vp)]),
    "ds_job_session_free": (None, [_vp]),
    "ds_job_result_records": (ctypes.c_size_t, [_vp, _P(_Record), ctypes.c_size_t]),
    "ds_job_result_summary": (ctypes.c_int, [_vp, _P(_Summary)]),
    "ds_job_result_profile": (ctypes.c_int, [_vp, _P(_Report)]),
    "ds_combination_sweep": (ctypes.c_int, [_P(_DnnProfile), ctypes.c_int, ctypes.c_char_p, _vp,
                                            ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_uint64, ctypes.c_double, _vp]),
    "ds_profile_dnn": (ctypes.c_int, [_P(_DnnProfile), ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                      _P(_SeamSpec), _P(_Report)]),
    "ds_job_result_tape": (ctypes.c_size_t, [_vp, _vp, ctypes.c_size_t]),
    "ds_job_result_energy_tape": (ctypes.c_size_t, [_vp, _vp, ctypes.c_size_t]),
    "ds_job_result_latencies": (ctypes.c_size_t, [_vp, _vp, ctypes.c_size_t]),
    "ds_job_result_readaptations": (ctypes.c_size_t, [_vp, _vp, _vp, ctypes.c_size_t]),
    "ds_job_result_error": (ctypes.c_char_p, [_vp]),
    "ds_job_result_free": (None, [_vp]),
    "ds_percentile": (ctypes.c_int, [_vp, ctypes.c_size_t, ctypes.c_double, _P(ctypes.c_double)]),
    "ds_band_verdict": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       _P(ctypes.c_int)]),
    "ds_batch_step": (ctypes.c_int, [_P(_BatchScaler), ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, _P(ctypes.c_int)]),
    "ds_mt_step": (ctypes.c_int, [_P(_MtScaler), ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, _P(ctypes.c_int), _P(ctypes.c_int)]),
    "ds_mt_init": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, ctypes.c_int, _vp, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_uint64,
                                  _P(ctypes.c_int)]),
    "ds_estimate_row": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_uint64, _vp]),
    "ds_decide": (ctypes.c_int, [_P(_Report), ctypes.c_double, _P(ctypes.c_int)]),
    "ds_calibrate_batching": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _P(ctypes.c_double),
                                             _P(ctypes.c_double)]),
    "ds_calibrate_mt": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _P(ctypes.c_double),
                                       _P(ctypes.c_double)]),
}

_bound = None


def _l():
    global _bound
    lib = _lib.load()
    if _bound is None:
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _bound = lib
    return lib


# ---------------------------------------------------------------- Python types

BATCHING, MULTI_TENANCY = 0, 1
CONTROLLERS = {"dnnscaler": 0, "clipper": 1, "static": 2}


@dataclass
class DnnProfile:
    """== reference DnnProfile (domain.hpp:26-34)."""

    id: str
    batching_points: list
    mt_points: list
    params_millions: float = 1.0
    mflops: float = 1.0
    sigma: Optional[float] = None
    u1: Optional[float] = None

    def to_json(self) -> dict:
        d = {"id": self.id, "params_millions": self.params_millions, "mflops": self.mflops,
             "batching_points": [[int(x), float(t)] for x, t in self.batching_points],
             "mt_points": [[int(x), float(t)] for x, t in self.mt_points]}
        if self.sigma is not None:
            d["sigma"] = self.sigma
        if self.u1 is not None:
            d["u1"] = self.u1
        return d


def load_catalog(path: str) -> list:
    """Reads a reference-format catalog JSON (catalog.cpp:51-94 schema)."""
    with open(path) as f:
        doc = json.load(f)
    return [DnnProfile(id=e["id"], batching_points=[tuple(p) for p in e["batching_points"]],
                       mt_points=[tuple(p) for p in e["mt_points"]],
                       params_millions=e.get("params_millions", 1.0), mflops=e.get("mflops", 1.0),
                       sigma=e.get("sigma"), u1=e.get("u1")) for e in doc]


@dataclass
class JobSpec:
    """== reference JobSpec (domain.hpp:41-48)."""

    job_id: int
    dnn_id: str
    slo_ms: float
    duration_s: float
    slo_schedule: list = field(default_factory=list)  # [(at_s, slo_ms)]
    dataset_tag: str = ""


@dataclass
class Scenario:
    """== reference Scenario (scenario.hpp:17-30)."""

    controller: str = "dnnscaler"
    static_knob: tuple = (BATCHING, 1)
    seed: int = 42
    alpha: float = 0.85
    m: int = 32
    n: int = 8
    abs_max_bs: int = 128
    max_mtl: int = 10
    window: int = 100
    sigma: float = 0.05

    def to_json(self, jobs: Sequence[JobSpec], catalog_path: str) -> dict:
        d = {"catalog_path": catalog_path, "controller": self.controller, "seed": self.seed,
             "alpha": self.alpha, "m": self.m, "n": self.n, "abs_max_bs": self.abs_max_bs,
             "max_mtl": self.max_mtl, "window": self.window, "sigma": self.sigma,
             "jobs": [{"job_id": j.job_id, "dnn_id": j.dnn_id, "slo_ms": j.slo_ms,
                       "duration_s": j.duration_s,
                       **({"slo_schedule": [list(s) for s in j.slo_schedule]}
                          if j.slo_schedule else {})} for j in jobs]}
        if self.controller == "static":
            d["static_knob"] = {"kind": "batching" if self.static_knob[0] == BATCHING
                                else "multi-tenancy", "value": self.static_knob[1]}
        return d


@dataclass
class JobResult:
    records: np.ndarray  # [periods, 10]: time_s, job_id, kind, value, p95, mean, tput, power, slo, violated
    summary: dict
    report: dict
    tape: np.ndarray
    latencies: np.ndarray
    readaptations: list
    error: str
    energy_tape: np.ndarray = None  # (mJ, wall ms) readings of a device run


class _Marshal:
    """Keeps ctypes buffers alive for one call."""

    def __init__(self, scenario: Scenario, job: JobSpec, catalog: Sequence[DnnProfile]):
        self.keep = []
        self.sc = _Scenario(CONTROLLERS[scenario.controller],
                            _Knob(int(scenario.static_knob[0]), int(scenario.static_knob[1])),
                            scenario.seed, scenario.alpha, scenario.m, scenario.n,
                            scenario.abs_max_bs, scenario.max_mtl, scenario.window, scenario.sigma)
        steps = (_SloStep * max(1, len(job.slo_schedule)))(*[_SloStep(a, s)
                                                            for a, s in job.slo_schedule])
        self.keep.append(steps)
        self.job = _JobSpec(job.job_id, job.dnn_id.encode(), job.slo_ms, job.duration_s,
                            len(job.slo_schedule), steps)
        arr = (_DnnProfile * max(1, len(catalog)))()
        for i, p in enumerate(catalog):
            bx = (ctypes.c_int * len(p.batching_points))(*[int(x) for x, _ in p.batching_points])
            bt = (ctypes.c_double * len(p.batching_points))(*[float(t) for _, t in p.batching_points])
            mx = (ctypes.c_int * len(p.mt_points))(*[int(x) for x, _ in p.mt_points])
            mt = (ctypes.c_double * len(p.mt_points))(*[float(t) for _, t in p.mt_points])
            pid = p.id.encode()
            self.keep += [bx, bt, mx, mt, pid]
            arr[i] = _DnnProfile(pid, len(p.batching_points), bx, bt, len(p.mt_points), mx, mt,
                                 int(p.sigma is not None), p.sigma or 0.0, int(p.u1 is not None),
                                 p.u1 or 0.0)
        self.catalog = arr
        self.n_catalog = len(catalog)

    def seam(self, kind: str, backend: Optional[GpuBackend] = None, device: int = 0,
             host_io: bool = False, tape: Optional[np.ndarray] = None,
             energy_tape: Optional[np.ndarray] = None) -> _SeamSpec:
        k = {"analytic": 0, "device": 1, "replay": 2}[kind]

        def arr(x):
            if x is None:
                return None, 0
            a = np.ascontiguousarray(x, dtype=np.float64)
            self.keep.append(a)
            return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), a.size

        t, tn = arr(tape)
        e, en = arr(energy_tape)
        return _SeamSpec(k, backend._h if backend is not None else None, device, int(host_io),
                         t, tn, e, en)


def _collect(lib, res) -> JobResult:
    n = lib.ds_job_result_records(res, None, 0)
    recs = (_Record * max(1, n))()
    lib.ds_job_result_records(res, recs, n)
    records = np.array([[r.time_s, r.job_id, r.knob.kind, r.knob.value, r.p95_ms, r.mean_ms,
                         r.throughput, r.power_w, r.slo_ms, r.violated] for r in recs[:n]],
                       dtype=np.float64).reshape(n, 10)
    s = _Summary()
    lib.ds_job_result_summary(res, ctypes.byref(s))
    summary = {}
    for name, _ in _Summary._fields_:
        v = getattr(s, name)
        summary[name] = (v.kind, v.value) if isinstance(v, _Knob) else v
    rp = _Report()
    lib.ds_job_result_profile(res, ctypes.byref(rp))
    report = {name: getattr(rp, name) for name, _ in _Report._fields_}
    nt = lib.ds_job_result_tape(res, None, 0)
    tape = np.empty(nt, dtype=np.float64)
    lib.ds_job_result_tape(res, tape.ctypes.data, nt)
    nl = lib.ds_job_result_latencies(res, None, 0)
    lat = np.empty(nl, dtype=np.float64)
    lib.ds_job_result_latencies(res, lat.ctypes.data, nl)
    nr = lib.ds_job_result_readaptations(res, None, None, 0)
    at = np.empty(max(1, nr), dtype=np.float64)
    pe = np.empty(max(1, nr), dtype=np.int32)
    lib.ds_job_result_readaptations(res, at.ctypes.data, pe.ctypes.data, nr)
    err = lib.ds_job_result_error(res).decode()
    ne = lib.ds_job_result_energy_tape(res, None, 0)
    etape = np.empty(ne, dtype=np.float64)
    lib.ds_job_result_energy_tape(res, etape.ctypes.data, ne)
    return JobResult(records, summary, report, tape, lat,
                     [(float(at[i]), int(pe[i])) for i in range(nr)], err, etape)


def run_job(scenario: Scenario, job: JobSpec, catalog: Sequence[DnnProfile], seam: str = "analytic",
            backend: Optional[GpuBackend] = None, device: int = 0, host_io: bool = False,
            tape: Optional[np.ndarray] = None,
            energy_tape: Optional[np.ndarray] = None) -> JobResult:
    """run_job (reference harness.cpp:329-333) on the chosen seam:
    'analytic' (the reference's simulated GPU), 'device' (B200), 'replay' (tape)."""
    lib = _l()
    m = _Marshal(scenario, job, catalog)
    spec = m.seam(seam, backend, device, host_io, tape, energy_tape)
    res = ctypes.c_void_p()
    _lib.check(lib.ds_job_run(ctypes.byref(m.sc), ctypes.byref(m.job), m.catalog, m.n_catalog,
                              ctypes.byref(spec), ctypes.byref(res)))
    try:
        return _collect(lib, res)
    finally:
        lib.ds_job_result_free(res)


def profile_dnn(catalog: Sequence[DnnProfile], dnn_id: str, m: int = 32, n: int = 8,
                batches: int = 10, seed: int = 42, sigma: float = -1.0, seam: str = "analytic",
                backend: Optional[GpuBackend] = None, device: int = 0) -> dict:
    """The Profiler alone on one catalog network (reference
    tools/dnnscaler_main.cpp:88-99): the ProfileReport fields as a dict."""
    lib = _l()
    mar = _Marshal(Scenario(), JobSpec(0, dnn_id, 1.0, 1.0), catalog)
    spec = mar.seam(seam, backend, device)
    rp = _Report()
    _lib.check(lib.ds_profile_dnn(mar.catalog, mar.n_catalog, dnn_id.encode(), m, n, batches, seed,
                                  sigma, ctypes.byref(spec), ctypes.byref(rp)))
    return {name: getattr(rp, name) for name, _ in _Report._fields_}


def combination_sweep(catalog: Sequence[DnnProfile], dnn_id: str, bs_list, mtl_list,
                      samples: int = 100, seed: int = 42, sigma: float = -1.0) -> list:
    """The B x MT grid on a catalog network's analytic model (reference
    harness.cpp:356-386 via the CLI's cmd_sweep): cells as dicts, bs-major."""
    lib = _l()
    mar = _Marshal(Scenario(), JobSpec(0, dnn_id, 1.0, 1.0), catalog)
    bs = np.ascontiguousarray(bs_list, dtype=np.int32)
    mt = np.ascontiguousarray(mtl_list, dtype=np.int32)
    out = np.zeros((max(1, bs.size * mt.size), 5), dtype=np.float64)
    _lib.check(lib.ds_combination_sweep(mar.catalog, mar.n_catalog, dnn_id.encode(), bs.ctypes.data,
                                        bs.size, mt.ctypes.data, mt.size, samples, seed, sigma,
                                        out.ctypes.data))
    return [{"bs": int(r[0]), "mtl": int(r[1]), "mean_ms": float(r[2]), "p95_ms": float(r[3]),
             "throughput": float(r[4])} for r in out[:bs.size * mt.size]]


class JobSession:
    """Incremental job: start() on construction, step() per control period."""

    def __init__(self, scenario: Scenario, job: JobSpec, catalog: Sequence[DnnProfile],
                 seam: str = "device", backend: Optional[GpuBackend] = None,
                 tape: Optional[np.ndarray] = None):
        self._lib = _l()
        self._m = _Marshal(scenario, job, catalog)
        spec = self._m.seam(seam, backend, 0, False, tape)
        self._h = ctypes.c_void_p()
        _lib.check(self._lib.ds_job_start(ctypes.byref(self._m.sc), ctypes.byref(self._m.job),
                                          self._m.catalog, self._m.n_catalog, ctypes.byref(spec),
                                          ctypes.byref(self._h)))

    def step(self):
        r = _Record()
        done = ctypes.c_int()
        _lib.check(self._lib.ds_job_step(self._h, ctypes.byref(r), ctypes.byref(done)))
        rec = dict(time_s=r.time_s, knob=(r.knob.kind, r.knob.value), p95_ms=r.p95_ms,
                   mean_ms=r.mean_ms, throughput=r.throughput, slo_ms=r.slo_ms,
                   violated=bool(r.violated))
        return rec, bool(done.value)

    def knob(self):
        k = _Knob()
        _lib.check(self._lib.ds_job_knob(self._h, ctypes.byref(k)))
        return (k.kind, k.value)

    def finish(self) -> JobResult:
        res = ctypes.c_void_p()
        _lib.check(self._lib.ds_job_finish(self._h, ctypes.byref(res)))
        try:
            return _collect(self._lib, res)
        finally:
            self._lib.ds_job_result_free(res)

    def close(self):
        if self._h:
            self._lib.ds_job_session_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- single steps

def percentile(samples, q: float) -> float:
    a = np.ascontiguousarray(samples, dtype=np.float64)
    out = ctypes.c_double()
    _lib.check(_l().ds_percentile(a.ctypes.data, a.size, q, ctypes.byref(out)))
    return out.value


def band_verdict(p95: float, slo: float, alpha: float = 0.85) -> int:
    v = ctypes.c_int()
    _lib.check(_l().ds_band_verdict(p95, slo, alpha, ctypes.byref(v)))
    return v.value


class BatchScaler:
    """make_batch_scaler / batch_step (reference scaler.cpp:17-63)."""

    def __init__(self, abs_max_bs: int = 128):
        if abs_max_bs < 1:
            raise ValueError("invalid batch size limit")
        self.s = _BatchScaler(1, abs_max_bs, 1, abs_max_bs, 0)

    def step(self, p95: float, slo: float, alpha: float = 0.85) -> bool:
        ch = ctypes.c_int()
        _lib.check(_l().ds_batch_step(ctypes.byref(self.s), p95, slo, alpha, ctypes.byref(ch)))
        return bool(ch.value)


class MtScaler:
    """make_mt_scaler / mt_step (reference scaler.cpp:65-109)."""

    def __init__(self, initial: int, max_mtl: int = 10):
        if max_mtl < 1:
            raise ValueError("invalid instance limit")
        if initial < 1 or initial > max_mtl:
            raise ValueError("initial instance count out of range")
        self.s = _MtScaler(initial, max_mtl, 0, 0)

    def step(self, p95: float, slo: float, alpha: float = 0.85):
        a, inf = ctypes.c_int(), ctypes.c_int()
        _lib.check(_l().ds_mt_step(ctypes.byref(self.s), p95, slo, alpha, ctypes.byref(a),
                                   ctypes.byref(inf)))
        return a.value, bool(inf.value)


def mt_init(lat1: float, latn: float, n_probe: int, rows, slo: float, max_mtl: int,
            seed: int = 0) -> int:
    r = np.ascontiguousarray(rows, dtype=np.float64).reshape(len(rows), -1) if len(rows) else \
        np.zeros((0, 1))
    out = ctypes.c_int()
    _lib.check(_l().ds_mt_init(lat1, latn, n_probe, r.ctypes.data, r.shape[0], r.shape[1], slo,
                               max_mtl, seed, ctypes.byref(out)))
    return out.value


def estimate_row(rows, observed: dict, width: int, seed: int = 0) -> np.ndarray:
    r = np.ascontiguousarray(rows, dtype=np.float64)
    lv = np.array(sorted(observed), dtype=np.int32)
    vals = np.array([observed[k] for k in sorted(observed)], dtype=np.float64)
    out = np.empty(width, dtype=np.float64)
    _lib.check(_l().ds_estimate_row(r.ctypes.data, r.shape[0], r.shape[1], lv.ctypes.data,
                                    vals.ctypes.data, lv.size, width, seed, out.ctypes.data))
    return out


def decide(ti_batching, ti_mt, lat_b=0.0, lat_mt=0.0, eps=0.5) -> int:
    r = _Report()
    r.ti_batching, r.ti_mt = ti_batching, ti_mt
    r.probe_latency_batching_ms, r.probe_latency_mt_ms = lat_b, lat_mt
    out = ctypes.c_int()
    _lib.check(_l().ds_decide(ctypes.byref(r), eps, ctypes.byref(out)))
    return out.value


def calibrate_batching(points):
    x = np.array([p[0] for p in points], dtype=np.int32)
    t = np.array([p[1] for p in points], dtype=np.float64)
    a, b = ctypes.c_double(), ctypes.c_double()
    _lib.check(_l().ds_calibrate_batching(x.ctypes.data, t.ctypes.data, x.size, ctypes.byref(a),
                                          ctypes.byref(b)))
    return a.value, b.value


def calibrate_mt(points):
    x = np.array([p[0] for p in points], dtype=np.int32)
    t = np.array([p[1] for p in points], dtype=np.float64)
    l1, cap = ctypes.c_double(), ctypes.c_double()
    _lib.check(_l().ds_calibrate_mt(x.ctypes.data, t.ctypes.data, x.size, ctypes.byref(l1),
                                    ctypes.byref(cap)))
    return l1.value, cap.value
