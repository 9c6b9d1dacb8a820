"""The UNMODIFIED reference control plane (oracle/_ref/libref_replay.so, built
by `make -C oracle ref` from /root/reference sources + the tape seam) —
TEST INFRASTRUCTURE ONLY: used by tests/ as the bit-exact oracle for the
Profiler decision and Scaler trajectory, and by bench.py's reference leg.
"""
from __future__ import annotations

import ctypes
import json
import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libref_replay.so")
RECORD_WIDTH = 10
SUMMARY_FIELDS = ["job_id", "approach_kind", "profiled", "ti_batching", "ti_mt",
                  "profiling_cost_ms", "steady_kind", "steady_value", "converged", "knob_changes",
                  "settle_period", "periods", "duration_s", "total_items", "avg_throughput",
                  "steady_throughput", "p95_overall_ms", "slo_compliance", "avg_power_w",
                  "power_efficiency", "final_slo_ms", "n_readaptations", "failed", "reserved"]
PROFILE_FIELDS = ["tput_base", "tput_batching", "tput_mt", "ti_batching", "ti_mt",
                  "base_latency_ms", "probe_latency_batching_ms", "probe_latency_mt_ms", "m", "n",
                  "batches_per_point", "base_elapsed_ms", "batching_elapsed_ms", "mt_elapsed_ms",
                  "transition_ms", "profiling_cost_ms", "items_served"]

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle ref` where "
                              "/root/reference exists")
        l = ctypes.CDLL(REF_LIB)
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        psz = ctypes.POINTER(ctypes.c_size_t)
        l.ref_run_job.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, vp, sz, vp, sz, psz,
                                  vp, vp, sz, psz, vp, sz, psz, psz, ctypes.c_char_p, sz]
        l.ref_profile_tape.argtypes = [vp, sz, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, vp,
                                       ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, sz]
        l.ref_render_scenario.argtypes = [ctypes.c_char_p, vp, sz, psz, vp, sz, psz,
                                          ctypes.c_char_p, sz]
        l.ref_render_profile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                         ctypes.c_double, vp, sz, psz, ctypes.c_char_p, sz]
        l.ref_render_sweep.argtypes = [ctypes.c_char_p, ctypes.c_char_p, vp, ctypes.c_int, vp,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                       vp, sz, psz, ctypes.c_char_p, sz]
        _lib = l
    return _lib


def write_scenario(scenario_dict: dict, catalog: list, directory: str) -> str:
    """Writes a reference-format scenario + catalog pair; returns the scenario path."""
    os.makedirs(directory, exist_ok=True)
    cpath = os.path.join(directory, "catalog.json")
    with open(cpath, "w") as f:
        json.dump(catalog, f)
    d = dict(scenario_dict)
    d["catalog_path"] = "catalog.json"
    spath = os.path.join(directory, "scenario.json")
    with open(spath, "w") as f:
        json.dump(d, f)
    return spath


def run_job(scenario_path: str, job_index: int = 0, mode: str = "stock", tape=None,
            max_periods: int = 1_000_000, max_tape: int = 50_000_000):
    """Reference run_job on the tape seam. mode: stock | record | replay."""
    l = lib()
    m = {"stock": 0, "record": 1, "replay": 2, "callback": 3}[mode]
    t = np.ascontiguousarray(tape if tape is not None else np.zeros(0), dtype=np.float64)
    n_rec, tape_n, n_ra, consumed = (ctypes.c_size_t() for _ in range(4))
    # first call sizes the outputs
    err = ctypes.create_string_buffer(512)
    recs = np.empty((max_periods, RECORD_WIDTH), dtype=np.float64) if max_periods <= 200_000 else None
    summ = np.empty(len(SUMMARY_FIELDS), dtype=np.float64)
    tape_out = np.empty(max_tape if m == 1 else 1, dtype=np.float64)
    ra = np.empty(128, dtype=np.float64)
    if recs is None:
        recs = np.empty((200_000, RECORD_WIDTH), dtype=np.float64)
    rc = l.ref_run_job(scenario_path.encode(), job_index, m, t.ctypes.data, t.size, recs.ctypes.data,
                       recs.shape[0], ctypes.byref(n_rec), summ.ctypes.data, tape_out.ctypes.data,
                       tape_out.size, ctypes.byref(tape_n), ra.ctypes.data, 64, ctypes.byref(n_ra),
                       ctypes.byref(consumed), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    out_tape = tape_out[:tape_n.value].copy() if m == 1 else None
    return {
        "records": recs[:n_rec.value].copy(),
        "summary": dict(zip(SUMMARY_FIELDS, summ.tolist())),
        "tape": out_tape,
        "consumed": consumed.value,
        "readaptations": [(ra[2 * i], int(ra[2 * i + 1])) for i in range(n_ra.value)],
    }


def profile_tape(tape, m=32, n=8, bpp=10, abs_max_bs=128, max_mtl=10):
    l = lib()
    t = np.ascontiguousarray(tape, dtype=np.float64)
    out = np.empty(17, dtype=np.float64)
    appr = ctypes.c_int()
    err = ctypes.create_string_buffer(512)
    rc = l.ref_profile_tape(t.ctypes.data, t.size, m, n, bpp, abs_max_bs, max_mtl, out.ctypes.data,
                            ctypes.byref(appr), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return dict(zip(PROFILE_FIELDS, out.tolist())), appr.value


def render_scenario(scenario_path: str):
    l = lib()
    a, b = ctypes.c_size_t(), ctypes.c_size_t()
    err = ctypes.create_string_buffer(512)
    rc = l.ref_render_scenario(scenario_path.encode(), None, 0, ctypes.byref(a), None, 0,
                               ctypes.byref(b), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    csv = ctypes.create_string_buffer(a.value + 1)
    js = ctypes.create_string_buffer(b.value + 1)
    l.ref_render_scenario(scenario_path.encode(), csv, a.value, ctypes.byref(a), js, b.value,
                          ctypes.byref(b), err, 512)
    return csv.raw[:a.value].decode(), js.raw[:b.value].decode()


def render_profile(catalog_path: str, dnn_id: str, m=32, n=8, batches=10, seed=42, sigma=-1.0):
    """The reference CLI's `profile` JSON (dnnscaler_main.cpp:88-111) on the
    stock simulator."""
    l = lib()
    a = ctypes.c_size_t()
    err = ctypes.create_string_buffer(512)
    args = (catalog_path.encode(), dnn_id.encode(), m, n, batches, seed, sigma)
    if l.ref_render_profile(*args, None, 0, ctypes.byref(a), err, 512) != 0:
        raise RuntimeError(err.value.decode())
    js = ctypes.create_string_buffer(a.value + 1)
    l.ref_render_profile(*args, js, a.value, ctypes.byref(a), err, 512)
    return js.raw[:a.value].decode()


def render_sweep(catalog_path: str, dnn_id: str, bs, mtl, samples=100, seed=42, sigma=-1.0):
    """The reference CLI's `sweep` sweep.csv (dnnscaler_main.cpp:186-199)."""
    l = lib()
    b = (ctypes.c_int * len(bs))(*bs)
    m = (ctypes.c_int * len(mtl))(*mtl)
    a = ctypes.c_size_t()
    err = ctypes.create_string_buffer(512)
    args = (catalog_path.encode(), dnn_id.encode(), b, len(bs), m, len(mtl), samples, seed, sigma)
    if l.ref_render_sweep(*args, None, 0, ctypes.byref(a), err, 512) != 0:
        raise RuntimeError(err.value.decode())
    buf = ctypes.create_string_buffer(a.value + 1)
    l.ref_render_sweep(*args, buf, a.value, ctypes.byref(a), err, 512)
    return buf.raw[:a.value].decode()


def tempdir():
    return tempfile.mkdtemp(prefix="refscen_")
