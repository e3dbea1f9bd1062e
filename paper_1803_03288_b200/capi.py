"""ctypes binding of the commsched C ABI (include/commsched.h).

The same binding drives any library that exports the reference interface:
this package's B200 build (`paper_1803_03288_b200/libcommsched.so`, the
default) or the reference's own libcommsched built from /root/reference
(tests pass its path to `Lib`). That is the drop-in claim made concrete: the
caller code is identical for both.

Handles own their C objects and free them on garbage collection. Errors
raise `CsError` carrying the status code and `cs_last_error()` text, the
same pair the reference returns (reference capi.cpp:37-52).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
PRODUCT_LIB = os.path.join(PKG_DIR, "libcommsched.so")


def _torch_nccl() -> str | None:
    """torch's bundled NCCL (nvidia-nccl wheel), found without importing
    torch: the library's multi-GPU path loads it (TICTAC_NCCL_LIB) instead of
    an older system copy that a later `import torch` would then be bound to
    through the shared soname."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


if not os.environ.get("TICTAC_NCCL_LIB"):
    _p = _torch_nccl()
    if _p:
        os.environ["TICTAC_NCCL_LIB"] = _p

CS_OK, CS_ERR_INTERNAL, CS_ERR_VALIDATION, CS_ERR_COVERAGE, CS_ERR_PARAMETER, CS_ERR_IO = range(6)
HIST_BINS = 1000
DSTATS_I64 = 2008
DSTATS_F64 = 2


class CsError(RuntimeError):
    def __init__(self, code: int, message: str, call: str = ""):
        super().__init__(f"{call}: [{code}] {message}" if call else f"[{code}] {message}")
        self.code = code
        self.message = message


class SimPolicy(C.Structure):
    _fields_ = [("counter_gate", C.c_int), ("choice_seed", C.c_uint64), ("reorder_noise", C.c_double)]


class SweepStats(C.Structure):
    _fields_ = [("count", C.c_int64), ("upper_us", C.c_int64), ("lower_us", C.c_int64),
                ("min_us", C.c_int64), ("argmin_seed", C.c_uint64), ("max_us", C.c_int64),
                ("argmax_seed", C.c_uint64), ("sum_us", C.c_int64), ("sumsq_us", C.c_double),
                ("e_hist", C.c_int64 * HIST_BINS), ("n_workers", C.c_int64),
                ("straggler_sum", C.c_double), ("straggler_hist", C.c_int64 * HIST_BINS),
                ("iter_min_us", C.c_int64), ("iter_argmin_seed", C.c_uint64), ("iter_max_us", C.c_int64),
                ("iter_argmax_seed", C.c_uint64), ("iter_sum_us", C.c_int64)]

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("e_hist", "straggler_hist")}
        d["e_hist"] = np.ctypeslib.as_array(self.e_hist).copy()
        d["straggler_hist"] = np.ctypeslib.as_array(self.straggler_hist).copy()
        return d


def policy(counter_gate: bool = True, choice_seed: int = 0, reorder_noise: float = 0.0) -> SimPolicy:
    return SimPolicy(1 if counter_gate else 0, choice_seed, reorder_noise)


_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_cp = C.c_char_p
_i64p = C.POINTER(C.c_int64)

# name -> argtypes (all return int unless listed in _VOID/_SPECIAL)
_SIGS = {
    "cs_graph_parse": [_cp, _pp], "cs_graph_serialize": [_vp, _pp],
    "cs_graph_generate": [_cp, C.c_int, C.c_int, _cp, C.c_uint64, _pp],
    "cs_graph_expand": [_vp, C.c_int, C.c_int, C.c_int64, _pp],
    "cs_graph_name": [_vp, _pp], "cs_graph_op_count": [_vp, _i64p],
    "cs_graph_edge_count": [_vp, _i64p], "cs_graph_recv_count": [_vp, _i64p],
    "cs_graph_is_cluster": [_vp, C.POINTER(C.c_int)], "cs_graph_topo_order": [_vp, _pp],
    "cs_graph_worker_devices": [_vp, _pp], "cs_graph_worker_partition": [_vp, _cp, _pp],
    "cs_oracle_declared": [_vp, _pp], "cs_oracle_general": [_vp, _pp],
    "cs_oracle_from_traces": [_vp, _cp, _pp], "cs_oracle_bandwidth": [_vp, C.c_int64, _pp],
    "cs_oracle_json": [_vp, _pp], "cs_properties_json": [_vp, _vp, _cp, _pp],
    "cs_schedule_tic": [_vp, _cp, _pp], "cs_schedule_tac": [_vp, _vp, _pp],
    "cs_schedule_random": [_vp, C.c_uint64, _pp], "cs_schedule_parse": [_cp, _pp],
    "cs_schedule_serialize": [_vp, _pp], "cs_schedule_total_order": [_vp, C.POINTER(C.c_int)],
    "cs_simulate": [_vp, _vp, _vp, C.POINTER(SimPolicy), _pp],
    "cs_report_makespan": [_vp, _i64p], "cs_report_violations": [_vp, _i64p],
    "cs_report_json": [_vp, _pp], "cs_report_chrome_trace": [_vp, _pp],
    "cs_report_iteration_json": [_vp, _pp],
    "cs_makespan_bounds": [_vp, _vp, _i64p, _i64p], "cs_metrics_json": [_vp, _vp, _vp, _pp],
    "cs_brute_force": [_vp, _vp, C.POINTER(SimPolicy), C.c_int, _pp],
    # extensions (product library only)
    "cs_sweep_random": [_vp, _vp, C.c_uint64, C.c_int64, C.POINTER(SimPolicy), _vp, _vp,
                        C.POINTER(SweepStats)],
    "cs_simulate_orders": [_vp, _vp, _vp, C.c_int64, C.POINTER(SimPolicy), _vp, _vp],
    "cs_sweep_random_multi": [_vp, _vp, C.c_uint64, C.c_int64, C.POINTER(SimPolicy), C.c_int, _vp, _vp,
                              C.POINTER(SweepStats)],
    "cs_sweep_plan_create": [_vp, _vp, C.POINTER(SimPolicy), _pp],
    "cs_sweep_plan_info": [_vp, _pp],
    "cs_sweep_path_json": [_vp, _vp, C.POINTER(SimPolicy), _pp],
    "cs_sweep_plan_reset": [_vp, _vp, _vp, _vp],
    "cs_sweep_plan_run": [_vp, C.c_uint64, C.c_int64, C.c_uint64, _vp, _vp, _vp, _vp],
    "cs_sweep_stats_finish": [_vp, _vp, _vp, C.c_uint64, C.POINTER(SweepStats)],
    "cs_sweep_stats_pack": [_vp, _vp, C.c_int, C.c_int, _vp, _vp],
    "cs_sweep_stats_unpack": [_vp, C.c_int, _vp, _vp, _vp],
    "cs_graph_generate_model": [_cp, C.c_uint64, _pp],
    "cs_tac_traffic": [_vp, _vp, _i64p, C.c_int],
}
_FREE = ["cs_graph_free", "cs_oracle_free", "cs_schedule_free", "cs_report_free",
         "cs_string_free", "cs_sweep_plan_free"]
REFERENCE_SYMBOLS = [k for k in _SIGS if k not in (
    "cs_sweep_random", "cs_sweep_random_multi", "cs_simulate_orders", "cs_sweep_plan_create", "cs_sweep_plan_info",
    "cs_sweep_path_json",
    "cs_sweep_plan_reset", "cs_sweep_plan_run", "cs_sweep_stats_finish", "cs_sweep_stats_pack",
    "cs_sweep_stats_unpack",
    "cs_graph_generate_model", "cs_tac_traffic")] + [f for f in _FREE if f != "cs_sweep_plan_free"] + [
    "cs_last_error", "cs_version"]


class Lib:
    """One loaded libcommsched-compatible shared library."""

    def __init__(self, path: str = PRODUCT_LIB):
        if not os.path.exists(path):
            raise ImportError(f"libcommsched not built: {path} (run __graft_entry__.build())")
        self.path = path
        self.L = C.CDLL(path)
        self.extended = hasattr(self.L, "cs_sweep_random")
        for name, args in _SIGS.items():
            if not hasattr(self.L, name):
                continue
            f = getattr(self.L, name)
            f.argtypes = args
            f.restype = C.c_int
        for name in _FREE:
            if hasattr(self.L, name):
                getattr(self.L, name).argtypes = [_vp]
                getattr(self.L, name).restype = None
        self.L.cs_last_error.restype = _cp
        self.L.cs_version.restype = _cp
        if hasattr(self.L, "cs_device_launches"):
            self.L.cs_device_launches.restype = C.c_int64

    def call(self, name: str, *args):
        rc = getattr(self.L, name)(*args)
        if rc != CS_OK:
            raise CsError(rc, self.L.cs_last_error().decode(), name)

    def take_str(self, p: C.c_void_p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.L.cs_string_free(p)
        return s

    def version(self) -> str:
        return self.L.cs_version().decode()

    def launches(self) -> int:
        return int(self.L.cs_device_launches()) if hasattr(self.L, "cs_device_launches") else 0

    # ---- handle constructors --------------------------------------------
    def graph(self, text: str) -> "Graph":
        h = C.c_void_p()
        self.call("cs_graph_parse", text.encode(), C.byref(h))
        return Graph(self, h)

    def generate(self, shape: str, layers: int, params: int, ratio: str, seed: int) -> "Graph":
        h = C.c_void_p()
        self.call("cs_graph_generate", shape.encode(), layers, params, ratio.encode(), seed, C.byref(h))
        return Graph(self, h)

    def model(self, name: str, seed: int = 1) -> "Graph":
        h = C.c_void_p()
        self.call("cs_graph_generate_model", name.encode(), seed, C.byref(h))
        return Graph(self, h)

    def schedule_parse(self, text: str) -> "Schedule":
        h = C.c_void_p()
        self.call("cs_schedule_parse", text.encode(), C.byref(h))
        return Schedule(self, h)


class _Handle:
    _free = ""

    def __init__(self, lib: Lib, h: C.c_void_p):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            if self.h:
                getattr(self.lib.L, self._free)(self.h)
                self.h = None
        except Exception:
            pass

    def _str(self, name: str, *args) -> str:
        p = C.c_void_p()
        self.lib.call(name, self.h, *args, C.byref(p))
        return self.lib.take_str(p)


class Graph(_Handle):
    _free = "cs_graph_free"

    def serialize(self) -> str:
        return self._str("cs_graph_serialize")

    def name(self) -> str:
        return self._str("cs_graph_name")

    def _i64(self, name):
        v = C.c_int64()
        self.lib.call(name, self.h, C.byref(v))
        return v.value

    def op_count(self) -> int:
        return self._i64("cs_graph_op_count")

    def edge_count(self) -> int:
        return self._i64("cs_graph_edge_count")

    def recv_count(self) -> int:
        return self._i64("cs_graph_recv_count")

    def is_cluster(self) -> bool:
        v = C.c_int()
        self.lib.call("cs_graph_is_cluster", self.h, C.byref(v))
        return bool(v.value)

    def topo_order(self) -> list:
        return json.loads(self._str("cs_graph_topo_order"))

    def worker_devices(self) -> list:
        return json.loads(self._str("cs_graph_worker_devices"))

    def partition(self, device: str) -> "Graph":
        h = C.c_void_p()
        self.lib.call("cs_graph_worker_partition", self.h, device.encode(), C.byref(h))
        return Graph(self.lib, h)

    def expand(self, n_workers: int, n_ps: int, ps_op_time_us: int) -> "Graph":
        h = C.c_void_p()
        self.lib.call("cs_graph_expand", self.h, n_workers, n_ps, ps_op_time_us, C.byref(h))
        return Graph(self.lib, h)

    # oracles
    def _oracle(self, name, *args) -> "Oracle":
        h = C.c_void_p()
        self.lib.call(name, self.h, *args, C.byref(h))
        return Oracle(self.lib, h)

    def declared(self) -> "Oracle":
        return self._oracle("cs_oracle_declared")

    def general(self) -> "Oracle":
        return self._oracle("cs_oracle_general")

    def traces(self, jsonl: str) -> "Oracle":
        return self._oracle("cs_oracle_from_traces", jsonl.encode())

    def bandwidth(self, bytes_per_us: int) -> "Oracle":
        return self._oracle("cs_oracle_bandwidth", bytes_per_us)

    # schedules
    def _sched(self, name, *args) -> "Schedule":
        h = C.c_void_p()
        self.lib.call(name, self.h, *args, C.byref(h))
        return Schedule(self.lib, h)

    def tic(self, mode: str = "amended") -> "Schedule":
        return self._sched("cs_schedule_tic", mode.encode())

    def tac(self, oracle: "Oracle") -> "Schedule":
        return self._sched("cs_schedule_tac", oracle.h)

    def random(self, seed: int) -> "Schedule":
        return self._sched("cs_schedule_random", seed)

    def properties(self, oracle: "Oracle", mode: str = "amended") -> dict:
        return json.loads(self.properties_text(oracle, mode))

    def properties_text(self, oracle: "Oracle", mode: str = "amended") -> str:
        p = C.c_void_p()
        self.lib.call("cs_properties_json", self.h, oracle.h, mode.encode(), C.byref(p))
        return self.lib.take_str(p)

    def simulate(self, oracle: "Oracle", schedule: "Schedule | None" = None,
                 pol: SimPolicy | None = None) -> "Report":
        h = C.c_void_p()
        self.lib.call("cs_simulate", self.h, oracle.h, schedule.h if schedule else None,
                      C.byref(pol) if pol is not None else None, C.byref(h))
        return Report(self.lib, h)

    def bounds(self, oracle: "Oracle") -> tuple[int, int]:
        u, l = C.c_int64(), C.c_int64()
        self.lib.call("cs_makespan_bounds", self.h, oracle.h, C.byref(u), C.byref(l))
        return u.value, l.value

    def tac_traffic(self, oracle: "Oracle") -> dict:
        """SURVEY §8d TAC traffic terms from the device closure, plus B_TAC
        (algorithmic bytes of one whole TAC ordering) and B_TIC (one TIC)."""
        out = (C.c_int64 * 7)()
        self.lib.call("cs_tac_traffic", self.h, oracle.h, out, 7)
        V, R, E, E_recv, nnz, rows, row_nnz = (int(x) for x in out)
        words = (R + 31) // 32
        b_tac = 4 * V * words + 20 * V * R + 6 * E_recv * (R + 1) + 12 * R * (R + 1) + 32 * nnz
        b_tic = 4 * V * words + 20 * V + 12 * E_recv + 24 * R
        return {"V": V, "R": R, "E": E, "E_recv": E_recv, "nnz": nnz, "rows": rows,
                "row_nnz": row_nnz, "B_TAC": b_tac, "B_TIC": b_tic}

    def metrics_text(self, oracle: "Oracle", report: "Report") -> str:
        p = C.c_void_p()
        self.lib.call("cs_metrics_json", self.h, oracle.h, report.h, C.byref(p))
        return self.lib.take_str(p)

    def brute_force_text(self, oracle: "Oracle", pol: SimPolicy | None = None, max_recvs: int = 8) -> str:
        p = C.c_void_p()
        self.lib.call("cs_brute_force", self.h, oracle.h, C.byref(pol) if pol is not None else None,
                      max_recvs, C.byref(p))
        return self.lib.take_str(p)

    # batched extensions
    def sweep_random(self, oracle: "Oracle", seed_lo: int, count: int, pol: SimPolicy | None = None,
                     makespans: bool = False, worker_makespans: bool = False):
        ms = np.zeros(max(count, 1), dtype=np.int64) if makespans else None
        nw = len(self.worker_devices()) if (worker_makespans and self.is_cluster()) else 0
        wms = np.zeros(max(count * nw, 1), dtype=np.int64) if nw else None
        st = SweepStats()
        self.lib.call("cs_sweep_random", self.h, oracle.h, seed_lo, count,
                      C.byref(pol) if pol is not None else None,
                      ms.ctypes.data if ms is not None else None,
                      wms.ctypes.data if wms is not None else None, C.byref(st))
        out = st.to_dict()
        if ms is not None:
            out["makespans"] = ms[:count]
        if wms is not None:
            out["worker_makespans"] = wms[:count * nw].reshape(count, nw)
        return out

    def sweep_random_multi(self, oracle: "Oracle", seed_lo: int, count: int, n_devices: int,
                           pol: SimPolicy | None = None, makespans: bool = False, worker_makespans: bool = False):
        ms = np.zeros(max(count, 1), dtype=np.int64) if makespans else None
        nw = len(self.worker_devices()) if (worker_makespans and self.is_cluster()) else 0
        wms = np.zeros(max(count * nw, 1), dtype=np.int64) if nw else None
        st = SweepStats()
        self.lib.call("cs_sweep_random_multi", self.h, oracle.h, seed_lo, count,
                      C.byref(pol) if pol is not None else None, n_devices,
                      ms.ctypes.data if ms is not None else None,
                      wms.ctypes.data if wms is not None else None, C.byref(st))
        out = st.to_dict()
        if ms is not None:
            out["makespans"] = ms[:count]
        if wms is not None:
            out["worker_makespans"] = wms[:count * nw].reshape(count, nw)
        return out

    def sweep_path(self, oracle: "Oracle", pol: SimPolicy | None = None) -> dict:
        out = C.c_void_p()
        self.lib.call("cs_sweep_path_json", self.h, oracle.h, C.byref(pol) if pol is not None else None,
                      C.byref(out))
        return json.loads(self.lib.take_str(out))

    def simulate_orders(self, oracle: "Oracle", orders: np.ndarray, pol: SimPolicy | None = None):
        orders = np.ascontiguousarray(orders, dtype=np.int32)
        n = orders.shape[0]
        ms = np.zeros(max(n, 1), dtype=np.int64)
        vi = np.zeros(max(n, 1), dtype=np.int64)
        self.lib.call("cs_simulate_orders", self.h, oracle.h, orders.ctypes.data, n,
                      C.byref(pol) if pol is not None else None, ms.ctypes.data, vi.ctypes.data)
        return ms[:n], vi[:n]


class Oracle(_Handle):
    _free = "cs_oracle_free"

    def json(self) -> str:
        return self._str("cs_oracle_json")


class Schedule(_Handle):
    _free = "cs_schedule_free"

    def serialize(self) -> str:
        return self._str("cs_schedule_serialize")

    def priorities(self) -> dict:
        return json.loads(self.serialize())["priorities"]

    def total_order(self) -> bool:
        v = C.c_int()
        self.lib.call("cs_schedule_total_order", self.h, C.byref(v))
        return bool(v.value)


class Report(_Handle):
    _free = "cs_report_free"

    def makespan(self) -> int:
        v = C.c_int64()
        self.lib.call("cs_report_makespan", self.h, C.byref(v))
        return v.value

    def violations(self) -> int:
        v = C.c_int64()
        self.lib.call("cs_report_violations", self.h, C.byref(v))
        return v.value

    def json(self) -> str:
        return self._str("cs_report_json")

    def chrome_trace(self) -> str:
        return self._str("cs_report_chrome_trace")

    def iteration_json(self) -> str:
        return self._str("cs_report_iteration_json")


class SweepPlan(_Handle):
    """Device-resident closed-form sweep (cs_sweep_plan_*), for drivers that
    keep statistics on the GPU and reduce them with NCCL across ranks."""
    _free = "cs_sweep_plan_free"

    @classmethod
    def create(cls, g: Graph, o: Oracle, pol: SimPolicy | None = None) -> "SweepPlan":
        h = C.c_void_p()
        g.lib.call("cs_sweep_plan_create", g.h, o.h, C.byref(pol) if pol is not None else None,
                   C.byref(h))
        return cls(g.lib, h)

    def info(self) -> dict:
        return json.loads(self._str("cs_sweep_plan_info"))

    def reset(self, stream: int, d_i64: int, d_f64: int):
        self.lib.call("cs_sweep_plan_reset", self.h, stream, d_i64, d_f64)

    def run(self, seed_lo: int, count: int, key_base: int, stream: int, d_makespans: int | None,
            d_i64: int, d_f64: int):
        self.lib.call("cs_sweep_plan_run", self.h, seed_lo, count, key_base, stream, d_makespans,
                      d_i64, d_f64)

    def finish(self, h_i64: np.ndarray, h_f64: np.ndarray, key_base: int) -> dict:
        st = SweepStats()
        h_i64 = np.ascontiguousarray(h_i64, dtype=np.int64)
        h_f64 = np.ascontiguousarray(h_f64, dtype=np.float64)
        self.lib.call("cs_sweep_stats_finish", self.h, h_i64.ctypes.data, h_f64.ctypes.data,
                      key_base, C.byref(st))
        return st.to_dict()
