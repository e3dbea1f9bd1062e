"""TEST INFRASTRUCTURE ONLY — Python loader for the plain-C oracle (oracle.c)
and for the reference library built from /root/reference (oracle/_ref/).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module, and only as the checker. The product path
(paper_1803_03288_b200/) never imports it.

`OracleGraph.from_json` restates the reference's index model
(graph.cpp:54-96): ops sorted by id in byte order, edges sorted and deduped,
adjacency lists ascending, resources sorted by (device, unit, name) with
Compute < Channel (graph.hpp:36-40).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcommsched_ref.so")
REF_SWEEP = os.path.join(HERE, "_ref", "ref_sweep")

KINDS = {"compute": 0, "recv": 1, "send": 2, "ps_aggregate": 3, "ps_read": 4,
         "ps_update": 5}
INF = (1 << 63) - 1


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_LIB) and os.path.exists(REF_SWEEP)


class _OrcGraph(C.Structure):
    _fields_ = [("n", C.c_int32),
                ("pred_off", C.POINTER(C.c_int32)), ("pred_idx", C.POINTER(C.c_int32)),
                ("succ_off", C.POINTER(C.c_int32)), ("succ_idx", C.POINTER(C.c_int32)),
                ("kind", C.POINTER(C.c_int8)), ("res", C.POINTER(C.c_int32)),
                ("n_res", C.c_int32), ("res_channel", C.POINTER(C.c_int8)),
                ("dur", C.POINTER(C.c_int64))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_mt_next.restype = C.c_uint64
        L.orc_bounded.restype = C.c_uint64
        L.orc_bounded.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_unit.restype = C.c_double
        L.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_mt_next.argtypes = [C.c_void_p]
        L.orc_unit.argtypes = [C.c_void_p]
        L.orc_random_order.argtypes = [C.c_int32, C.c_uint64, P(C.c_int32)]
        L.orc_dep_words.argtypes = [P(_OrcGraph)]
        L.orc_dep_words.restype = C.c_int32
        L.orc_dependencies.argtypes = [P(_OrcGraph), P(C.c_uint64)]
        L.orc_properties.argtypes = [P(_OrcGraph), P(C.c_uint8), C.c_int,
                                     P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        L.orc_precedes.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int32, C.c_int64, C.c_int64, C.c_int64]
        L.orc_tic.argtypes = [P(_OrcGraph), C.c_int, P(C.c_int32)]
        L.orc_tac.argtypes = [P(_OrcGraph), P(C.c_int32)]
        L.orc_tac_incremental.argtypes = [P(_OrcGraph), P(C.c_int32)]
        L.orc_tac_rows.argtypes = [P(_OrcGraph), P(C.c_int32)]
        L.orc_simulate.argtypes = [P(_OrcGraph), P(C.c_int32), C.c_int, C.c_uint64,
                                   C.c_double, P(C.c_int64), P(C.c_int64),
                                   P(C.c_int64), P(C.c_int64)]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class MT:
    """std::mt19937_64 (rng.hpp:14-33) through the C oracle."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(312 * 8 + 8)
        lib().orc_mt_seed(self._buf, seed)

    def next(self) -> int:
        return lib().orc_mt_next(self._buf)

    def bounded(self, n: int) -> int:
        return lib().orc_bounded(self._buf, n)

    def unit(self) -> float:
        return lib().orc_unit(self._buf)


def splitmix64(x: int) -> int:
    return lib().orc_splitmix64(x)


def random_order(n_recv: int, seed: int) -> np.ndarray:
    perm = np.zeros(max(n_recv, 1), dtype=np.int32)
    lib().orc_random_order(n_recv, seed, _ptr(perm, C.c_int32))
    return perm[:n_recv]


def _res_key(r):
    return (r["device"].encode(), 0 if r["unit"] == "compute" else 1, r["name"].encode())


class OracleGraph:
    """Index-model view of a reference-format graph document."""

    def __init__(self, doc: dict, durations: dict | None = None):
        ops = sorted(doc["ops"], key=lambda o: o["id"].encode())
        self.doc = doc
        self.ids = [o["id"] for o in ops]
        self.index = {s: i for i, s in enumerate(self.ids)}
        n = len(ops)
        edges = sorted({(a, b) for a, b in doc.get("edges", [])},
                       key=lambda e: (e[0].encode(), e[1].encode()))
        preds = [[] for _ in range(n)]
        succs = [[] for _ in range(n)]
        for a, b in edges:
            succs[self.index[a]].append(self.index[b])
            preds[self.index[b]].append(self.index[a])
        for l in preds + succs:
            l.sort()
        self.preds, self.succs = preds, succs
        self.kind = np.array([KINDS[o["kind"]] for o in ops], dtype=np.int8)
        keys = sorted({_res_key(o["resource"]) for o in ops})
        self.resources = keys
        rindex = {k: i for i, k in enumerate(keys)}
        self.res = np.array([rindex[_res_key(o["resource"])] for o in ops], dtype=np.int32)
        self.res_channel = np.array([k[1] for k in keys], dtype=np.int8)
        self.devices = [o["resource"]["device"] for o in ops]
        if durations is None:
            durations = {o["id"]: o.get("time_us", 0) for o in ops}
        self.dur = np.array([durations[s] for s in self.ids], dtype=np.int64)
        self.recv_cols = [i for i in range(n) if self.kind[i] == 1]
        self.recv_ids = [self.ids[i] for i in self.recv_cols]
        self._arrays(preds, succs)

    @classmethod
    def from_json(cls, text: str, durations: dict | None = None):
        return cls(json.loads(text), durations)

    def _arrays(self, preds, succs):
        def csr(lists):
            off = np.zeros(len(lists) + 1, dtype=np.int32)
            off[1:] = np.cumsum([len(l) for l in lists])
            idx = np.array([x for l in lists for x in l] or [0], dtype=np.int32)
            return off, idx
        self.pred_off, self.pred_idx = csr(preds)
        self.succ_off, self.succ_idx = csr(succs)
        self._s = _OrcGraph(len(self.ids), _ptr(self.pred_off, C.c_int32),
                            _ptr(self.pred_idx, C.c_int32), _ptr(self.succ_off, C.c_int32),
                            _ptr(self.succ_idx, C.c_int32), _ptr(self.kind, C.c_int8),
                            _ptr(self.res, C.c_int32), len(self.resources),
                            _ptr(self.res_channel, C.c_int8), _ptr(self.dur, C.c_int64))

    def with_durations(self, dur: np.ndarray) -> "OracleGraph":
        g = OracleGraph.__new__(OracleGraph)
        g.__dict__.update(self.__dict__)
        g.dur = np.ascontiguousarray(dur, dtype=np.int64)
        g._arrays(self.preds, self.succs)
        return g

    # ---- restated reference functions -------------------------------------
    def dependencies(self) -> dict:
        w = lib().orc_dep_words(C.byref(self._s))
        bits = np.zeros(max(1, w * len(self.ids)), dtype=np.uint64)
        lib().orc_dependencies(C.byref(self._s), _ptr(bits, C.c_uint64))
        out = {}
        for v, s in enumerate(self.ids):
            row = bits[v * w:(v + 1) * w]
            out[s] = [self.recv_ids[c] for c in range(len(self.recv_ids))
                      if (int(row[c >> 6]) >> (c & 63)) & 1]
        return out

    def properties(self, outstanding=None, mode: str = "amended"):
        nr = len(self.recv_cols)
        out = np.ones(max(nr, 1), dtype=np.uint8)
        if outstanding is not None:
            out[:] = 0
            for s in outstanding:
                out[self.recv_ids.index(s)] = 1
        M = np.zeros(max(1, len(self.ids)), dtype=np.int64)
        P = np.zeros(max(1, nr), dtype=np.int64)
        Mp = np.zeros(max(1, nr), dtype=np.int64)
        lib().orc_properties(C.byref(self._s), _ptr(out, C.c_uint8),
                             1 if mode == "amended" else 0, _ptr(M, C.c_int64),
                             _ptr(P, C.c_int64), _ptr(Mp, C.c_int64))
        keep = [c for c in range(nr) if out[c]]
        return ({s: int(M[i]) for i, s in enumerate(self.ids)},
                {self.recv_ids[c]: int(P[c]) for c in keep},
                {self.recv_ids[c]: (None if Mp[c] == INF else int(Mp[c])) for c in keep})

    def tic(self, mode: str = "amended"):
        prio = np.zeros(max(1, len(self.recv_cols)), dtype=np.int32)
        total = lib().orc_tic(C.byref(self._s), 1 if mode == "amended" else 0,
                              _ptr(prio, C.c_int32))
        return {s: int(prio[c]) for c, s in enumerate(self.recv_ids)}, bool(total)

    def tac(self, incremental: bool = False, rows: bool = False):
        prio = np.zeros(max(1, len(self.recv_cols)), dtype=np.int32)
        f = (lib().orc_tac_rows if rows else
             lib().orc_tac_incremental if incremental else lib().orc_tac)
        f(C.byref(self._s), _ptr(prio, C.c_int32))
        return {s: int(prio[c]) for c, s in enumerate(self.recv_ids)}

    def random_schedule(self, seed: int):
        perm = random_order(len(self.recv_cols), seed)
        return {self.recv_ids[c]: k for k, c in enumerate(perm)}

    def simulate(self, priorities: dict | None, gated=True, choice_seed=0, noise=0.0,
                 events=False):
        n = len(self.ids)
        prio = np.full(max(n, 1), -1, dtype=np.int32)
        for s, r in (priorities or {}).items():
            prio[self.index[s]] = r
        m = C.c_int64()
        v = C.c_int64()
        st = np.zeros(max(n, 1), dtype=np.int64)
        en = np.zeros(max(n, 1), dtype=np.int64)
        rc = lib().orc_simulate(C.byref(self._s), _ptr(prio, C.c_int32), int(bool(gated)),
                                choice_seed, noise, C.byref(m), C.byref(v),
                                _ptr(st, C.c_int64), _ptr(en, C.c_int64))
        if rc:
            raise RuntimeError("simulation stalled with no runnable op")
        if events:
            return m.value, v.value, st[:n].copy(), en[:n].copy()
        return m.value, v.value

    def bounds(self):
        U = int(self.dur.sum())
        per = {}
        for i in range(len(self.ids)):
            per[self.res[i]] = per.get(self.res[i], 0) + int(self.dur[i])
        return U, (max(per.values()) if per else 0)

    def worker_devices(self):
        return sorted({self.devices[i] for i in range(len(self.ids)) if self.kind[i] in (0, 1, 2)},
                      key=lambda d: d.encode())

    def partition(self, device: str) -> "OracleGraph":
        """worker_partition (sim.cpp:43-59)."""
        keep = {s for s, d in zip(self.ids, self.devices) if d == device}
        doc = {"name": self.doc["name"] + "/" + device, "partition": "worker",
               "ops": [o for o in self.doc["ops"] if o["id"] in keep],
               "edges": [e for e in self.doc.get("edges", []) if e[0] in keep and e[1] in keep]}
        return OracleGraph(doc, {s: int(self.dur[self.index[s]]) for s in keep})

    def iteration_stats(self, end: np.ndarray):
        """iteration_stats (sim.cpp:258-279): per-worker makespans + straggler."""
        pw = {d: 0 for d in self.worker_devices()}
        for i in range(len(self.ids)):
            d = self.devices[i]
            if d in pw:
                pw[d] = max(pw[d], int(end[i]))
        hi, lo = max(pw.values()), min(pw.values())
        return pw, (hi - lo, hi)


def schedule_for(g: OracleGraph, algo: str, seed: int = 0, mode: str = "amended"):
    """cluster.cpp:91-122 — per-worker partitions with derived seeds."""
    def one(part, s):
        if algo == "tic":
            return part.tic(mode)[0]
        if algo == "tac":
            return part.tac()
        return part.random_schedule(s)
    if g.doc["partition"] == "worker":
        return one(g, seed)
    merged = {}
    for i, d in enumerate(g.worker_devices()):
        derived = splitmix64((seed ^ ((0x9e3779b97f4a7c15 * (i + 1)) & (2**64 - 1))) & (2**64 - 1))
        merged.update(one(g.partition(d), derived))
    return merged


# ---- the reference library itself (oracle/_ref), for pinning ---------------

class RefLib:
    """ctypes view of the reference libcommsched built from /root/reference."""

    def __init__(self):
        L = C.CDLL(REF_LIB)
        vp, cp = C.c_void_p, C.c_char_p
        for name in ["cs_graph_parse", "cs_graph_serialize", "cs_oracle_declared",
                     "cs_oracle_general", "cs_oracle_bandwidth", "cs_schedule_tic",
                     "cs_schedule_tac", "cs_schedule_random", "cs_schedule_serialize",
                     "cs_simulate", "cs_report_makespan", "cs_report_violations",
                     "cs_report_json", "cs_properties_json", "cs_makespan_bounds",
                     "cs_metrics_json", "cs_report_iteration_json", "cs_brute_force",
                     "cs_graph_generate", "cs_graph_expand", "cs_oracle_json",
                     "cs_schedule_parse", "cs_report_chrome_trace"]:
            getattr(L, name).restype = C.c_int
        L.cs_last_error.restype = cp
        L.cs_string_free.argtypes = [vp]
        L.cs_schedule_random.argtypes = [vp, C.c_uint64, C.POINTER(vp)]
        L.cs_oracle_bandwidth.argtypes = [vp, C.c_int64, C.POINTER(vp)]
        L.cs_graph_generate.argtypes = [cp, C.c_int, C.c_int, cp, C.c_uint64, C.POINTER(vp)]
        L.cs_graph_expand.argtypes = [vp, C.c_int, C.c_int, C.c_int64, C.POINTER(vp)]
        self.L = L
