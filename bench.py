#!/usr/bin/env python
"""Benchmark: recv-order makespan sims/sec (BASELINE.json metric) on B200.

Workload (one "step"): SURVEY §8d config 4 — the ResNet-v2-101-shaped
training DAG (5,380 ops / 7,090 edges / 244 recvs, seed 1; the committed
bench_data/resnet_v2_101_training-s1.json.gz, which both arms read), 2^24 =
16,777,216 random recv orders (seeds 1..2^24), each = random_schedule(seed)
+ gated simulate with choice_seed = seed (the `sched sweep` loop,
sched_main.cpp:472-477), reduced to min/argmin makespan + 1000-bin
efficiency histogram. At N > 1 GPUs the same fixed 2^24 orders are split
into contiguous shards (strong scaling, one NCCL all-reduce per step); the
weak view (2^24 per GPU) is reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. `value` = device-timed sims/s of the whole
job; `e2e` = the same through the C ABI with host buffers (cs_sweep_random);
`roofline` = the binding resource of the dominant kernel (instruction issue,
warp-instructions per ordering from the committed ncu capture x this run's
orderings/s), with SURVEY §8d's HBM-equivalent B_sim = 12R + 2V + 2E + 16
bytes per ordering in `roofline_hbm`; `cpu_baseline` times the reference
library (oracle/_ref, built from /root/reference) on this host.
`--impl reference` runs only the reference library (never this one) on the
same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL = "resnet_v2_101_training"
BRANCHY = "resnet_v2_101_training_branchy"
COUNT = 1 << 24
SEED_LO = 1
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled every 5 ms (NVML) during the timed
    region; falls back to `nvidia-smi -lms 100` when NVML is unavailable."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu, self.sm, self.mx, self.reasons = gpu, [], None, set()
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
        except Exception:
            self.nvml = None
            self.t = threading.Thread(target=self._smi_loop, daemon=True)
        self.t.start()
        return self

    def _nvml_loop(self):
        p = self.nvml
        while not self.stop.is_set():
            try:
                self.sm.append(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
                bits = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons |= {n for b, n in self.REASONS.items() if bits & b}
            except Exception:
                pass
            time.sleep(0.005)

    def _smi_loop(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                     "--format=csv,noheader,nounits", "-lms", "100"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) >= 6 and r[0].isdigit():
                self.sm.append(float(r[0]))
                self.mx = float(r[1])
                self.reasons |= {n for n, v in zip(names, r[2:6]) if v.lower() == "active"}
            if self.stop.is_set():
                break
        proc.terminate()

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=2)

    def summary(self, load_mhz_floor=300):
        loaded = [s for s in self.sm if s > load_mhz_floor] or self.sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}



def bench_json(model):
    """The committed input DAG (reference-format JSON, tools/make_bench_data.py)."""
    import gzip
    with gzip.open(os.path.join(ROOT, "bench_data", f"{model}-s1.json.gz"), "rb") as f:
        return f.read().decode()


def graph_file(model):
    d = tempfile.mkdtemp(prefix="tictac_bench_")
    p = os.path.join(d, f"{model}.json")
    with open(p, "w") as f:
        f.write(bench_json(model))
    return p


def shape(text):
    doc = json.loads(text)
    return {"ops": len(doc["ops"]), "edges": len(doc["edges"]),
            "recvs": sum(op["kind"] == "recv" for op in doc["ops"])}


def workload_config(world):
    """The `config` object, identical in both arms."""
    s = shape(bench_json(MODEL))
    return {"workload": f"config4: {MODEL} DAG seed 1 ({s['ops']} ops / {s['edges']} edges / {s['recvs']} recvs, "
                        f"bench_data/{MODEL}-s1.json.gz), {COUNT} random recv orders per step (seeds 1..{COUNT}), "
                        f"gated, choice_seed=seed; min/argmin makespan + E histogram",
            "parallelism": f"{COUNT} orders split into {world} contiguous seed shards (one per GPU), "
                           f"one NCCL all-reduce per step" if world > 1 else "1 GPU",
            "l2": "flushed between steps (256 MiB write)"}


def b_sim(info):
    """SURVEY §8d algorithmic bytes per ordering: 12R + 2V + 2E + 16."""
    return 12 * info["recvs_per_worker"] + 2 * info["ops"] + 2 * info["edges"] + 16


def ncu_summary(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def issue_roofline(summary, orders_per_s, mhz, traffic_scale):
    """Binding roofline of a sweep kernel: warp-instructions per ordering
    (ncu, committed summary) x this run's orderings/s against 148 SMs x 4
    schedulers x SM clock; traffic = ncu DRAM bytes scaled to the launch."""
    if not summary:
        return None
    ipo = summary["warp_instructions_per_ordering"]
    peak = 148 * 4 * mhz * 1e6
    ach = ipo * orders_per_s
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s", "frac": ach / peak,
            "traffic": summary["dram_bytes_per_launch"] * traffic_scale / summary["orderings"],
            "warp_inst_per_order": ipo, "kernel": summary["kernel"].split("(")[0],
            "source": "instructions per ordering and DRAM bytes from the committed ncu capture (profiles/); "
                      "orderings/s from this run's CUDA events; peak = 148 SMs x 4 schedulers x SM clock under load"}


def hbm_roofline(bsim, orders_per_s, hbm, peak_src):
    ach = bsim * orders_per_s / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "algorithmic_bytes_per_order": bsim, "peak_source": peak_src,
            "note": "SURVEY §8d B_sim = 12R+2V+2E+16 bytes per ordering for a design that streams per-ordering "
                    "state through HBM; the fused kernels keep it on chip (DRAM traffic ~0), so this "
                    "HBM-equivalent exceeds 1 and the binding resource is instruction issue (roofline)"}


def device_rate(plan, lo, n, key_base, stream, d_i64, d_f64, steps=5, flush=None):
    """Median kernel time of plan.run over n seeds (CUDA events, launching stream)."""
    import torch
    ts = []
    for _ in range(steps + 2):
        if flush is not None:
            flush.fill_(1)
        plan.reset(stream.cuda_stream, d_i64.data_ptr(), d_f64.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.run(lo, n, key_base, stream.cuda_stream, None, d_i64.data_ptr(), d_f64.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts[2:])[len(ts[2:]) // 2]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_sweep(path, seed_lo, count, threads, noise=None, out_path="-"):
    import oracle
    cmd = [oracle.REF_SWEEP, "sweep", path, "declared", str(seed_lo), str(count), str(threads), out_path]
    if noise is not None:
        cmd.append(repr(float(noise)))
    r = subprocess.run(cmd, capture_output=True, text=True, check=True)
    return json.loads(r.stdout)


def single_report(lib, reps=7):
    """One cs_simulate + cs_report_json (the event list) for a random order,
    configs 1 and 4, median of `reps` calls — this library, and the
    reference library on one host core when oracle/_ref is built; also
    cs_simulate + cs_report_makespan alone (no event list requested)."""
    from paper_1803_03288_b200 import capi
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    libs = {"ours": lib}
    if oracle.ref_available():
        libs["reference_cpu"] = capi.Lib(oracle.REF_LIB)
    out = {}
    for m in ("resnet_v2_50_inference", MODEL):
        text = lib.model(m, 1).serialize()
        row, docs = {}, {}
        for name, L in libs.items():
            g = L.graph(text)
            o = g.declared()
            s = g.random(1)
            ts, tm = [], []
            for _ in range(reps + 1):
                t = time.perf_counter()
                js = g.simulate(o, s, capi.policy(True, 1, 0.0)).json()
                ts.append(time.perf_counter() - t)
                t = time.perf_counter()
                g.simulate(o, s, capi.policy(True, 1, 0.0)).makespan()
                tm.append(time.perf_counter() - t)
            row[f"{name}_ms"] = 1000 * sorted(ts[1:])[reps // 2]
            row[f"{name}_makespan_only_ms"] = 1000 * sorted(tm[1:])[reps // 2]
            docs[name] = js
        if len(docs) == 2:
            row["identical_json"] = docs["ours"] == docs["reference_cpu"]
        out[m] = row
    return out


def sweep_vs_reference(lib, g, gpath, workload, noise=None, count=1 << 18, ref_target_s=5.0):
    """A sweep through cs_sweep_random (host buffers, per-seed makespans out)
    beside the reference library on all host cores for the same seeds, whose
    sample's makespans are compared value by value."""
    from paper_1803_03288_b200.capi import policy
    o = g.declared()
    pol = policy(True, 0, noise or 0.0)
    g.sweep_random(o, SEED_LO, count, pol, makespans=True)  # warm (plans, scratch)
    t = time.perf_counter()
    res = g.sweep_random(o, SEED_LO, count, pol, makespans=True)
    dt = time.perf_counter() - t
    out = {"workload": workload, "sims": count, "seconds": round(dt, 4), "sims_per_s": count / dt,
           "path": g.sweep_path(o, pol)["path"]}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    if oracle.ref_available():
        cores = os.cpu_count() or 1
        cal = ref_sweep(gpath, SEED_LO, cores * 2, cores, noise)
        n = min(count, max(cores, int(cal["sims"] / max(cal["seconds"], 1e-9) * ref_target_s)))
        binp = os.path.join(os.path.dirname(gpath), "ref_cmp.bin")
        r = ref_sweep(gpath, SEED_LO, n, cores, noise, binp)
        ref_ms = np.fromfile(binp, dtype=np.int64)[:n]  # (clusters: per-worker makespans follow)
        out["reference_cpu"] = {"sims_per_s": r["sims"] / r["seconds"], "cores": cores, "sims": n,
                                "seconds": round(r["seconds"], 3)}
        out["sample_identical"] = bool(np.array_equal(ref_ms, res["makespans"][:n]))
    return out


def exact_paths(lib, path):
    """Outside the plain gated closed form: (a) config 4 with reorder noise
    0.1 — still the closed form, on the noise-permuted gate sequence; (b)
    config 3 (VGG-16 x 4 workers / 1 PS) with PS operations that take time
    (100 us each): closed-form workers + the exact send phase; (c) the same
    with two parameter servers; (d) branchy workers in such a cluster, which
    only the exact event replica covers."""
    g4 = lib.graph(bench_json(MODEL))
    a = sweep_vs_reference(lib, g4, path, f"config4 {MODEL}, counter gate + reorder noise 0.1 "
                                          f"(closed form on the noise-permuted gate order)", 0.1, 1 << 22)
    c3 = lib.model("vgg16_training", 1).expand(4, 1, 100)
    p3 = os.path.join(os.path.dirname(path), "config3_ps100.json")
    with open(p3, "w") as f:
        f.write(c3.serialize())
    b = sweep_vs_reference(lib, c3, p3, "config3 vgg16_training x 4 workers / 1 PS with 100 us PS ops, full "
                                        "makespans (closed-form workers + exact send phase, cluster_ps_kernel)",
                           None, 1 << 22)
    c4 = lib.model("vgg16_training", 1).expand(4, 2, 100)
    p4 = os.path.join(os.path.dirname(path), "config3_2ps.json")
    with open(p4, "w") as f:
        f.write(c4.serialize())
    c = sweep_vs_reference(lib, c4, p4, "config3 vgg16_training x 4 workers / 2 PS with 100 us PS ops, full "
                                        "makespans (two channels per worker, two PS cores: cluster_ps_kernel)",
                           None, 1 << 22)
    c5 = lib.model("vgg16_training_branchy", 1).expand(4, 1, 100)
    p5 = os.path.join(os.path.dirname(path), "config3_branchy_ps100.json")
    with open(p5, "w") as f:
        f.write(c5.serialize())
    e = sweep_vs_reference(lib, c5, p5, "vgg16_training_branchy x 4 workers / 1 PS with 100 us PS ops, full "
                                        "makespans (branchy workers: compute ops compete while PS ops take time, "
                                        "outside every closed form: exact event replica, thread per run)",
                           None, 1 << 18)
    return {"noise_sweep_config4": a, "ps_send_phase_config3_ps100": b, "ps_send_phase_config3_2ps": c,
            "event_replica_branchy_cluster": e}


def cpu_baseline(path, target_s=10.0, g=None, o=None):
    """Reference library on this host: calibrate, then ~target_s of wall time
    (and at least 100,000 seeds) with one thread per core over contiguous
    seed slices. When the product
    graph/oracle are given, the sample's makespans are compared value by
    value with this library's for the same seeds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    if not oracle.ref_available():
        return None
    cores = os.cpu_count() or 1
    cal = ref_sweep(path, SEED_LO, cores * 2, cores)
    rate = cal["sims"] / max(cal["seconds"], 1e-9)
    n = max(cores, int(rate * target_s), 100_000)  # >= 100k seeds at config 4
    binp = os.path.join(os.path.dirname(path), "ref_sample.bin")
    r = ref_sweep(path, SEED_LO, n, cores, None, binp)
    out = {"value": r["sims"] / r["seconds"], "unit": "sims/s", "cores": cores, "kind": "reference",
           "nproc": os.cpu_count(), "cpu_model": cpu_model(),
           "sample": f"seeds {SEED_LO}..{SEED_LO + n - 1} of the same workload ({n} sims, "
                     f"{r['seconds']:.1f} s wall, {cores} threads, oracle/_ref libcommsched -O3)"}
    if g is not None:
        ours = g.sweep_random(o, SEED_LO, n, None, makespans=True)["makespans"]
        out["sample_identical_to_ours"] = bool(np.array_equal(ours, np.fromfile(binp, dtype=np.int64)))
    # reference TIC/TAC wall time on config 1 (single thread: the reference has none)
    try:
        p1 = os.path.join(os.path.dirname(path), "config1.json")
        with open(p1, "w") as f:
            f.write(bench_json("resnet_v2_50_inference"))
        for algo, arg in (("tac", "declared"), ("tic", "amended")):
            rr = subprocess.run([oracle.REF_SWEEP, algo, p1, arg], capture_output=True, text=True, check=True)
            out[f"{algo}_config1_seconds"] = json.loads(rr.stderr.strip().splitlines()[-1])["seconds"]
    except Exception as e:  # reported, not fatal
        out["tac_error"] = str(e)[:200]
    return out


def tac_times(lib, top=False, hbm=None):
    """TAC wall time through cs_schedule_tac (device), seconds; SURVEY §8d
    configs 1, 2, 4 and the config-5 layered sweep. With `hbm`, also the
    SURVEY's algorithmic bytes B_TAC and B_TIC (cs_tac_traffic) over those
    times."""
    out, roof, tic, tic_roof = {}, {}, {}, {}
    names = ["resnet_v2_50_inference", "inception_v3_training", "resnet_v2_101_training",
             "layered:10000:1000", "layered:100000:10000"] + (["layered:1000000:100000"] if top else [])
    for name in names:
        g = lib.model(name, 1)
        o = g.declared()
        g.tac(o)  # warm (upload, allocator pools, context)
        t = time.perf_counter()
        g.tac(o)
        dt = time.perf_counter() - t
        out[name] = round(dt, 6)
        t = time.perf_counter()
        g.tic("amended")
        dt_tic = time.perf_counter() - t
        tic[name] = round(dt_tic, 6)
        if hbm:
            tr = g.tac_traffic(o)
            gbs = tr["B_TAC"] / dt / 1e9
            R = g.recv_count()
            # TAC is R dependent rounds: the binding limit is the round latency
            # (grid/block barriers + dependent loads), not bytes; SURVEY §8d's
            # B_TAC over the time is kept as the secondary HBM-equivalent (the
            # kernels retire over row_nnz (row, recv) pairs, not nnz)
            roof[name] = {"bound": "round latency", "rounds": R, "us_per_round": 1e6 * dt / max(1, R),
                          "B_TAC_bytes": tr["B_TAC"], "hbm_equivalent_GBps": gbs, "hbm_equivalent_frac": gbs / hbm,
                          "nnz": tr["nnz"], "row_nnz": tr["row_nnz"], "rows": tr["rows"]}
            gbs = tr["B_TIC"] / dt_tic / 1e9
            tic_roof[name] = {"bound": "launch latency (one round of dependent kernels)", "B_TIC_bytes": tr["B_TIC"],
                              "hbm_equivalent_GBps": gbs, "hbm_equivalent_frac": gbs / hbm}
    return (out, roof, tic, tic_roof) if hbm else out


def sweep_rate(g, o, count):
    g.sweep_random(o, 1, min(count, 1 << 16))  # plan + warm
    t = time.perf_counter()
    st = g.sweep_random(o, 1, count)
    return st, count / (time.perf_counter() - t)


def config2(lib, model):
    g = lib.model(model, 1)
    o = g.declared()
    U, L = g.bounds(o)
    g.tac(o)
    t = time.perf_counter()
    s = g.tac(o)
    tac_s = time.perf_counter() - t
    m_tac = g.simulate(o, s).makespan()
    st, rate = sweep_rate(g, o, 1_000_000)
    h = st["e_hist"]
    mean_e = (U * st["count"] - st["sum_us"]) / (st["count"] * (U - L))
    return {f"config2_{model}": {
        "ops": g.op_count(), "edges": g.edge_count(), "recvs": g.recv_count(), "path": g.sweep_path(o)["path"],
        "tac_seconds": round(tac_s, 6), "tac_makespan_us": m_tac,
        "tac_E": (U - m_tac) / (U - L), "random_orders": st["count"], "sims_per_s": rate,
        "min_us": st["min_us"], "argmin_seed": st["argmin_seed"], "mean_E": mean_e,
        "E_hist_nonzero_bins": int((h > 0).sum()), "E_best_bin": int(max(i for i in range(1000) if h[i]))}}


def dag_config4(lib, hbm, peak_src, mhz, stream, d_i64, d_f64, flush):
    """The general-DAG closed form (dag_sweep_kernel) at config-4 size: the
    Inception-style branchy ResNet-v2-101-shaped DAG (same recvs, bytes and
    compute times as config 4, not nested), 2^24 orders per step, device
    kernel time; e2e through cs_sweep_random; the reference library on the
    host cores for a bounded sample, compared value by value."""
    from paper_1803_03288_b200 import capi
    text = bench_json(BRANCHY)
    g = lib.graph(text)
    o = g.declared()
    plan = capi.SweepPlan.create(g, o)
    info = plan.info()
    ms = device_rate(plan, SEED_LO, COUNT, SEED_LO, stream, d_i64, d_f64, flush=flush)
    rate = COUNT / (ms / 1000.0)
    st = plan.finish(d_i64.cpu().numpy(), d_f64.cpu().numpy(), SEED_LO)
    t = time.perf_counter()
    g.sweep_random(g.declared(), SEED_LO, COUNT)
    e2e = COUNT / (time.perf_counter() - t)
    path = os.path.join(tempfile.mkdtemp(prefix="tictac_bench_"), f"{BRANCHY}.json")
    with open(path, "w") as f:
        f.write(text)
    out = {"workload": f"{BRANCHY} DAG seed 1 ({info['ops']} ops / {info['edges']} edges / "
                       f"{info['recvs_per_worker']} recvs, {info['joins']} join classes, "
                       f"{info['program_records']} program records), {COUNT} random orders per step",
           "kernel": info["kernel"], "kernel_ms": ms, "sims_per_s": rate, "e2e_sims_per_s": e2e,
           "min_us": st["min_us"], "argmin_seed": st["argmin_seed"],
           "roofline_hbm": hbm_roofline(b_sim(info), rate, hbm, peak_src),
           "roofline": issue_roofline(ncu_summary("dag_ncu_summary.json"), rate, mhz, COUNT)}
    ref = sweep_vs_reference(lib, g, path, "reference sample", None, 1 << 18)
    out["reference_cpu"] = ref.get("reference_cpu")
    out["sample_identical"] = ref.get("sample_identical")
    return out


def other_configs(lib):
    """SURVEY §8d configs 1-3 through the public C ABI (e2e, host buffers)."""
    from paper_1803_03288_b200 import capi
    out = {}
    # config 1: ResNet-v2-50 inference — TIC (both modes) + TAC, each simulated
    g = lib.model("resnet_v2_50_inference", 1)
    o = g.declared()
    U, L = g.bounds(o)
    c1 = {"ops": g.op_count(), "recvs": g.recv_count()}
    for name, fn in (("tic_amended", lambda: g.tic("amended")), ("tic_literal", lambda: g.tic("literal")),
                     ("tac", lambda: g.tac(o))):
        fn()
        t = time.perf_counter()
        s = fn()
        dt = time.perf_counter() - t
        r = g.simulate(o, s)
        m = json.loads(g.metrics_text(o, r))
        c1[name] = {"seconds": round(dt, 6), "makespan_us": r.makespan(), "E": m["E"]}
    st, rate = sweep_rate(g, o, 1000)
    c1["random_1000"] = {"min_us": st["min_us"], "mean_us": st["sum_us"] / st["count"], "sims_per_s": rate}
    out["config1_resnet_v2_50_inference"] = c1
    # config 2: Inception-v3 training — TAC + 1M random orders, E histogram,
    # on the survey's backbone DAG and on the branchy Inception-style one
    out.update(config2(lib, "inception_v3_training"))
    out.update(config2(lib, "inception_v3_training_branchy"))
    # config 3: VGG-16 training, 4 workers / 1 PS — straggler spread
    v = lib.model("vgg16_training", 1).expand(4, 1, 0)
    o = v.declared()
    st, rate = sweep_rate(v, o, 1_000_000)
    sh = st["straggler_hist"]
    r_tic = v.simulate(o, v.tic())
    strag_tic = json.loads(r_tic.iteration_json())["straggler"]
    out["config3_vgg16_4workers"] = {
        "random_orders": st["count"], "sims_per_s": rate, "workers": st["n_workers"],
        "path": v.sweep_path(o)["path"],
        "straggler_mean": st["straggler_sum"] / st["count"],
        "straggler_max_bin": int(max(i for i in range(1000) if sh[i])),
        "makespan_min_us": st["min_us"], "makespan_max_us": st["max_us"],
        "iteration_min_us": st["iter_min_us"], "iteration_max_us": st["iter_max_us"],
        "tic_common_order_straggler": strag_tic}
    # batched brute force: all R! orders on the device
    bf = {}
    for R in (8, 10, 12):
        g = lib.generate("chain", R, 1, "1", 5)
        o = g.declared()
        g.brute_force_text(o, None, R)  # warm (plan, pool buffers)
        t = time.perf_counter()
        res = json.loads(g.brute_force_text(o, None, R))
        bf[f"R{R}"] = {"permutations": int(np.prod(np.arange(1, R + 1, dtype=np.float64))),
                       "seconds": round(time.perf_counter() - t, 4), "best_us": res["makespan_us"],
                       "distinct_makespans": len(res["distribution"])}
    out["brute_force_chain"] = bf
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference library's own per-seed loop (oracle/_ref,
    compiled from /root/reference; this library is never loaded) on the host
    cores, rank 0 only, on the same committed DAG and config."""
    if rank != 0:
        return
    path = graph_file(MODEL)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    cores = os.cpu_count() or 1
    base = {"metric": "recv-order makespan sims/sec", "unit": "sims/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "dtype": "int64", "data": "synthetic",
            "config": workload_config(world)}
    if not oracle.ref_available():
        base["unavailable"] = "oracle/_ref (reference build) missing"
        emit(base)
        return
    cal = ref_sweep(path, SEED_LO, cores * 2, cores)
    rate = cal["sims"] / max(cal["seconds"], 1e-9)
    per_step = max(cores, int(rate * 4.0))  # ~4 s of wall per step
    for _ in range(args.warmup):
        ref_sweep(path, SEED_LO, max(cores, per_step // 8), cores)
    secs, sims = 0.0, 0
    for k in range(args.steps):
        r = ref_sweep(path, SEED_LO + k * per_step, per_step, cores)
        secs += r["seconds"]
        sims += r["sims"]
    v = sims / secs
    base.update({"value": v, "ms_per_step": 1000 * secs / args.steps, "vs_baseline": None,
                 "cpu_baseline": {"value": v, "unit": "sims/s", "cores": cores, "kind": "reference",
                                  "nproc": os.cpu_count(), "cpu_model": cpu_model(),
                                  "sample": f"{per_step} seeds per step (a bounded sample of the {COUNT}-order "
                                            f"step), {cores} threads, oracle/_ref libcommsched -O3"},
                 "e2e": {"value": v, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    emit(base)


_JSON_FD = None


def emit(obj):
    """The one JSON line on stdout. Library/NCCL chatter that would land on
    fd 1 is routed to stderr for the whole run (see main)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(obj) + "\n").encode())


def timed_steps(step, steps, world, stream, flush):
    """K timed steps (CUDA events on the launching stream), L2 flushed and a
    barrier before each; returns the per-step times (ms)."""
    import torch
    import torch.distributed as dist
    out = []
    for _ in range(steps):
        flush.fill_(1)  # L2 flush between timed steps (outside the timing)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return out


def max_over_ranks(x, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # anything else written to stdout (e.g. NCCL's version banner) goes to stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tac", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--config5-top", action="store_true", help="also TAC at 10^6 ops / 10^5 recvs")
    args = ap.parse_args()
    rank, world, local = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1803_03288_b200 import capi
    from paper_1803_03288_b200 import dist as pdist
    lib = capi.Lib()
    text = bench_json(MODEL)
    path = graph_file(MODEL)
    g = lib.graph(text)
    o = g.declared()
    plan = capi.SweepPlan.create(g, o)
    info = plan.info()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    d_i64 = torch.zeros(capi.DSTATS_I64, dtype=torch.int64, device="cuda")
    d_f64 = torch.zeros(capi.DSTATS_F64, dtype=torch.float64, device="cuda")
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    buf = torch.zeros(pdist.packed_words(world), dtype=torch.int64, device="cuda")
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def make_step(lo, n):
        def step():
            plan.reset(sptr, d_i64.data_ptr(), d_f64.data_ptr())
            k0.record(stream)
            plan.run(lo, n, SEED_LO, sptr, None, d_i64.data_ptr(), d_f64.data_ptr())
            k1.record(stream)
            if world > 1:  # the step's one reduction: pack, one NCCL all-reduce, unpack
                pdist.reduce_stats_device(lib, d_i64, d_f64, rank, world, buf, sptr)
        return step

    # headline: config 4's fixed 2^24 orders, contiguous shards over the ranks
    lo, n = pdist.shard(SEED_LO, COUNT, rank, world)
    step = make_step(lo, n)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches0 = lib.launches()
    kern_ms = []
    with ClockSampler(local) as clocks:
        def kstep():
            step()
        step_ms = []
        for _ in range(args.steps):
            step_ms += timed_steps(kstep, 1, world, stream, flush)
            kern_ms.append(k0.elapsed_time(k1))
    launches = lib.launches() - launches0
    stats = plan.finish(d_i64.cpu().numpy(), d_f64.cpu().numpy(), SEED_LO)
    ms_per_step = max_over_ranks(sum(step_ms), world) / args.steps
    kern_per_step = max_over_ranks(sum(kern_ms), world) / args.steps
    value = COUNT / (ms_per_step / 1000.0)

    # weak view at N > 1: 2^24 orders per GPU
    weak = None
    if world > 1:
        wstep = make_step(SEED_LO + rank * COUNT, COUNT)
        for _ in range(3):
            wstep()
        torch.cuda.synchronize()
        wms = max_over_ranks(sum(timed_steps(wstep, args.steps, world, stream, flush)), world) / args.steps
        weak = {"orders_per_gpu": COUNT, "total_orders": COUNT * world, "ms_per_step": wms,
                "value": COUNT * world / (wms / 1000.0), "unit": "sims/s"}

    # e2e: the user path through the public C ABI with host buffers: the DAG
    # is parsed once (cs_graph_parse, as the reference's CLI does); every step
    # builds a fresh time oracle (cs_oracle_declared) and calls cs_sweep_random
    # on the rank's shard, which weights the graph's cached analysis with the
    # oracle's durations, uploads the tables, runs and reads the statistics
    # back; then the cross-rank reduction of the host results.
    ge = lib.graph(text)
    e2e_ms = []
    for _ in range(max(2, min(4, args.steps)) + 1):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st = ge.sweep_random(ge.declared(), lo, n)
        hv = torch.tensor([st["min_us"], st["sum_us"]] + list(st["e_hist"]), dtype=torch.int64, device="cuda")
        if world > 1:
            dist.all_reduce(hv[1:])
            dist.all_reduce(hv[:1], op=dist.ReduceOp.MIN)
        hv.cpu()
        e2e_ms.append((time.perf_counter() - t0) * 1000)
    e2e_t = max_over_ranks(statistics.median(e2e_ms[1:]), world)
    e2e_value = COUNT / (e2e_t / 1000.0)
    h2d = info["uploaded_bytes"]  # tables and images uploaded per call (counted by the plan builder)
    d2h = 8 * capi.DSTATS_I64 + 8 * capi.DSTATS_F64

    clocks_summary = clocks.summary()
    if rank == 0:
        hbm, peak_src = peaks()
        mhz = clocks_summary.get("sm_mhz") or 1965.0
        per_gpu_rate = (COUNT / world) / (kern_per_step / 1000.0)
        summary = ncu_summary("sweep_ncu_summary.json")
        roof = issue_roofline(summary, per_gpu_rate, mhz, COUNT / world)
        out = {
            "metric": "recv-order makespan sims/sec", "value": value, "unit": "sims/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": workload_config(world),
            "gpu_launches": launches,  # this library's kernels inside the timed region (all K steps)
            "gpu_launches_per_step": launches // max(1, args.steps),
            "kernel_ms_per_step": kern_per_step,
            "roofline": roof,
            "roofline_hbm": hbm_roofline(b_sim(info), per_gpu_rate, hbm, peak_src),
            "roofline_smem": {"bound": "smem", "achieved": b_sim(info) * per_gpu_rate / 1e9,
                              "peak": 148 * 128 * mhz * 1e6 / 1e9, "unit": "GB/s",
                              "frac": b_sim(info) * per_gpu_rate / (148 * 128 * mhz * 1e6),
                              "note": "SURVEY §8d secondary: B_sim against 148 SMs x 128 B/clk x SM clock"},
            "e2e": {"value": e2e_value, "unit": "sims/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_t,
                    "call": "per step: cs_oracle_declared + cs_sweep_random on the rank's shard (per-oracle tables "
                            "built and uploaded, statistics read back to the host); DAG parsed once"},
            "result": {"min_us": stats["min_us"], "argmin_seed": stats["argmin_seed"],
                       "max_us": stats["max_us"], "mean_us": stats["sum_us"] / max(1, stats["count"]),
                       "count_checked": int(stats["count"])},
            "clocks": clocks_summary,
        }
        if weak:
            out["weak_scaling"] = weak
        if not args.no_tac:
            (out["tac_seconds"], out["tac_roofline"], out["tic_amended_seconds"],
             out["tic_roofline"]) = tac_times(lib, top=args.config5_top, hbm=hbm)
            if world > 1:
                out["tac_note"] = ("TAC is R dependent rounds and runs on one GPU (rank 0) at any N: a "
                                   "sharded round needs >= 2 cross-GPU exchanges (NCCL all-reduce 16-29 us, "
                                   "NVLink peer-flag round trip 2.6 us; profiles/r01_cross_gpu_latency.json) "
                                   "on rounds of 1.3-6.3 us; DESIGN.md section 5")
        if not args.no_configs and world == 1:
            out["configs"] = {"dag_branchy_config4": dag_config4(lib, hbm, peak_src, mhz, stream, d_i64, d_f64,
                                                                 flush)}
            out["configs"].update(other_configs(lib))
            out["configs"].update(exact_paths(lib, path))
            out["configs"]["single_report_simulate_json"] = single_report(lib)
        if not args.no_cpu and world == 1:
            out["cpu_baseline"] = cpu_baseline(path, g=g, o=o)
        emit(out)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
