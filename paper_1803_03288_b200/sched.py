"""Batched drivers with the reference CLI's behaviour for `sweep` and
`bruteforce` (reference tools/sched_main.cpp; the reference CLI itself needs
CLI11 and is not built here):

    python -m paper_1803_03288_b200.sched sweep --graph g.json --oracle declared \
        --algo random --seeds 1..100000 --out sweep.csv
    python -m paper_1803_03288_b200.sched bruteforce --graph g.json --max-recvs 12

Same flags, `--config file.json` defaults (JSON keys = flag names, flags win;
sched_main.cpp:142-255), seed lists `a..b` (capped below 10^6) or `a,b,c`
(sched_main.cpp:112-140), CSV bytes and stdout summary of cmd_sweep
(sched_main.cpp:452-502), artifacts staged and committed all-or-nothing
(sched_main.cpp:65-87), exit codes = status codes. The per-seed loop of the
reference becomes one cs_sweep_random call per contiguous seed run.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from fractions import Fraction

from .capi import CS_ERR_INTERNAL, CS_ERR_IO, CS_ERR_PARAMETER, CS_ERR_VALIDATION, CsError, Lib, SimPolicy


class Exit(Exception):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.message = message


def read_file(path: str) -> str:
    try:
        with open(path, "rb") as f:
            return f.read().decode()
    except OSError:
        raise Exit(CS_ERR_IO, "cannot read " + path)


def decimal6(num: int, den: int) -> str:
    """sched_main.cpp:89-101: six places, half away from zero."""
    scaled = num * 1000000
    neg = scaled < 0
    scaled = -scaled if neg else scaled
    q, r = divmod(scaled, den)
    if 2 * r >= den:
        q += 1
    return f"{'-' if neg else ''}{q // 1000000}.{q % 1000000:06d}"


def parse_uint(s: str) -> int:
    # std::stoull accepts leading whitespace and '+'; the whole string must parse
    t = s.lstrip(" \t\n\v\f\r")
    if t.startswith("+"):
        t = t[1:]
    if not t or not t.isdigit() or int(t) >= 1 << 64:
        raise Exit(CS_ERR_PARAMETER, "bad seed value: " + s)
    return int(t)


def parse_seeds(text: str) -> list:
    if ".." in text:
        a, b = text.split("..", 1)
        lo, hi = parse_uint(a), parse_uint(b)
        if hi < lo:
            raise Exit(CS_ERR_PARAMETER, "seed range is empty: " + text)
        if hi - lo >= 1000000:
            raise Exit(CS_ERR_PARAMETER, "seed range too large: " + text)
        return list(range(lo, hi + 1))
    seeds = [parse_uint(x) for x in text.split(",") if x]
    if not seeds:
        raise Exit(CS_ERR_PARAMETER, "no seeds in: " + text)
    return seeds


class Artifacts:
    def __init__(self):
        self.files = []

    def add(self, path: str, content: str):
        if path:
            self.files.append((path, content))

    def commit(self):
        written = []
        for path, content in self.files:
            try:
                with open(path, "wb") as f:
                    f.write(content.encode())
                written.append(path)
            except OSError:
                for w in written + [path]:
                    try:
                        os.remove(w)
                    except OSError:
                        pass
                raise Exit(CS_ERR_IO, "cannot write " + path)


FLAGS = {  # flag -> (config key, type, default)
    "graph": ("graph", str, ""), "oracle": ("oracle", str, "declared"), "traces": ("traces", str, ""),
    "bandwidth": ("bandwidth", int, 0), "algo": ("algo", str, "none"), "mode": ("mode", str, "amended"),
    "seed": ("seed", int, 0), "schedule": ("schedule", str, ""), "enforce": ("enforce", str, "counter"),
    "noise": ("noise", float, 0.0), "choice_seed": ("choice-seed", int, None), "seeds": ("seeds", str, ""),
    "out": ("out", str, ""), "max_recvs": ("max-recvs", int, 8),
}


def options(argv):
    ap = argparse.ArgumentParser(prog="sched")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("sweep", "bruteforce"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        for flag, (key, typ, _) in FLAGS.items():
            if name == "bruteforce" and flag in ("seeds", "algo", "mode", "seed", "schedule", "choice_seed"):
                continue
            p.add_argument("--" + flag.replace("_", "-"), dest=flag, type=typ, default=None)
    o = ap.parse_args(argv)
    cfg = {}
    if o.config:
        try:
            cfg = json.loads(read_file(o.config))
        except json.JSONDecodeError as e:
            raise Exit(CS_ERR_VALIDATION, f"config: {e}")
        if not isinstance(cfg, dict):
            raise Exit(CS_ERR_VALIDATION, "config must be a JSON object")
    for flag, (key, typ, default) in FLAGS.items():
        if not hasattr(o, flag):
            setattr(o, flag, default)
        elif getattr(o, flag) is None:  # flags win over the config file
            setattr(o, flag, typ(cfg[key]) if key in cfg else default)
    return o


def load(lib: Lib, o):
    if not o.graph:
        raise Exit(CS_ERR_PARAMETER, "--graph is required")
    g = lib.graph(read_file(o.graph))
    if o.oracle == "declared":
        oracle = g.declared()
    elif o.oracle == "general":
        oracle = g.general()
    elif o.oracle == "traces":
        if not o.traces:
            raise Exit(CS_ERR_PARAMETER, "--oracle traces needs --traces")
        oracle = g.traces(read_file(o.traces))
    elif o.oracle == "bandwidth":
        if o.bandwidth <= 0:
            raise Exit(CS_ERR_PARAMETER, "--oracle bandwidth needs --bandwidth > 0")
        oracle = g.bandwidth(o.bandwidth)
    else:
        raise Exit(CS_ERR_PARAMETER, "unknown oracle source: " + o.oracle)
    return g, oracle


def make_policy(o) -> SimPolicy:
    if o.enforce not in ("counter", "none"):
        raise Exit(CS_ERR_PARAMETER, "unknown enforcement: " + o.enforce)
    cs = o.choice_seed if o.choice_seed is not None else o.seed
    return SimPolicy(1 if o.enforce == "counter" else 0, cs, o.noise)


def fixed_schedule(lib, g, oracle, o):
    if o.schedule and o.algo != "file":
        raise Exit(CS_ERR_PARAMETER, "--schedule needs --algo file")
    if o.algo == "none":
        return None
    if o.algo == "tic":
        return g.tic(o.mode)
    if o.algo == "tac":
        return g.tac(oracle)
    if o.algo == "file":
        if not o.schedule:
            raise Exit(CS_ERR_PARAMETER, "--algo file needs --schedule")
        text = read_file(o.schedule)
        s = lib.schedule_parse(text)
        if json.loads(text)["graph"] != g.name():
            raise Exit(CS_ERR_VALIDATION, f"schedule was computed for graph '{json.loads(text)['graph']}', "
                                          f"not '{g.name()}'")
        return s
    raise Exit(CS_ERR_PARAMETER, "unknown algorithm: " + o.algo)


def runs(seeds):
    """Split a seed list into maximal contiguous ascending runs."""
    out, start = [], 0
    for i in range(1, len(seeds) + 1):
        if i == len(seeds) or seeds[i] != seeds[i - 1] + 1:
            out.append((seeds[start], i - start))
            start = i
    return out


def cmd_sweep(lib: Lib, o) -> int:
    if not o.out:
        raise Exit(CS_ERR_PARAMETER, "--out is required")
    if not o.seeds:
        raise Exit(CS_ERR_PARAMETER, "--seeds is required")
    seeds = parse_seeds(o.seeds)
    g, oracle = load(lib, o)
    cluster = g.is_cluster()
    pol = make_policy(o)
    lines = ["seed,makespan_us,iteration_us,straggler" if cluster else "seed,makespan_us"]
    ms_all = []
    if o.algo == "random":
        for lo, n in runs(seeds):
            res = g.sweep_random(oracle, lo, n, pol, makespans=True, worker_makespans=cluster)
            for k in range(n):
                m = int(res["makespans"][k])
                ms_all.append(m)
                if cluster:
                    wm = [int(x) for x in res["worker_makespans"][k]]
                    hi, lo_m = max(wm), min(wm)
                    f = Fraction(hi - lo_m, hi) if hi else Fraction(0)
                    lines.append(f"{lo + k},{m},{hi},{decimal6(f.numerator, f.denominator)}")
                else:
                    lines.append(f"{lo + k},{m}")
    else:
        fixed = fixed_schedule(lib, g, oracle, o)
        for s in seeds:
            p = SimPolicy(pol.counter_gate, s, pol.reorder_noise)
            r = g.simulate(oracle, fixed, p)
            m = r.makespan()
            ms_all.append(m)
            if cluster:
                it = json.loads(r.iteration_json())
                st = it["straggler"]
                lines.append(f"{s},{m},{it['iteration_us']},{decimal6(st['num'], st['den'])}")
            else:
                lines.append(f"{s},{m}")
    arts = Artifacts()
    arts.add(o.out, "\n".join(lines) + "\n")
    arts.commit()
    print(f"sweep seeds={len(seeds)} min_us={min(ms_all)} max_us={max(ms_all)}")
    return 0


def cmd_bruteforce(lib: Lib, o) -> int:
    g, oracle = load(lib, o)
    text = g.brute_force_text(oracle, make_policy(o), o.max_recvs)
    arts = Artifacts()
    arts.add(o.out, text)
    arts.commit()
    res = json.loads(text)
    print(f"best m_us={res['makespan_us']} order={','.join(res['order'])}")
    return 0


def main(argv=None, lib: Lib | None = None) -> int:
    try:
        o = options(sys.argv[1:] if argv is None else argv)
    except Exit as e:
        print(f"error: {e.message}", file=sys.stderr)
        return e.code
    except SystemExit as e:  # argparse usage errors
        return CS_ERR_PARAMETER if e.code else 0
    try:
        lib = lib or Lib()
        return cmd_sweep(lib, o) if o.cmd == "sweep" else cmd_bruteforce(lib, o)
    except Exit as e:
        print(f"error: {e.message}", file=sys.stderr)
        return e.code
    except CsError as e:
        print(f"error: {e.message}", file=sys.stderr)
        return e.code
    except Exception as e:  # noqa: BLE001 — mirrors the reference's catch-all
        print(f"error: {e}", file=sys.stderr)
        return CS_ERR_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
