"""The batched `sweep` / `bruteforce` drivers (paper_1803_03288_b200/sched.py)
against the reference CLI's behaviour (tools/sched_main.cpp): seed parsing,
decimal6, config defaults, and — on the GPU — CSV bytes equal to the
reference library driven seed by seed exactly as cmd_sweep does."""
import json
import os

import pytest

import corpus
from paper_1803_03288_b200 import sched
from paper_1803_03288_b200.capi import policy


def test_seed_parsing_and_decimal6():
    assert sched.parse_seeds("3..6") == [3, 4, 5, 6]
    assert sched.parse_seeds("5,1,,9") == [5, 1, 9]
    assert sched.parse_seeds("0..999999")[-1] == 999999
    for bad, msg in (("5..4", "seed range is empty: 5..4"), ("0..1000000", "seed range too large: 0..1000000"),
                     ("x", "bad seed value: x"), (",,", "no seeds in: ,,"), ("1..2x", "bad seed value: 2x")):
        with pytest.raises(sched.Exit) as e:
            sched.parse_seeds(bad)
        assert e.value.code == 4 and e.value.message == msg
    assert sched.decimal6(2, 3) == "0.666667" and sched.decimal6(1, 8) == "0.125000"
    assert sched.decimal6(0, 1) == "0.000000" and sched.decimal6(-2, 3) == "-0.666667"


def test_config_defaults_and_required_flags(tmp_path, lib, toy_text):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"seeds": "1..3", "algo": "tic", "out": "ignored.csv"}))
    o = sched.options(["sweep", "--config", str(cfg), "--out", "x.csv"])
    assert (o.seeds, o.algo, o.out, o.oracle) == ("1..3", "tic", "x.csv", "declared")
    assert sched.main(["sweep", "--seeds", "1..2"], lib=lib) == 4  # --out is required
    bad = tmp_path / "bad.json"
    bad.write_text("[1]")
    assert sched.main(["sweep", "--config", str(bad)], lib=lib) == 2


def reference_csv(ref, text, seeds, algo):
    """cmd_sweep's loop (sched_main.cpp:452-502) over the reference library."""
    g = ref.graph(text)
    o = g.declared()
    cluster = g.is_cluster()
    fixed = {"none": None, "tic": g.tic("amended") if algo == "tic" else None}.get(algo)
    lines = ["seed,makespan_us,iteration_us,straggler" if cluster else "seed,makespan_us"]
    for s in seeds:
        sc = g.random(s) if algo == "random" else fixed
        r = g.simulate(o, sc, policy(True, s, 0.0))
        if cluster:
            it = json.loads(r.iteration_json())
            lines.append(f"{s},{r.makespan()},{it['iteration_us']},"
                         f"{sched.decimal6(it['straggler']['num'], it['straggler']['den'])}")
        else:
            lines.append(f"{s},{r.makespan()}")
    return "\n".join(lines) + "\n"


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["random", "tic", "none"])
def test_sweep_csv_matches_reference_loop(tmp_path, lib, ref, algo, capsys):
    graphs = corpus.worker_graphs(lib)[:4] + corpus.cluster_graphs(lib)[:2]
    for name, text in graphs:
        gp = tmp_path / "g.json"
        gp.write_text(text)
        out = tmp_path / "s.csv"
        seeds = "1..40" if algo == "random" else "3,1,2,9"
        rc = sched.main(["sweep", "--graph", str(gp), "--algo", algo, "--seeds", seeds, "--out", str(out)],
                        lib=lib)
        assert rc == 0
        want = reference_csv(ref, text, sched.parse_seeds(seeds), algo)
        assert out.read_text() == want, name
        line = capsys.readouterr().out.strip().splitlines()[-1]
        ms = [int(x.split(",")[1]) for x in want.splitlines()[1:]]
        assert line == f"sweep seeds={len(ms)} min_us={min(ms)} max_us={max(ms)}"


@pytest.mark.gpu
def test_bruteforce_driver(tmp_path, lib, ref):
    text = lib.generate("layered", 3, 2, "1", 4).serialize()
    gp = tmp_path / "g.json"
    gp.write_text(text)
    out = tmp_path / "bf.json"
    assert sched.main(["bruteforce", "--graph", str(gp), "--out", str(out)], lib=lib) == 0
    g = ref.graph(text)
    assert out.read_text() == g.brute_force_text(g.declared(), policy(True, 0, 0.0), 8)
    assert os.path.getsize(out) > 0
