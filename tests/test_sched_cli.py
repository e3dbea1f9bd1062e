"""The batched `sweep` / `bruteforce` drivers — paper_1803_03288_b200/sched.py
and the native paper_1803_03288_b200/tictac_sched (csrc/cli/sched_main.cpp) —
against the reference CLI's behaviour (tools/sched_main.cpp): seed parsing,
decimal6, config defaults, error codes and messages, and — on the GPU — CSV
bytes equal to the reference library driven seed by seed exactly as
cmd_sweep does."""
import json
import os
import subprocess

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


def run_native(cli, args):
    r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


def test_native_cli_arguments_and_errors(tmp_path, cli, toy_text):
    """Argument handling of the native driver mirrors sched.py: required
    flags, seed-list errors (same codes and messages), config files (flags
    win, bad documents are validation errors), unknown options."""
    gp = tmp_path / "g.json"
    gp.write_text(toy_text)
    cases = [
        (["sweep", "--seeds", "1..2"], 4, "error: --out is required"),
        (["sweep", "--out", str(tmp_path / "x.csv")], 4, "error: --seeds is required"),
        (["sweep", "--seeds", "5..4", "--out", "x"], 4, "error: seed range is empty: 5..4"),
        (["sweep", "--seeds", "0..1000000", "--out", "x"], 4, "error: seed range too large: 0..1000000"),
        (["sweep", "--seeds", ",,", "--out", "x"], 4, "error: no seeds in: ,,"),
        (["sweep", "--seeds", "1..2x", "--out", "x"], 4, "error: bad seed value: 2x"),
        (["sweep", "--seeds", "1", "--out", "x"], 4, "error: --graph is required"),
        (["sweep", "--seeds", "1", "--out", "x", "--graph", str(tmp_path / "none.json")], 5,
         "error: cannot read " + str(tmp_path / "none.json")),
        (["sweep", "--bogus", "1"], 4, "error: unknown option: --bogus"),
        (["bruteforce", "--seeds", "1"], 4, "error: unknown option: --seeds"),
        (["sweep", "--seeds", "1", "--out", "x", "--graph", str(gp), "--enforce", "maybe"], 4,
         "error: unknown enforcement: maybe"),
        (["sweep", "--seeds", "1", "--out", "x", "--graph", str(gp), "--oracle", "psychic"], 4,
         "error: unknown oracle source: psychic"),
    ]
    for args, code, msg in cases:
        rc, _, err = run_native(cli, args)
        assert (rc, err.strip()) == (code, msg), args
        if code == 4 and "--graph" not in args:  # the Python driver agrees
            assert sched.main(args) == code
    bad = tmp_path / "bad.json"
    bad.write_text("[1]")
    rc, _, err = run_native(cli, ["sweep", "--config", str(bad)])
    assert (rc, err.strip()) == (2, "error: config must be a JSON object")
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"seeds": "1..3", "out": str(tmp_path / "cfg.csv")}))
    rc, _, err = run_native(cli, ["sweep", "--config", str(cfg), "--seeds", "9..8"])
    assert (rc, err.strip()) == (4, "error: seed range is empty: 9..8")  # the flag won


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
def test_sweep_csv_matches_reference_loop(tmp_path, lib, ref, cli, algo, capsys):
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
        native = tmp_path / "n.csv"  # the native driver: same bytes, same summary line
        rc, stdout, err = run_native(cli, ["sweep", "--graph", str(gp), "--algo", algo, "--seeds", seeds,
                                           "--out", str(native)])
        assert rc == 0, err
        assert native.read_text() == want, name
        assert stdout.strip() == line


@pytest.mark.gpu
def test_bruteforce_driver(tmp_path, lib, ref, cli):
    text = lib.generate("layered", 3, 2, "1", 4).serialize()
    gp = tmp_path / "g.json"
    gp.write_text(text)
    out = tmp_path / "bf.json"
    assert sched.main(["bruteforce", "--graph", str(gp), "--out", str(out)], lib=lib) == 0
    g = ref.graph(text)
    assert out.read_text() == g.brute_force_text(g.declared(), policy(True, 0, 0.0), 8)
    assert os.path.getsize(out) > 0
    native = tmp_path / "bf_native.json"
    rc, stdout, err = run_native(cli, ["bruteforce", "--graph", str(gp), "--out", str(native)])
    assert rc == 0, err
    assert native.read_text() == out.read_text()
    res = json.loads(native.read_text())
    assert stdout.strip() == f"best m_us={res['makespan_us']} order={','.join(res['order'])}"
