"""The C++ CLI (tools/krb200_cli.cpp) over both C ABIs, mirroring the
reference's `kronriver sparsify` / `solve` session in README.md:73-82 and the
pipeline checks of tools/cli_pipeline.sh."""
import json
import os
import subprocess

import pytest

from paper_2112_03804_b200 import build

CLI = os.path.join(build.LIBDIR, "krb200")


@pytest.fixture(scope="module")
def twenty_card(tmp_path_factory, instance_fixtures):
    build.build_cli()
    d = tmp_path_factory.mktemp("cli")
    path = d / "twenty_card.json"
    path.write_text(json.dumps(instance_fixtures["twenty_card"], indent=2))
    return d, str(path)


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


def test_sparsify_prints_the_readme_rows(twenty_card):
    d, inst = twenty_card
    r = run("sparsify", "--instance", inst, "--technique", "b", "--out", str(d / "bundle"))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    fields = lines[1].split()
    assert fields[0] == "twenty_card" and fields[1] == "152916" and fields[2] == "55760" and fields[4] == "2.74"
    assert lines[2] == "factors: ahat=28350 u=2205 m=1649 v=23556 k=835 technique=b postprocessed=1"
    # sparsify twice -> identical bundles (cli_pipeline.sh:12-14)
    assert run("sparsify", "--instance", inst, "--out", str(d / "bundle2")).returncode == 0
    for n in ("header.json", "ahat.mtx", "u.mtx", "m.mtx", "v.mtx"):
        assert (d / "bundle" / n).read_bytes() == (d / "bundle2" / n).read_bytes()


def test_errors_exit_two(twenty_card):
    d, _ = twenty_card
    r = run("sparsify", "--instance", str(d / "missing.json"))
    assert r.returncode == 2 and r.stderr.startswith("error code=IO")


@pytest.mark.gpu
def test_solve_reproduces_the_readme_line(twenty_card):
    """README.md:81-82: `solve --bundle bundle --iters 600` prints
    exploitability=0.000189332132512 gradient_flops=67228200."""
    d, inst = twenty_card
    assert run("sparsify", "--instance", inst, "--technique", "b", "--out", str(d / "b3")).returncode == 0
    r = run("solve", "--instance", inst, "--bundle", str(d / "b3"), "--iters", "600", "--out", str(d / "run"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("solve: iterations=600 exploitability=0.000189332132512 gradient_flops=67228200")
    # bundle solve == in-memory solve (cli_pipeline.sh:16-27)
    r2 = run("solve", "--instance", inst, "--technique", "b", "--iters", "600", "--out", str(d / "run2"))
    assert r2.stdout.split()[1:4] == r.stdout.split()[1:4]
    assert (d / "run" / "trace.csv").read_text() == (d / "run2" / "trace.csv").read_text()


def test_bad_engine_or_rule_exit_two(twenty_card):
    d, inst = twenty_card
    r = run("solve", "--instance", inst, "--engine", "dense", "--iters", "5", "--out", str(d / "bad"))
    assert r.returncode == 2 and "INVALID_INPUT" in r.stderr
    r = run("solve", "--instance", inst, "--rule", "mccfr", "--iters", "5", "--out", str(d / "bad"))
    assert r.returncode == 2 and "INVALID_INPUT" in r.stderr


@pytest.mark.gpu
def test_solve_implicit_engine_and_cfr_plus(twenty_card):
    """--engine implicit reproduces the README solve to the printed 12 digits
    within 1e-7 relative; --rule cfr+ runs BASELINE config 1's 1000 CFR+ iterations."""
    d, inst = twenty_card
    r = run("solve", "--instance", inst, "--engine", "implicit", "--iters", "600", "--out", str(d / "imp"))
    assert r.returncode == 0, r.stderr
    expl = float(r.stdout.split("exploitability=")[1].split()[0])
    assert abs(expl - 0.000189332132512) <= 1e-7 * 0.000189332132512
    r = run("solve", "--instance", inst, "--rule", "cfr+", "--iters", "1000", "--out", str(d / "cfrp"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("solve: iterations=1000 ") and "rule=cfr+" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["kfactored", "factored", "implicit"])
def test_solve_turn_matches_the_library_solver(engine):
    """krb200 solve-turn: config 3's boards sharded over --gpus N (here 1: the
    box has one GPU) through the C++ driver; the printed trace equals the
    Python-driven solve of the same boards bit for bit."""
    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import host as H
    from paper_2112_03804_b200.solver import CudaSolver, DcfrParams
    build.build_cli()
    r = run("solve-turn", "--boards", "4", "--iters", "40", "--checkpoint-every", "20", "--gpus", "1",
            "--engine", engine)
    assert r.returncode == 0, r.stderr
    got = [float(ln.split("exploitability=")[1]) for ln in r.stdout.splitlines() if ln.startswith("checkpoint")]
    boards = H.turn_instances(nboards=4, factors=engine == "factored")
    insts = [i for i, _ in boards]
    eng = (CudaEngine([f for _, f in boards]) if engine == "factored" else
           CudaEngine.kfactored(insts) if engine == "kfactored" else CudaEngine.kron(insts))
    i0 = insts[0]
    ref = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts],
                     i0.pot).run(DcfrParams(max_iters=40, checkpoint_every=20))
    assert got == list(ref.trace_expl)
    assert "gpus=1" in r.stdout and f"engine={engine}" in r.stdout
    bad = run("solve-turn", "--gpus", "64")
    assert bad.returncode == 2 and "INVALID_INPUT" in bad.stderr
