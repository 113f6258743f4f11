"""The player step compiled per treeplex (kr_jit.cu), checked without a GPU:
the generated CUDA C for the configs' trees compiles for sm_100a with the
library's flags, keeps every regret in a register (one `double rK` per
sequence), and follows the reference tree (one block per decision node, the
children summed in descending node order).  Bitwise agreement with the
generic kernels and the oracle is tests/test_gpu_jit_step.py."""
import os
import re
import shutil
import subprocess

import pytest

from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import jit_step_source

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def config3_tree():
    return H.turn_instances(nboards=1, factors=False)[0][0].treeplex(0)


def test_source_shape(config3_tree):
    t = config3_tree
    src = jit_step_source(t, 0)
    assert 'extern "C" __global__' in src and "kr_step" in src
    for k in range(t.n_seq):
        assert re.search(rf"\bdouble r{k} = Gh\[{k}\];", src)
    assert src.count("double nv") == len(t.parent)       # one node value per decision node
    assert "-fmad" not in src                              # contraction is a compile flag, not source
    # PRM+ matches R + d
    assert "w0 = " in jit_step_source(t, 2)


def test_children_in_descending_order(config3_tree):
    t = config3_tree
    src = jit_step_source(t, 0)
    for line in src.splitlines():
        kids = [int(m) for m in re.findall(r"cs \+= nv(\d+);", line)]
        assert kids == sorted(kids, reverse=True)


@pytest.mark.skipif(not os.path.exists(NVCC) and not shutil.which("nvcc"), reason="nvcc absent")
@pytest.mark.parametrize("rule", [0, 2])
def test_compiles_for_sm100a_without_local_arrays(config3_tree, tmp_path, rule):
    src = tmp_path / "kr_step.cu"
    src.write_text(jit_step_source(config3_tree, rule))
    r = subprocess.run([NVCC, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-Xptxas", "-v",
                        "-o", str(tmp_path / "k.cubin"), str(src)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    regs = int(re.search(r"Used (\d+) registers", r.stderr).group(1))
    assert regs <= 168   # three 128-hand CTAs per SM


@pytest.mark.skipif(not os.path.exists(NVCC) and not shutil.which("nvcc"), reason="nvcc absent")
def test_warp_group_form_compiles(config3_tree, tmp_path, monkeypatch):
    """The single-board form (the tree split over four warp groups, node
    values exchanged through shared memory) compiles for sm_100a without
    spills, and every group section ends on the same barrier sequence."""
    monkeypatch.setenv("KR_JIT_SOURCE_GROUPS", "4")
    src = jit_step_source(config3_tree, 0)
    assert "#define NT (4 * HB)" in src
    sections = src.split("if (grp == ")
    counts = {sec.count("bar_all();") for sec in sections[1:]}
    assert len(sections) == 5 and len(counts) == 1, counts   # groups 0..3, same barrier count each
    f = tmp_path / "kr_step_g4.cu"
    f.write_text(src)
    r = subprocess.run([NVCC, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-Xptxas", "-v",
                        "-o", str(tmp_path / "g4.cubin"), str(f)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert " 0 bytes spill stores" in r.stderr
