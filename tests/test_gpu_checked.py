"""The bounds-checked build (KR_CHECKED, lib/libkrcuda_checked.so): the
stand-in for compute-sanitizer, which this pool's GPUs do not take
(profiles/r02/compute_sanitizer_refused.log).  Every device allocation of the
library gets poisoned guard zones, verified when it is freed and by
kr_checked_verify after every GPU test (conftest.py); device index checks trap
with the file and line.  These tests show that both mechanisms fire.  The
whole GPU suite is run under this build with KR_CUDA_LIB_VARIANT=checked."""
import os
import subprocess
import sys

import pytest

from paper_2112_03804_b200 import build as B

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys
sys.path.insert(0, {root!r})
os.environ["KR_CUDA_LIB_VARIANT"] = "checked"
from paper_2112_03804_b200 import _native as N
print("RESULT", N.cuda().kr_checked_selftest({mode}), flush=True)
'''


def run_child(mode):
    if not os.path.exists(os.path.join(B.LIBDIR, "libkrcuda_checked.so")):
        B.build_cuda_variant("checked", ["KR_CHECKED"])
    p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, mode=mode)], capture_output=True, text=True,
                       timeout=300)
    return p.stdout + p.stderr


def test_guard_zone_overwrite_is_found():
    out = run_child(0)
    assert "RESULT 1" in out, out


def test_device_index_check_traps():
    out = run_child(1)
    assert "KR_CHECKED" in out and "i < n" in out, out
    res = [ln for ln in out.splitlines() if ln.startswith("RESULT")]
    assert res and int(res[0].split()[1]) < 0, out
