"""SASS invariants of the built library (CPU: cuobjdump only).

Bit-exact forward results need one rounding per operation (SURVEY.md §7 hard
part 1): no kernel on the message-passing path may contain a fused
multiply-add. nvcc runs with -fmad=false, but ptxas still contracts
mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (found in round 2), so the built code
is checked, not the flags.
"""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1910_10892_b200",
                   "libmrf_cuda.so")
PATH_KERNELS = re.compile(r"(fwd_|bwd_|sgm_|aggregate_kernel|dtheta_acc|reduce_gvacc|pack_)")


def test_no_fma_in_path_kernels():
    if not shutil.which("cuobjdump") or not os.path.exists(LIB):
        pytest.skip("cuobjdump or library missing")
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    bad, func, checked = [], None, 0
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            func = m.group(1)
            if PATH_KERNELS.search(func):
                checked += 1
            continue
        if func and PATH_KERNELS.search(func) and re.search(r"\bFFMA2?\b", ln):
            bad.append((func, ln.strip()[:80]))
    assert checked > 50, "no path kernels found in the SASS"
    assert not bad, f"fused multiply-adds on the path: {bad[:5]}"
