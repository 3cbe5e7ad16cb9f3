"""SASS guard for the reference-exact kernels (CPU: cuobjdump on the built
library).  ptxas contracts a packed `mul.rn.f32x2` feeding an
`add.rn.f32x2` into one FFMA2 despite the `.rn` (scripts/micro/
f32x2_exact.cu), which drops one of the reference's roundings; the exact
kernels therefore keep every product that is later added in scalar `.rn`
ops.  This test fails if a packed multiply (FMUL2) appears in any kernel that
must reproduce the reference's float arithmetic bit for bit."""
import re
import shutil
import subprocess

import pytest

from paper_1509_04394_b200 import fuseplan

# kernels whose float arithmetic must be the reference's, op for op
EXACT = [r"k_chain_pairILi\d+ELb[01]ELb1E",  # exact frame-pair pipeline (+ F345 planes)
         r"k_chain_exact", r"k_gauss_grad_thr", r"k_gaussian_rows", r"k_gradient_rows",
         r"k_gray_iir", r"k_iir", r"k_rgba2gray", r"k_pointwise"]


def test_no_packed_multiply_in_exact_kernels():
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    import os
    if not os.path.exists(fuseplan.LIB_PATH):
        pytest.skip("library not built")
    sass = subprocess.run(["cuobjdump", "-sass", fuseplan.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    fn, seen, bad = None, set(), {}
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1) if any(re.search(p, m.group(1)) for p in EXACT) else None
            if fn:
                seen.add(fn)
            continue
        if fn and "FMUL2" in line:
            bad[fn] = bad.get(fn, 0) + 1
    assert len(seen) >= 10, f"exact kernels not found in the SASS ({len(seen)})"
    assert not bad, f"packed multiplies in exact kernels: {bad}"
