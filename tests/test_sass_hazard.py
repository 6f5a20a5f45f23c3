"""The built library carries no SASS memory instruction whose L2-policy descriptor register
is never written in its kernel (the pattern behind the f64 backward fault found with
compute-sanitizer, "A code-generation hazard"). CPU-only: cuobjdump + nvdisasm."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_29155_b200", "libdiffmpc.so")


@pytest.mark.skipif(not os.path.exists(LIB) or not shutil.which("nvdisasm") or not shutil.which("cuobjdump"),
                    reason="needs the built library and the CUDA binary utilities")
def test_no_unwritten_descriptor_registers():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_desc_check.py"), LIB],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert " 0 instructions" in r.stdout
