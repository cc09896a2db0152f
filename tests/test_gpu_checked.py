"""The pipeline under the CHECKED build (libisprime_checked.so, -DISP_CHECKS=1:
device-side bounds checks on queue segments, the sort's output positions,
the staged appends of the witness kernels, the indices they read, and the
dense kernel's element / segment indices).  A failed check turns the call
into ISP_ECUDA.  compute-sanitizer is closed on the GPU pool; this is the
stand-in for its out-of-bounds reports.  Each workload runs in a subprocess
with ISPRIME_LIB pointing at the checked library and compares with the oracle
(tools/sanitize.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2108_04791_b200", "libisprime_checked.so")


@pytest.mark.parametrize("workload", ["dense", "pipeline", "c3", "small", "chunks", "full"])
def test_checked_build(workload):
    sys.path.insert(0, ROOT)
    from paper_2108_04791_b200 import _build
    if not os.path.exists(CHECKED) or any(os.path.getmtime(src) > os.path.getmtime(CHECKED)
                                          for src in _build._sources()):
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import build_checked
        build_checked.build()  # absent or older than the sources it checks
    env = dict(os.environ, ISPRIME_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py"), workload], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"sanitize workload ok {workload}" in r.stdout
