"""Build paper_2108_04791_b200/libisprime_checked.so: the same sources with
-DISP_CHECKS=1 (device-side bounds checks on the queues, the sort, the dense
kernel's indices; kernels.cuh ISP_CHECK).  Load it with ISPRIME_LIB=<path>.
compute-sanitizer is closed on the GPU pool; this build stands in for its
out-of-bounds reports (tests/test_gpu_checked.py)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_04791_b200 import _build  # noqa: E402

OUT = os.path.join(ROOT, "paper_2108_04791_b200", "libisprime_checked.so")


def build():
    cmd = [os.environ.get("NVCC", "nvcc"), *_build.NVCC_FLAGS, "-DISP_CHECKS=1", "-o", OUT,
           os.path.join(_build.CSRC, "isprime.cu")]
    subprocess.run(cmd, check=True, capture_output=True)
    return OUT


if __name__ == "__main__":
    print(build())
