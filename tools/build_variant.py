"""Build an alternative libsp200 for A/B timing (selected with SP200_LIB).

    python tools/build_variant.py out.so -DSP200_PROFILE_KNOBS=1
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1006_3148_b200 import _build  # noqa: E402

out = sys.argv[1]
cmd = ["/usr/local/cuda/bin/nvcc"] + _build.NVCC_FLAGS + sys.argv[2:] + ["-o", out] + _build.sources()
subprocess.check_call(cmd)
print(out)
