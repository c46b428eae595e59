"""Build A/B variants of the kernel library: python tools/ab_build.py NAME [-DFLAG ...]
-> paper_2506_19693_b200/_lib/variants/NAME/libckks_b200.so (load with CKB_LIB=...)."""
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import build as b  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(b.LIB_DIR, "variants", name, "libckks_b200.so")
b.build(out=out, defines=defines, verbose=True)
# the objects stay out of the gpurun snapshot (512 MiB cap): only the .so travels
shutil.rmtree(os.path.join(os.path.dirname(out), "obj"), ignore_errors=True)
