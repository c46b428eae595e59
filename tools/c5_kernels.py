"""Per-kernel breakdown of one steady training step through the layer code:
python tools/c5_kernels.py [c4|c5] [step]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import train_dropin  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
step = int(sys.argv[2]) if len(sys.argv) > 2 else 2
train_dropin.run(name, step, verbose=True, kernels_step=step)
