"""Host-side cProfile of one steady config-4 step through the layer code
(deferred mode): python tools/c4_hostprof.py [config] [step]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import train_dropin  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
step = int(sys.argv[2]) if len(sys.argv) > 2 else 3
train_dropin.run(name, step, verbose=True, profile_step=step)
