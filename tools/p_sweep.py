"""Special-modulus size sweep: bootstrap precision/latency (config 3)
and the config-4 step at P = 11 x 60 bits vs P = 9 x 60 bits (= the widest
digit, 9 x 60-bit bootstrap primes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import c4_run  # noqa: E402

for sp in [int(a) for a in sys.argv[1:]] or [660, 540]:
    r = bench.run_c3_bootstrap(special=sp)
    print(json.dumps({"special_bits": sp, "c3": {k: r[k] for k in ("ms", "ms_eager", "precision_bits")}}), flush=True)
    c4 = c4_run.run(reps=2, verbose=False, special=sp)
    print(json.dumps({"special_bits": sp, "c4": {k: c4[k] for k in ("ms_per_step", "ms_per_step_eager_waves", "weights_max_abs_err_vs_sim", "velocities_max_abs_err_vs_sim")}}), flush=True)
