"""Print the headline numbers of a bench.py log (the last JSON line)."""
import json
import sys

line = [ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1]
d = json.loads(line)
print("c2 %.1f GB/s  hmult %.1f us/ct  hrot %.1f us/ct  stages %s" % (
    d["value"], d["hmult_us_per_ct"], d["hrot_us_per_ct"],
    {k: round(v, 2) for k, v in d["stages_ms"].items()}))
print("kernels", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
print("roofline frac %.3f alu %.3f | e2e %.1f | c1 %.2f ms | c3 %.1f ms | c4 %.0f ms | c5 %.0f ms | clocks %s" % (
    d["roofline"]["frac"], d["roofline"]["alu"]["frac"], d.get("e2e", {}).get("value", float("nan")),
    d.get("c1_train", {}).get("ms_per_step", float("nan")), d.get("c3_bootstrap", {}).get("ms", float("nan")),
    d.get("c4_train", {}).get("ms_per_step", float("nan")),
    d.get("c5_train", {}).get("ms_per_step", float("nan")), d.get("clocks")))
for k in ("c4_train", "c5_train"):
    if k in d:
        print(k, {kk: (round(v, 6) if isinstance(v, float) else v) for kk, v in d[k].items()
                  if kk in ("ms_per_step", "step1_ms", "steady_step_ms", "weights_max_abs_err_vs_sim",
                            "step2_weights_max_abs_err_vs_sim", "step2_velocities_max_abs_err_vs_sim")})
