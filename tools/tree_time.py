"""us per APG iteration of the default / forced kernel paths on a given branching:
tree_time.py "4,4,4,4,2,2" [ENV=V,...]  (graph replay, CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for kv in (sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] else []):
    k, v = kv.split("="); os.environ[k] = v
from paper_1904_10548_b200 import factor_step
from paper_1904_10548_b200 import _native as nat
from paper_1904_10548_b200 import solver as S
from paper_1904_10548_b200.synthetic import barcelona_instance
br = [int(x) for x in sys.argv[1].split(",")]
inst = barcelona_instance(br)
cache = factor_step(inst)
ctx = cache._bind()
S._upload_bounds(ctx, inst)
it = 200
th = S.theta_sequence(it + 5); be = S._beta_table(th)
best = 1e9
for _ in range(3):
    ctx.call("wmpc_apg_begin", 1 / 2e9, it + 5, nat.ptr(th), nat.ptr(be))
    ctx.call("wmpc_apg_run", 5)
    ms = nat.C.c_float(0.0)
    ctx.call("wmpc_apg_run_timed", it, nat.C.byref(ms))
    best = min(best, ms.value / it * 1e3)
info = nat.path_info(ctx)
print(json.dumps({"branching": br, "env": sys.argv[2] if len(sys.argv) > 2 else "", "nodes": inst.n_nonroot,
                  "us": round(best, 2), "fused_dp": info["fused_dp"], "dp_segm": info["dp_segm"],
                  "nchain": info["nchain"]}))
