"""One-GPU projection of the 8-GPU strong-scaling run.

Only one GPU is available, so this times what one rank of a C4 / 8 run would
execute: its shard of the tree (plan(C4, 8): stage-2 subtrees, 2 per rank,
~9.9k nodes incl. the 4 replicated stage-1 rows) as the captured iteration
graph with the NCCL all-reduce of the replicated rows' partial sums inside it,
on a one-rank communicator (the all-reduce is then a local copy: the
8-GPU NVLink all-reduce of 16 x 256 doubles costs more, ~10-20 us, stated as a
range). Prints JSON: us per iteration of the shard graph (first and last
shard), the one-GPU C4 iteration, and the projected speed-up.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_10548_b200 import factor_step, shard  # noqa: E402
from paper_1904_10548_b200 import _native as nat  # noqa: E402
from paper_1904_10548_b200 import solver as S  # noqa: E402
from paper_1904_10548_b200.synthetic import config_instance  # noqa: E402


def us_per_iteration(ctx, iters=100, gamma=1 / 2e9):
    th = S.theta_sequence(iters + 5)
    be = S._beta_table(th)
    best = 1e30
    for _ in range(3):
        ctx.call("wmpc_apg_begin", float(gamma), iters + 5, nat.ptr(th), nat.ptr(be))
        ctx.call("wmpc_apg_run", 5)
        ms = nat.C.c_float(0.0)
        ctx.call("wmpc_apg_run_timed", iters, nat.C.byref(ms))
        best = min(best, ms.value / iters * 1e3)
    return best


def main():
    G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    inst = config_instance("C4")
    cache = factor_step(inst)
    ctx1 = cache._bind()
    S._upload_bounds(ctx1, inst)
    t1 = us_per_iteration(ctx1, 50)
    specs = shard.plan(inst, G)
    out = {"gpus": G, "shard_stage": int(specs[0].k) + 1, "one_gpu_us": t1, "one_gpu_path": nat.path_info(ctx1),
           "shards": []}
    for r in sorted({0, G - 1}):
        sp = dataclasses.replace(specs[r], rank=0, size=1)
        sv = shard.ShardedSolver(inst, specs=[sp], device_exchange=specs[r].k > 0)
        sh = sv.shards[0]
        S._upload_bounds(sh.ctx, sh.inst)
        t = us_per_iteration(sh.ctx)
        out["shards"].append({"rank": r, "nodes": int(sp.rows.size), "replicated_rows": int(sp.n_rep_global),
                              "us_per_iteration": t, "path": nat.path_info(sh.ctx)})
    ts = max(s["us_per_iteration"] for s in out["shards"])
    out["projected_speedup_1_rank_exchange"] = t1 / ts
    out["projected_speedup_with_nvlink_allreduce_10_20us"] = [t1 / (ts + 10.0), t1 / (ts + 20.0)]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
