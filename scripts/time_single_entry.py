"""Per-entry drop-in cost on config 5 (BA n=1e7): host-API entry_estimate
calls, one row each (the reference's usage pattern), with the staged-v cache
off (every call copies v and repacks it into the walk layout) and on (v
staged once).  Prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1904_12759_b200 as pb  # noqa: E402

cfg = pb.build_config(5)
m = pb.split(cfg.csr)
v = torch.from_numpy(cfg.v).pin_memory().numpy()
p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang, 3)
rows = np.random.default_rng(0).choice(cfg.csr.n, 64, replace=False)
out = {"workload": "cfg5 single-entry host calls", "W": cfg.walkers, "calls": len(rows)}
for mode in ("off", "on"):
    pb.set_v_cache(m, mode == "on")
    pb.invalidate_v(m)
    pb.entry_estimate(m, v, int(rows[0]), p)  # warm (and stage, when on)
    torch.cuda.synchronize()
    s0 = pb.v_stagings(m)
    t = time.perf_counter()
    vals = [pb.entry_estimate(m, v, int(i), p).value for i in rows]
    dt = (time.perf_counter() - t) / len(rows)
    out[f"cache_{mode}_ms_per_call"] = 1e3 * dt
    out[f"cache_{mode}_stagings"] = pb.v_stagings(m) - s0
    out[f"cache_{mode}_first_value"] = vals[0]
print(json.dumps(out))
