"""e2e (pinned host in/out through fbp_volume) at several host chunk sizes,
2048^3 by default.  Prints one JSON line per chunk size."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1704_08364_b200 import fourier_bp as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
chunks = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [31, 16, 8, 4]
plan = F.BstPlan(n_theta=n, n_t=n)
host_in = torch.empty((n, n, n), dtype=torch.float32, pin_memory=True)
g = torch.Generator().manual_seed(0)
for s in range(0, n, 64):
    host_in[s:s + 64].uniform_(0, 1, generator=g)
host_out = torch.empty((n, n, n), dtype=torch.float32, pin_memory=True)
for c in chunks:
    F.fbp_volume(host_in, plan, out=host_out, devices=[0], chunk=c)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        F.fbp_volume(host_in, plan, out=host_out, devices=[0], chunk=c)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"n": n, "chunk": c, "s": [round(t, 4) for t in ts],
                      "GB_per_s_per_direction": round(n ** 3 * 4 / min(ts) / 1e9, 1)}), flush=True)
