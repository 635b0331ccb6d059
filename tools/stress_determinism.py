"""Repeat the device path on fixed inputs and count results that are not
bitwise identical to the first (races show up as sporadic mismatches).
usage: stress_determinism.py [n] [slices] [repeats] [host]
With "host" every repeat runs the pinned-host pipeline (H2D / compute / D2H
streams, small chunks) and compares it with the device-path result."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1704_08364_b200 import fourier_bp as F  # noqa: E402
from paper_1704_08364_b200 import phantom  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
host = len(sys.argv) > 4 and sys.argv[4] == "host"
plan = F.BstPlan(n, n)
x = phantom.ellipsoid_volume(S, n, n, device="cuda")
g = torch.Generator("cuda").manual_seed(3)
z = torch.randn(x.shape, device="cuda", generator=g)
inputs = [x, z, 2.0 * x - 0.5 * z]
ref = [F.fbp_volume(v, plan) for v in inputs]
bad = []
for r in range(reps):
    for k, v in enumerate(inputs):
        if host:
            hv = v.cpu().pin_memory()
            o = F.fbp_volume(hv, plan, devices=[0], chunk=3, batch=2).cuda()
        else:
            o = F.fbp_volume(v, plan)
        if not torch.equal(o, ref[k]):
            d = (o - ref[k]).abs()
            rows = torch.nonzero(d.amax(dim=2) > 0)
            bad.append({"rep": r, "input": k, "max_abs": d.max().item(),
                        "rel": (torch.linalg.norm(o - ref[k]) / torch.linalg.norm(ref[k])).item(),
                        "rows": rows[:8].tolist(), "n_rows": int(rows.shape[0])})
lin = (torch.linalg.norm(ref[2] - (2.0 * ref[0] - 0.5 * ref[1])) / torch.linalg.norm(ref[2])).item()
print(json.dumps({"n": n, "slices": S, "host": host, "repeats": reps, "calls": reps * 3, "mismatches": len(bad),
                  "linearity_first": lin, "detail": bad[:10]}))
