"""Device time of one rank's z-slab of the 2048^3 workload on one B200: the
slab a rank of an N-GPU strong-scaling run reconstructs (2048 / N slices),
timed like bench.py (device-resident input, CUDA events, warm-up, median of
5).  Since the slabs are independent (no collective), this is each rank's
expected device time at N GPUs on an NVSwitch node.

usage: python tools/slab_times.py [--size 2048]  (one JSON line per N)
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_08364_b200 import fourier_bp as F  # noqa: E402
from paper_1704_08364_b200 import phantom  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=2048)
a = ap.parse_args()
n = a.size
plan = F.BstPlan(n, n)
nat = F.native_plan(plan, F.FilterPlan(), False, 0)
batch = F.default_batch(plan)
ws = nat.new_workspace(batch)
full = phantom.ellipsoid_volume(n, n, n, device="cuda")
img = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
for N in (1, 2, 4, 8):
    S = n // N
    sino = full[:S]
    for _ in range(3):
        nat.run("fbp", sino, img, S, batch, ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nat.run("fbp", sino, img, S, batch, ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(json.dumps({"n_gpus": N, "slab_slices": S, "ms_per_slab": ms,
                      "expected_job_voxels_per_s": n ** 3 / (ms / 1e3)}), flush=True)
