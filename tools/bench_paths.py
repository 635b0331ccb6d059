"""Per-slice device time of the BST paths other than the benchmark's
half-turn bilinear one, at n_t = V = n = 2048 (CUDA events around
fbp_volume on device-resident input, after warm-up):

  half_bilinear   the benchmark path (K2_TEX)
  half_nearest    interp="nearest" (K2_ANY: lattice_value per node)
  full_bilinear   full-turn input, 2V rows (K2_ANY + Hermitian average)
  half_notex      TB_NOTEX=1 plain-load gathers (K2_PLAIN), separate process

usage: python tools/bench_paths.py [--slices 62] [--size 2048]  (one JSON line per path)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(path, size, slices, reps=3):
    import torch
    from paper_1704_08364_b200 import fourier_bp as F

    full = path == "full_bilinear"
    interp = "nearest" if path == "half_nearest" else "bilinear"
    plan = F.BstPlan(size, size, interp=interp)
    rows = 2 * size if full else size
    g = torch.Generator(device="cuda").manual_seed(0)
    sino = torch.randn((slices, rows, size), device="cuda", dtype=torch.float32, generator=g)
    out = torch.empty((slices, size, size), device="cuda", dtype=torch.float32)
    F.fbp_volume(sino, plan, full_turn=full, out=out)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.fbp_volume(sino, plan, full_turn=full, out=out, check=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return {"path": path, "size": size, "slices": slices, "ms_per_slice": best / slices,
            "ms_per_volume_equiv": best / slices * size}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", type=int, default=62)
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--path", default=None)
    a = ap.parse_args()
    if a.path:
        print(json.dumps(run(a.path, a.size, a.slices)), flush=True)
    else:
        for p in ["half_bilinear", "half_nearest", "full_bilinear"]:
            print(json.dumps(run(p, a.size, a.slices)), flush=True)
        env = dict(os.environ, TB_NOTEX="1")
        r = subprocess.run([sys.executable, __file__, "--path", "half_bilinear", "--slices", str(a.slices),
                            "--size", str(a.size)], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"error": r.stderr[-300:]})
        d = json.loads(line)
        d["path"] = "half_notex"
        print(json.dumps(d), flush=True)
