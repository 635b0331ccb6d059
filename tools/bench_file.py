"""End-to-end from disk: write a synthetic frame-major TOMOVOL1 sinogram
volume (n^3, layout 0 = [angle][slice][det], as measured data is stored),
then time volio.reconstruct_file (pinned slab reads -> H2D -> fbp on the
frame-major slab -> D2H -> slice-major writer) and print one JSON line.

    python tools/bench_file.py [--size 1024] [--block 32] [--dir /tmp]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1704_08364_b200 import fourier_bp as F, phantom, volio as V  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--block", type=int, default=32)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    n = a.size
    src, dst = os.path.join(a.dir, f"sino_{n}.tomovol"), os.path.join(a.dir, f"recon_{n}.tomovol")
    hdr = V.VolumeHeader(V.LAYOUT_FRAMES, (n, n, n))
    with open(src, "wb") as f:  # frame-major payload, written slab by slab
        f.write(hdr.pack())
        f.truncate(V.HEADER_SIZE + hdr.payload_bytes)
        for s0 in range(0, n, 64):
            s1 = min(n, s0 + 64)
            slab = phantom.ellipsoid_volume(n, n, n, device="cuda", slices=(s0, s1)).cpu().numpy()  # [s][a][t]
            fr = slab.transpose(1, 0, 2)  # [a][s][t]
            for j in range(n):
                f.seek(V.HEADER_SIZE + 4 * (j * n * n + s0 * n))
                f.write(np.ascontiguousarray(fr[j]).tobytes())
        f.flush()
        os.fsync(f.fileno())
    plan = F.BstPlan(n, n)
    V.reconstruct_file(src, dst, plan, block=min(a.block, n))  # warm-up (plan, page cache)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    V.reconstruct_file(src, dst, plan, block=min(a.block, n))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"what": "TOMOVOL1 frame-major sinograms -> GPU fbp -> slice-major images (volio.reconstruct_file)",
                      "n": n, "block": a.block, "seconds": dt, "voxels_per_s": n ** 3 / dt,
                      "bytes_read": hdr.payload_bytes, "bytes_written": 4 * n ** 3,
                      "note": "second run: input likely in the page cache"}))
    os.remove(src)
    os.remove(dst)


if __name__ == "__main__":
    main()
