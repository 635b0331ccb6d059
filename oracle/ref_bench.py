"""Time the UNMODIFIED reference (tomoblocks) with its own benchmark harness.

MEASUREMENT INFRASTRUCTURE ONLY (like the rest of ``oracle/``): called by
``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm, never by the
product.  The package is installed into ``oracle/_ref/`` by
``oracle/build_ref.sh`` (a pip install of /root/reference/pkg; git-ignored,
shipped to the GPU box with the snapshot).

Method = the reference's ``cmd_bench`` cell (``cli.py:300-371``):
``cmd_phantom`` writes an analytic-ellipsoid TOMOVOL1 volume, then
``build_reconstruction_pipeline(ReconConfig(kernel="bst", normalize=False,
write=False, workers=W, block_size=q))`` + ``run_pipeline`` over
``block_descriptors`` with a discarding sink.  Every run builds a fresh
``BstPlan`` whose gridding tables (``fourier_bp.py:222-249``) are part of the
timed region, so each step times a run of K_a = W slices (one wave of the
W workers: plan tables, thread start-up, pipeline fill and drain) and one of
K_b = 3 W slices; the marginal per-slice time (t_b - t_a) / (K_b - K_a)
extrapolates the full S-slice volume as t_a + (S - K_a) * marginal.
"""

from __future__ import annotations

import argparse
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "tomoblocks"))


def _import():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from tomoblocks import cli, pipeline  # noqa: F401
    return cli, pipeline


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _phantom(cli, path: str, n: int, slices: int) -> None:
    args = cli._build_parser().parse_args(
        ["phantom", "--output", path, "--n", str(n), "--angles", str(n), "--slices", str(slices)])
    with open(os.devnull, "w") as null:
        old, sys.stdout = sys.stdout, null
        try:
            cli.cmd_phantom(args)
        finally:
            sys.stdout = old


def _run(cli, pipeline, path: str, workers: int, q: int) -> float:
    cfg = cli.ReconConfig(input_path=path, output_path=None, kernel="bst", block_size=q, workers=workers,
                          queue_capacity=2, normalize=False, write=False)
    plan = pipeline.build_reconstruction_pipeline(cfg)
    n_slices = plan.resources[0].header.n_slices
    t0 = time.perf_counter()
    try:
        pipeline.run_pipeline(plan, pipeline.block_descriptors(n_slices, q), lambda block: None)
    finally:
        plan.close_resources()
    return time.perf_counter() - t0


class RefBench:
    """Phantom files written once; ``step()`` times one (K_a, K_b) pair."""

    def __init__(self, n: int, workers: int | None = None, q: int = 1, waves: int = 3):
        self.cli, self.pipeline = _import()
        self.n, self.q = n, q
        self.workers = workers or os.cpu_count() or 1
        self.ka, self.kb = self.workers, waves * self.workers
        self.tmp = tempfile.TemporaryDirectory(prefix="tb-refbench-")
        self.pa = os.path.join(self.tmp.name, "a.tomovol")
        self.pb = os.path.join(self.tmp.name, "b.tomovol")
        _phantom(self.cli, self.pa, n, self.ka)
        _phantom(self.cli, self.pb, n, self.kb)

    def step(self, total_slices: int) -> dict:
        ta = _run(self.cli, self.pipeline, self.pa, self.workers, self.q)
        tb = _run(self.cli, self.pipeline, self.pb, self.workers, self.q)
        marginal = max((tb - ta) / (self.kb - self.ka), 1e-9)
        total = ta + max(total_slices - self.ka, 0) * marginal
        return {"t_a_s": ta, "t_b_s": tb, "marginal_s_per_slice": marginal, "volume_s": total,
                "voxels_per_s": total_slices * self.n * self.n / total}

    def describe(self, total_slices: int) -> str:
        return (f"tomoblocks (reference, unmodified, oracle/_ref) cmd_bench cell: build_reconstruction_pipeline"
                f"(kernel bst, normalize off, write off, workers {self.workers}, block_size {self.q}) + run_pipeline"
                f" on {self.n}^2 x {self.n}-angle phantoms of {self.ka} and {self.kb} slices; the {total_slices}-slice"
                f" volume extrapolated as t_a + (S - K_a)(t_b - t_a)/(K_b - K_a) (plan tables inside t_a)")

    def close(self):
        self.tmp.cleanup()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--workers", type=int, default=None)
    a = ap.parse_args()
    rb = RefBench(a.n, a.workers)
    print(rb.step(a.n), rb.describe(a.n))
    rb.close()


if __name__ == "__main__":
    main()
