"""Benchmark: 2048^3 BST filtered backprojection (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--size 2048] [--impl ours|reference]

One "step" reconstructs the whole synthetic 2048^3 sinogram volume
(V = n_t = 2048 angles x detector samples per slice, 2048 slices, n = 2048
output) -- configs[3] of BASELINE.json, which fits one B200.  Under torchrun
(N > 1) the volume is slab-sharded over the ranks (contiguous z-slabs, no
data-path collective; a barrier and a MAX all-reduce of the timings only):
total work is fixed, so scaling is "strong".

value       voxels/s of the whole job, inputs resident in HBM, CUDA events on
            the launching stream around K steps, max over ranks.
e2e         the same metric through the public API `fbp_volume` with pinned
            HOST input/output: H2D, compute and D2H inside the timed region.
roofline    dominant kernel: algorithmic bytes per launch (SURVEY.md 8d:
            K1 = 4 V n_t + 8 V H, K2 = 8 V H + 8 (H+1) n, K3 = 8 (H+1) n + 4 n^2
            per slice) / its average CUDA-event launch time, against the
            measured HBM copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline  the CPU oracle restatement of the reference (oracle/bst_oracle.py,
            kind "port") on a bounded slice sample using all host cores.

`--impl reference` times that CPU reference restatement alone on the host
(rank 0 only) and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2048^3 volume recon seconds & voxels/s at 1/2/4/8 B200; % HBM roofline"
UNIT = "voxels/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--size", type=int, default=2048, help="N for the N^3 workload (V = n_t = n = N)")
    ap.add_argument("--batch", type=int, default=None, help="slices per launch group")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-slices", type=int, default=None)
    ap.add_argument("--no-ss", action="store_true", help="skip the slant-stack comparator sample")
    ap.add_argument("--no-counts", action="store_true", help="skip the fused-normalisation counts step")
    ap.add_argument("--ss-slices", type=int, default=8)
    ap.add_argument("--ref-budget-s", type=float, default=240.0,
                    help="--impl reference: wall-clock bound of its warm-up + timed steps (0 = run all)")
    return ap.parse_args()


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _workload(n):
    return {"workload": f"{n}^3 BST FBP: {n} slices x {n} angles x {n} detector -> {n}^3 image, fp32",
            "n_slices": n, "n_angles": n, "n_t": n, "output_n": n}


def _algorithmic_bytes(V, n_t, L, n):
    H = L // 2
    k1 = 4 * V * n_t + 8 * V * H
    k2 = 8 * V * H + 8 * (H + 1) * n
    k3 = 8 * (H + 1) * n + 4 * n * n
    return {"k1_radial": k1, "k2_columns": k2, "k3_rows": k3, "total": k1 + k2 + k3}


# ---------------------------------------------------------------------------
# CPU reference (oracle port) timing
# ---------------------------------------------------------------------------

def _cpu_sample(n, slices, threads):
    """Time the oracle restatement of the reference on `slices` slices of the
    n^3 workload with a `threads`-wide pool (the reference pipeline's
    backproject-stage workers); returns (seconds, voxels/s)."""
    import numpy as np
    from oracle import bst_oracle as O
    plan = O.OraclePlan(n, n)
    first = n // 2 - slices // 2
    vol = O.ellipsoid_volume_sinogram(n, n, n, slices=(first, first + slices))
    vol = vol.astype(np.float32).astype(np.float64)
    O.fbp(vol[0], plan)  # warm caches / allocator outside the clock
    t0 = time.perf_counter()
    O.fbp_volume(vol, plan, workers=threads)
    dt = time.perf_counter() - t0
    return dt, slices * n * n / dt


def _cpu_reference(n, steps, warmup, threads, budget_s=None):
    """The reference's own CPU path on this host: the unmodified tomoblocks
    pipeline (oracle/_ref, oracle/ref_bench.py) when installed, else the
    oracle port.  Returns (voxels/s median, kind, sample, detail).

    ``budget_s`` bounds the wall clock of the warm-up plus timed steps (each
    step is a (K_a, K_b) pair of pipeline runs, ~20 s at 2048 on 16 threads):
    steps stop once the next one would overrun it (the first requested
    warm-up step and one timed step always run); ``detail`` records how many
    ran."""
    from oracle import ref_bench
    if ref_bench.available():
        rb = ref_bench.RefBench(n, threads)
        t0 = time.perf_counter()
        done_w, runs = 0, []
        try:
            for _ in range(warmup):
                t1 = time.perf_counter()
                rb.step(n)
                done_w += 1
                if budget_s and (time.perf_counter() - t0) + (time.perf_counter() - t1) * (max(1, steps) + 1) > budget_s:
                    break  # keep the budget for the timed steps
            for _ in range(max(1, steps)):
                t1 = time.perf_counter()
                runs.append(rb.step(n))
                if budget_s and (time.perf_counter() - t0) + (time.perf_counter() - t1) > budget_s:
                    break
        finally:
            rb.close()
        value = statistics.median(r["voxels_per_s"] for r in runs)
        for r in runs:
            r["warmup_steps_run"] = done_w
        return value, "reference", rb.describe(n), runs
    slices = max(threads, 4)
    for _ in range(warmup):
        _cpu_sample(n, min(slices, threads), threads)
    rates = [_cpu_sample(n, slices, threads)[1] for _ in range(max(1, steps))]
    sample = f"{slices} of {n} slices of the {n}^3 workload per step (oracle fbp_volume, {threads} threads), extrapolated"
    return statistics.median(rates), "port", sample, None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref_bench
    n = args.size
    threads = os.cpu_count() or 1
    value, kind, sample, runs = _cpu_reference(n, args.steps, args.warmup, threads, args.ref_budget_s)
    ran = len(runs) if runs else args.steps
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": ran, "warmup": runs[0]["warmup_steps_run"] if runs else args.warmup,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 * (n ** 3) / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic ellipsoid phantom)",
        "config": _workload(n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "cpu": ref_bench.cpu_model(), "runs": runs},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------

def _transfer_lines(torch, host_in, host_out, dev, bytes_per_dir, e2e_s):
    """H2D alone, D2H alone and both at once (pinned, 256 MiB copies, 4 GiB
    per direction) on the e2e buffers: the PCIe floor the e2e number sits on."""
    chunk = 64 << 20  # floats = 256 MiB
    nchunk = 16
    hi, ho = host_in.view(-1), host_out.view(-1)
    nchunk = min(nchunk, hi.numel() // chunk)
    dbuf = torch.empty(2 * chunk, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def run(h2d, d2h):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(nchunk):
            if h2d:
                with torch.cuda.stream(s1):
                    dbuf[:chunk].copy_(hi[i * chunk:(i + 1) * chunk], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    ho[i * chunk:(i + 1) * chunk].copy_(dbuf[chunk:], non_blocking=True)
        torch.cuda.synchronize()
        return nchunk * chunk * 4 / (time.perf_counter() - t0) / 1e9

    if nchunk == 0:
        return None
    run(True, True)
    h2d, d2h, both = run(True, False), run(False, True), run(True, True)
    floor = bytes_per_dir / (both * 1e9)
    return {"h2d_GBps": h2d, "d2h_GBps": d2h, "concurrent_GBps_per_direction": both,
            "pcie_floor_s": floor, "e2e_frac_of_pcie_floor": floor / e2e_s}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200 import phantom, slabs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TB_BENCH_BACKEND=gloo: ranks may share a GPU (exercises the multi-rank
    # path on one device; the timing reductions then run on host tensors)
    backend = os.environ.get("TB_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return slabs.max_over_ranks(x, device=dev if backend == "nccl" else None)

    n = args.size
    plan = F.BstPlan(n, n)
    b, e = slabs.rank_slab(n, world, rank)
    S = e - b
    batch = args.batch or F.default_batch(plan)

    # synthetic input: per-slice analytic ellipsoid sinogram of this rank's slab
    sino = phantom.ellipsoid_volume(n, n, n, device=dev, chunk=32, slices=(b, e))
    img = torch.empty((S, n, n), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    tp = time.perf_counter()
    nat = F.native_plan(plan, F.FilterPlan(), False, local)  # host tables + device gridding table
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - tp) * 1e3
    ws = nat.new_workspace(batch)
    stream = torch.cuda.current_stream(dev)

    def step():
        nat.run("fbp", sino, img, S, batch, ws, stream)

    nat.reset_status(ws)
    for _ in range(args.warmup):
        step()
    nat.read_status(ws)

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one event between consecutive steps as well (per-step median, SURVEY
    # §8d); recording an event does not perturb the stream
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
    ev0.record(stream)
    for i in range(args.steps):
        step()
        if i < args.steps - 1:
            marks[i].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    bounds = [ev0] + marks + [ev1]
    per_step = [max_over_ranks(bounds[i].elapsed_time(bounds[i + 1])) for i in range(args.steps)]
    step_stats = {"median": statistics.median(per_step), "min": min(per_step), "max": max(per_step)}
    value = (n ** 3) / (ms_step / 1e3)

    # per-kernel device times on the same workload (one extra profiled step)
    torch.cuda.synchronize()
    stage = nat.run_profiled(sino, img, S, batch, ws, stream)
    launches = {"k1_radial": math.ceil(S / batch), "k1b_common": math.ceil(S / batch),
                "k2_columns": math.ceil(S / batch), "k3_rows": math.ceil(S / batch)}
    alg = _algorithmic_bytes(n, n, plan.radial_samples, n)
    dom = max(("k1_radial", "k2_columns", "k3_rows"), key=lambda k: stage[k])
    per_launch_ms = stage[dom] / launches[dom]
    slices_per_launch = S / launches[dom]
    achieved = alg[dom] * slices_per_launch / (per_launch_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    traffic = None
    issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("size") == n and dom in tr.get("kernels", {}):
            traffic = tr["kernels"][dom]["dram_bytes_per_slice"] * slices_per_launch
        # the path is bound by instruction issue, not HBM: every SM issues at
        # most 4 warp instructions per clock, so the ncu-counted warp
        # instructions per slice set a floor on the step time
        if tr.get("size") == n:
            wi = sum(k.get("warp_inst_per_slice", 0.0) for k in tr["kernels"].values()) * S
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            mhz = (clk or {}).get("sm_mhz") or 1965.0
            floor_ms = wi / (sms * 4 * mhz * 1e6) * 1e3
            issue = {"bound": "issue", "warp_inst_per_step": wi, "floor_ms": floor_ms,
                     "frac": floor_ms / ms_step, "source": tr.get("source"),
                     # FP32 (FMA pipe) utilisation per kernel: the SURVEY 8d co-bound
                     "fp32_pipe_pct": {k: v.get("fp32_pipe_pct") for k, v in tr["kernels"].items()}}
    except Exception:
        pass
    nat.read_status(ws)

    # the same volume as raw transmission counts with the reference pipeline's
    # normalize stage fused into K1 (tb_fbp_counts; flat 2, dark 0 frames)
    counts_path = None
    if not args.no_counts:
        nat.run_counts_const(sino, 2.0, 0.0, 1e-6, img, S, batch, ws, stream)  # warm-up
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        nat.run_counts_const(sino, 2.0, 0.0, 1e-6, img, S, batch, ws, stream)
        c1.record(stream)
        torch.cuda.synchronize()
        cms = max_over_ranks(c0.elapsed_time(c1))
        counts_path = {"what": "fbp of transmission counts with the pipeline's constant i0/dark frames, "
                               "normalize fused into K1 (tb_fbp_counts_const)",
                       "ms_per_step": cms, "voxels_per_s": (n ** 3) / (cms / 1e3),
                       "overhead_vs_line_integrals": cms / ms_step - 1.0}
        nat.read_status(ws)

    # the reference pipeline's center ("auto") and rings (window 9) stages on
    # the device, on a bounded slab sample: fused into K1's row load through
    # the public fbp_volume (tb_pre_params + tb_fbp_pre), and as separate
    # device passes (preprocess_volume) followed by the fbp
    pre_path = None
    if not args.no_counts and S > 0:
        from paper_1704_08364_b200.preprocess import CenteringError, preprocess_volume
        k = min(S, 64)
        m0 = max(0, S // 2 - k // 2)  # central slices of this rank's slab
        samp = sino[m0:m0 + k]
        try:
            outk = img[:k]
            F.fbp_volume(samp, plan, center="auto", rings=9, out=outk, batch=batch)  # warm-up
            preprocess_volume(samp, plan, center="auto", rings=9)
            torch.cuda.synchronize()
            p0, p1, p2, p3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            p0.record(stream)
            F.fbp_volume(samp, plan, center="auto", rings=9, out=outk, batch=batch, check=False)
            p1.record(stream)
            pre = preprocess_volume(samp, plan, center="auto", rings=9)
            p2.record(stream)
            nat.run("fbp", pre, img, k, batch, ws, stream)
            p3.record(stream)
            torch.cuda.synchronize()
            pre_path = {"what": "center (estimate) + rings (window 9) stages on the device, then fbp",
                        "slices_sampled": k,
                        "fused_ms_per_slice": p0.elapsed_time(p1) / k,
                        "separate_passes_ms_per_slice": p1.elapsed_time(p3) / k,
                        "preprocess_ms_per_slice": p1.elapsed_time(p2) / k,
                        "fbp_ms_per_slice": p2.elapsed_time(p3) / k}
            nat.read_status(ws)
            del pre
        except CenteringError as exc:  # a slab outside the phantom has no centre to find
            pre_path = {"skipped": f"CenteringError on this rank's slab: {exc}"}

    # the forward projector (K6, fp64 rays) on a one-slice
    # sample of this rank's reconstructions, back onto the n x n sinogram grid
    fwd = None
    if not args.no_ss and S > 0:
        one = torch.empty((1, n, n), dtype=torch.float32, device=dev)
        nat.forward(img[:1], one, 1, 0.5, False, stream)  # warm-up
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        nat.forward(img[:1], one, 1, 0.5, False, stream)
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1)
        fwd = {"kernel": "k6_forward_tex (projector.forward_project, step 0.5, bilinear, TLD4)", "slices_sampled": 1,
               "ms_per_slice": fms, "ray_samples_per_s": n * n * math.ceil(2 * math.sqrt(2) * n) / (fms / 1e3)}
        del one

    # BASELINE configs[4]: the brute-force O(N^3) slant-stack backprojection
    # (fbp kernel "ss", projector.py:126-158) on the same inputs, timed on a
    # bounded sample of this rank's slices (device-resident, CUDA events)
    ss = None
    if not args.no_ss and S > 0:
        k = min(S, args.ss_slices)
        nat.run("fbp_ss", sino, img, k, batch, ws, stream)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nat.run("fbp_ss", sino, img, k, batch, ws, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ss_ms = e0.elapsed_time(e1) / k
        ss = {"kernel": "k5_slant (fbp kernel='ss')", "slices_sampled": k, "ms_per_slice": ss_ms,
              "voxels_per_s": n * n / (ss_ms / 1e3), "bst_ms_per_slice": ms_step / S,
              "bst_speedup": ss_ms / (ms_step / S)}
        nat.read_status(ws)

    # the BST paths the benchmark shape does not take (nearest interpolation:
    # K2_ANY; full-turn input, 2V rows: K2_TEXF), device-resident through the
    # public fbp_volume on a bounded sample of slices (any data: timing only)
    paths = None
    if not args.no_ss and S > 0:
        k = min(S, 31)
        paths = {}
        for name, interp, full in (("half_nearest", "nearest", False), ("full_turn_bilinear", "bilinear", True)):
            pl = F.BstPlan(n, n, interp=interp)
            src = torch.cat([sino[:k], sino[:k].flip(2)], dim=1).contiguous() if full else sino[:k]
            o = torch.empty((k, n, n), dtype=torch.float32, device=dev)
            with torch.cuda.stream(stream):
                F.fbp_volume(src, pl, full_turn=full, out=o)  # warm-up (plan tables, textures)
                torch.cuda.synchronize()
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                p0.record(stream)
                F.fbp_volume(src, pl, full_turn=full, out=o, check=False)
                p1.record(stream)
            torch.cuda.synchronize()
            paths[name] = {"slices_sampled": k, "ms_per_slice": p0.elapsed_time(p1) / k,
                           "vs_benchmark_path": p0.elapsed_time(p1) / k / (ms_step / S)}
            del src, o, pl

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty((S, n, n), dtype=torch.float32, pin_memory=True)
        host_in.copy_(sino)
        host_out = torch.empty((S, n, n), dtype=torch.float32, pin_memory=True)
        del img
        torch.cuda.empty_cache()
        F.fbp_volume(host_in, plan, out=host_out, devices=[local], batch=batch)  # warm-up
        k = args.e2e_steps or max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            F.fbp_volume(host_in, plan, out=host_out, devices=[local], batch=batch)
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / k)
        e2e = {"value": (n ** 3) / e2e_s, "unit": UNIT, "s_per_step": e2e_s,
               "h2d_bytes_per_step": n ** 3 * 4, "d2h_bytes_per_step": n ** 3 * 4,
               "bytes_per_rank_per_direction": S * n * n * 4}
        e2e["transfers"] = _transfer_lines(torch, host_in, host_out, dev, S * n * n * 4, e2e_s)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import ref_bench
        if not args.no_e2e:
            del host_in, host_out  # 2 x 32 GiB of pinned host memory back before the CPU run
        threads = os.cpu_count() or 1
        rate, kind, sample, runs = _cpu_reference(n, 1, 0, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
               "cpu": ref_bench.cpu_model(), "runs": runs}

    if rank == 0:
        cfg = _workload(n)
        cfg.update({"batch": batch, "slab_slices_per_rank": S, "parallelism": f"slab{world}",
                    "l2": f"inputs larger than L2 ({S * n * n * 4 / 2**30:g} GiB sinogram slab streamed per step per rank)"})
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "seconds_per_volume": ms_step / 1e3,
            "ms_per_step_stats": step_stats,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (analytic off-centre ellipsoid sinograms, generated on device)",
            "config": cfg,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_slice": alg[dom],
                         # every main kernel against the same HBM peak: its algorithmic bytes
                         # over its summed device time in the profiled step
                         "per_kernel": {k: {"algorithmic_bytes_per_slice": alg[k], "ms_per_step": stage[k],
                                            "achieved_gbs": alg[k] * S / (stage[k] / 1e3) / 1e9,
                                            "frac": alg[k] * S / (stage[k] / 1e3) / 1e9 / peak}
                                        for k in ("k1_radial", "k2_columns", "k3_rows") if stage[k] > 0}},
            "path_roofline": {"algorithmic_bytes_per_volume": alg["total"] * n,
                              "achieved_gbs": alg["total"] * n / (ms_step / 1e3) / 1e9 / world,
                              "frac_per_gpu": alg["total"] * n / (ms_step / 1e3) / 1e9 / world / peak},
            "issue_roofline": issue,
            "stage_ms_per_step": {k: v for k, v in stage.items() if v > 0},
            "gpu_launches": sum(launches.values()) * args.steps,
            "ss_comparator": ss,
            "forward_projector": fwd,
            "other_paths": paths,
            "counts_path": counts_path,
            "preprocess_path": pre_path,
            "e2e": e2e,
            "plan_create_ms": plan_ms,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
