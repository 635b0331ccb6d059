"""Summarise one gpurun evidence directory (tools/gpu_round_profile.sh output)
into profiles/<round>/: the bench line, the ncu launch list with per-kernel
shares, and per-kernel SOL / pipe / stall / DRAM-traffic numbers from the
`ncu --set full` captures (raw CSV exported on the box).

usage: python tools/ncu_summary.py gpurun_out/<tag> profiles/<round>
"""
import collections
import csv
import json
import os
import shutil
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_sol_pct"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_sol_pct"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "wait", "not_selected", "dispatch_stall", "no_instruction", "tex_throttle", "branch_resolving"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
         "msecond": 1e6, "nsecond": 1}


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h, u, v = rows[i], rows[i + 1], rows[i + 2]
    out = {"kernel": v[h.index("Kernel Name")]}
    for k, name in KEYS:
        if k in h:
            j = h.index(k)
            val = v[j].replace(",", "")
            try:
                x = float(val) * SCALE.get(u[j], 1)
            except ValueError:
                x = val
            out[name] = x
    st = {}
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in h:
            try:
                st[s] = round(float(v[h.index(k)]), 3)
            except ValueError:
                pass
    out["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1])[:6])
    return out


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[i + 1:]:
        if len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        ns = float(r[h.index("Metric Value")].replace(",", "")) * SCALE.get(r[h.index("Metric Unit")], 1)
        tot[name] += ns
        cnt[name] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "avg_us": tot[k] / cnt[k] / 1e3, "share": tot[k] / s} for k in tot}


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    res = {}
    bench = os.path.join(src, "bench.json")
    if os.path.exists(bench):
        shutil.copy(bench, os.path.join(dst, "bench.json"))
        try:
            res["bench"] = json.loads(open(bench).read().strip().splitlines()[-1])
        except Exception:
            pass
    if os.path.exists(os.path.join(src, "launches.csv")):
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "ncu_launches.csv"))
        res["launch_shares"] = launch_shares(os.path.join(src, "launches.csv"))
    res["kernels"] = {}
    for f in sorted(os.listdir(src)):
        if f.startswith("raw_") and f.endswith(".csv"):
            k = f[4:-4]
            try:
                res["kernels"][k] = raw_metrics(os.path.join(src, f))
            except Exception as e:  # noqa: BLE001
                res["kernels"][k] = {"error": str(e)}
    for f in os.listdir(src):
        if f.startswith("source_") or f == "pytest_gpu.log":
            pass
    if os.path.exists(os.path.join(src, "pytest_gpu.log")):
        shutil.copy(os.path.join(src, "pytest_gpu.log"), os.path.join(dst, "pytest_gpu.log"))
    # per-launch DRAM traffic of each captured kernel, read by bench.py for
    # roofline.traffic (bytes per slice = per launch / slices per launch)
    spl = res.get("bench", {}).get("config", {}).get("batch")
    n = res.get("bench", {}).get("config", {}).get("n_slices")
    traffic = {"source": dst, "size": n, "slices_per_launch": spl, "kernels": {}}
    for k, m in res["kernels"].items():
        if "dram_read" in m and "dram_write" in m and spl:
            traffic["kernels"][k] = {"dram_bytes_per_launch": m["dram_read"] + m["dram_write"],
                                     "dram_bytes_per_slice": (m["dram_read"] + m["dram_write"]) / spl,
                                     "warp_inst_per_slice": m.get("warp_inst", 0.0) / spl,
                                     "fp32_pipe_pct": m.get("fma_pipe_pct")}
    with open(os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(dst, "ncu_summary.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
