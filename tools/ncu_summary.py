"""Summarise an .ncu-rep: key SOL / pipe / stall metrics (reads ncu --page raw)."""
import csv, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_sol_pct"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_sol_pct"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("l1tex__t_bytes.sum", "l1_bytes"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_cycles_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "gld_requests"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_lg.sum", "lg_wavefronts"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "wait", "not_selected", "selected", "dispatch_stall", "no_instruction", "tex_throttle", "membar", "drain",
          "branch_resolving", "sleeping", "misc"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    d = dict(zip(h, v))
    res = {"kernel": d.get("Kernel Name", "")[:60]}
    for k, name in KEYS:
        if k in d:
            res[name] = d[k]
    st = {}
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in d:
            try:
                st[s] = round(float(d[k]), 3)
            except ValueError:
                pass
    res["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1])[:6])
    return res


if __name__ == "__main__":
    import json
    for p in sys.argv[1:]:
        print(json.dumps(summary(p), indent=1))
