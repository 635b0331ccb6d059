"""Register / spill / stack table of every kernel in the per-L instantiation
unit (nvcc -Xptxas -v on tb_inst.cu with the Makefile's flags).

usage: python tools/ptxas_table.py 4096 [2048 ...] > table.md"""
import re
import subprocess
import sys

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def table(L):
    r = subprocess.run(["nvcc", *FLAGS, f"-DTB_L={L}", "-c", "-o", f"/tmp/ptxas_{L}.o",
                        "paper_1704_08364_b200/csrc/tb_inst.cu"], capture_output=True, text=True, check=True)
    rows, cur = [], None
    for ln in r.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\w+)'", ln)
        if m:
            cur = {"name": subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()}
            rows.append(cur)
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m:
            cur["stack"], cur["spill_st"], cur["spill_ld"] = m.groups()
        m = re.search(r"Used (\d+) registers", ln)
        if m:
            cur["regs"] = m.group(1)
    out = [f"### L = {L}", "", "| kernel | registers | spill stores (B) | spill loads (B) | stack (B) |", "|---|---|---|---|---|"]
    for row in sorted(rows, key=lambda x: x["name"]):
        name = row["name"].replace("tb::", "").replace("(tb::DevPlan, tb::Work, int, int, int, int)", "")
        name = re.sub(r"\(.*\)$", "", name)
        out.append(f"| `{name}` | {row.get('regs', '?')} | {row.get('spill_st', '?')} | {row.get('spill_ld', '?')} | "
                   f"{row.get('stack', '?')} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("# ptxas -v (sm_100a) per kernel instantiation\n")
    print("K2 path template argument: 0 = K2_ANY (full turn / nearest), 1 = K2_PLAIN (no texture view), "
          "2 = K2_TEX (the shipped half-turn bilinear path).  The second template argument of k2/k3 is "
          "CROP_HALF (n = L/2, the benchmark shape).\n")
    for L in sys.argv[1:] or ["4096"]:
        print(table(int(L)))
        print()
