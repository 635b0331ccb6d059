"""Executed warp instructions and stall samples per CUDA source line.

Joins an ncu source-page CSV (SASS rows with "Instructions Executed" and
"Warp Stall Sampling", exported by tools/gpu_round_profile.sh) with the
line table of the same build (nvdisasm --print-line-info of the cubin in the
kernel's object file), so hot lines show up by file:line instead of by
opcode.  The object must be the one the profiled library was linked from.

usage: line_mix.py <source_<kernel>.csv> <object.o> <mangled-kernel-substring> [top]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, fn_sub):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                       stdout=subprocess.DEVNULL)
        cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cubin)], check=True,
                              capture_output=True, text=True).stdout
    table, inside, cur = {}, False, None
    for ln in sass.splitlines():
        if ln.startswith(".text."):
            inside = fn_sub in ln
            cur = None
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(\S+)", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2))
    return table


def main():
    src, obj, fn_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(obj, fn_sub)
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    cols = rows[hdr]
    ia, ie, iw = cols.index("Address"), cols.index("Instructions Executed"), cols.index(
        "Warp Stall Sampling (All Samples)")
    body = [r for r in rows[hdr + 1:] if len(r) == len(cols) and r[ia].startswith("0x")]
    base = int(body[0][ia], 16)
    by_line = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    tot_i = tot_s = 0
    miss = 0
    for r in body:
        off = int(r[ia], 16) - base
        n, smp = int(r[ie] or 0), int(r[iw] or 0)
        tot_i += n
        tot_s += smp
        ent = table.get(off)
        if ent is None:
            miss += 1
            continue
        (line, op) = ent
        b = by_line[line]
        b[0] += n
        b[1] += smp
        b[2][op.split(".")[0]] += n
    print(f"total warp insts {tot_i}  stall samples {tot_s}  (unmapped rows {miss})")
    for line, (n, smp, ops) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        mix = " ".join(f"{o}:{c * 100 // max(n, 1)}" for o, c in ops.most_common(4))
        print(f"{str(line):40s} {n:12d} {100 * n / tot_i:5.1f}%  stalls {100 * smp / max(tot_s, 1):5.1f}%  {mix}")


if __name__ == "__main__":
    main()
