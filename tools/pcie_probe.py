"""PCIe ceiling probe for the e2e leg: pinned H2D alone, D2H alone, and both
directions concurrently (separate streams), at several chunk sizes.
Prints one JSON line per configuration (GB/s per direction)."""
import json
import torch

GiB = 1 << 30


def run(total, chunk, h2d, d2h):
    n = total // chunk
    dev = torch.device("cuda:0")
    hin = torch.empty(total // 4, dtype=torch.float32, pin_memory=True)
    hout = torch.empty(total // 4, dtype=torch.float32, pin_memory=True)
    din = torch.empty(2 * chunk // 4, dtype=torch.float32, device=dev)
    dout = torch.empty(2 * chunk // 4, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c = chunk // 4
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for i in range(n):
            j = (i % 2) * c
            if h2d:
                with torch.cuda.stream(s1):
                    din[j:j + c].copy_(hin[i * c:(i + 1) * c], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    hout[i * c:(i + 1) * c].copy_(dout[j:j + c], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    return total / s / 1e9


if __name__ == "__main__":
    for chunk_mib in (16, 64, 256):
        for h2d, d2h in ((True, False), (False, True), (True, True)):
            gbs = run(8 * GiB, chunk_mib << 20, h2d, d2h)
            print(json.dumps({"chunk_MiB": chunk_mib, "h2d": h2d, "d2h": d2h, "GB_per_s_per_direction": round(gbs, 1)}), flush=True)
