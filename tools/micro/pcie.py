"""Host<->device copy bandwidth on this box (pinned host memory), one and two
streams, for sizing the e2e path."""
import time
import torch

def bw(nbytes, d2h=True, streams=1, reps=5):
    dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    host = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = dev.numel() // streams
    def go():
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                a, b = slice(i * chunk, (i + 1) * chunk), None
                if d2h:
                    host[a].copy_(dev[a], non_blocking=True)
                else:
                    dev[a].copy_(host[a], non_blocking=True)
        torch.cuda.synchronize()
    go()
    t = time.perf_counter()
    for _ in range(reps):
        go()
    dt = (time.perf_counter() - t) / reps
    return nbytes / dt / 1e9

for n in (38 << 20, 512 << 20, 2 << 30):
    print(f"{n >> 20} MiB  D2H {bw(n):.1f} GB/s  D2H x2 streams {bw(n, streams=2):.1f}  "
          f"H2D {bw(n, d2h=False):.1f} GB/s")
