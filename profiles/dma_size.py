"""D2H / H2D copy-engine throughput vs DMA size (pinned host), back-to-back on 1 and 2 streams."""
import json
import torch
dev = torch.empty(1 << 30, dtype=torch.uint8, device="cuda").fill_(1)
host = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
s = [torch.cuda.Stream(), torch.cuda.Stream()]
for mb in [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024]:
    n = mb << 20
    k = max(1, (1 << 30) // n)
    for nst in (1, 2):
        for d2h in (True, False):
            best = 0
            for rep in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s[0])
                s[1].wait_event(e0)
                for i in range(k):
                    st = s[i % nst]
                    with torch.cuda.stream(st):
                        if d2h:
                            host[i * n:(i + 1) * n].copy_(dev[i * n:(i + 1) * n], non_blocking=True)
                        else:
                            dev[i * n:(i + 1) * n].copy_(host[i * n:(i + 1) * n], non_blocking=True)
                ev = torch.cuda.Event(); ev.record(s[1]); s[0].wait_event(ev)
                e1.record(s[0])
                e1.synchronize()
                best = max(best, k * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            print(json.dumps({"MB": mb, "streams": nst, "dir": "d2h" if d2h else "h2d", "GBps": round(best, 2)}), flush=True)
