"""K1 / K8 device time vs registered size (fixed-overhead fit)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2502_16631_b200 import gcr, synth
res = []
for mib in [128, 256, 512, 1024, 2048, 4096, 8192]:
    n = mib << 20
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), n, 1, 0, synth.RANDOM)
    torch.cuda.synchronize()
    ctx = gcr.Context(0)
    ctx.register_tensor(t)
    ctx.reserve_host(n + (64 << 20))
    k1, k8 = [], []
    for it in range(6):
        ctx.lock(); img = ctx.checkpoint(gcr.GCR_FULL); s1 = ctx.stats(); ctx.restore([img]); s2 = ctx.stats(); ctx.unlock(); img.free()
        if it >= 2:
            k1.append(s1["scan_dev_ns"]); k8.append(s2["verify_dev_ns"])
    ctx.close(); del t; torch.cuda.empty_cache()
    r = {"MiB": mib, "k1_us": min(k1) / 1e3, "k8_us": min(k8) / 1e3, "k1_TBps": n / min(k1) / 1e3, "k8_TBps": n / min(k8) / 1e3}
    print(json.dumps(r), flush=True)
