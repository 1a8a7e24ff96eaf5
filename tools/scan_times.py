"""GCR_SCAN_TIMES diagnostics: K8 (verify) per-warp stamps over registries of
several sizes -> where a launch's fixed cost goes (run with GCR_SCAN_TIMES=1)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_16631_b200 import gcr, synth  # noqa: E402

for mib in [int(x) for x in (sys.argv[1:] or ["128", "1024", "4096"])]:
    n = mib << 20
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), n, 1, 0, synth.RANDOM)
    torch.cuda.synchronize()
    ctx = gcr.Context(0)
    ctx.register_tensor(t)
    ctx.reserve_host(n + (64 << 20))
    ctx.lock()
    img = ctx.checkpoint()
    for _ in range(3):
        ctx.restore([img])
        s = ctx.stats()
        print(f"MiB {mib}: verify {s['verify_dev_ns'] / 1e3:.1f} us = {n / s['verify_dev_ns']:.0f} GB/s; "
              f"scan {s['scan_dev_ns'] / 1e3:.1f} us", file=sys.stderr, flush=True)
    ctx.unlock()
    img.free()
    ctx.close()
    del t
    torch.cuda.empty_cache()
