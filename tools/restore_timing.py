"""Host-side cost of a restore (validation + planning) vs its transfer phase,
for C2 at a page size, compressed or not: restore_ns (whole call) vs
restore_h2d_ns (first H2D issued -> verified)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_16631_b200 import gcr, synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for compress in (0, 1):
    w = synth.make_workload("C2", page_size=P)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(0, page_size=P, compress=compress)
    for t in ts:
        ctx.register_tensor(t)
    ctx.reserve_host(w.total_bytes + (256 << 20))
    ctx.lock()
    img = ctx.checkpoint()
    for _ in range(3):
        ctx.restore([img])
        s = ctx.stats()
        print(f"P={P} compress={compress}: restore {s['restore_ns'] / 1e6:.2f} ms, transfer phase "
              f"{s['restore_h2d_ns'] / 1e6:.2f} ms, host validation+planning {(s['restore_ns'] - s['restore_h2d_ns']) / 1e6:.2f} ms, "
              f"decode {s['decode_dev_ns'] / 1e6:.2f} ms, checkpoint {s['checkpoint_ns'] / 1e6:.2f} ms, codec {s['codec_dev_ns'] / 1e6:.2f} ms",
              flush=True)
    ctx.unlock()
    ctx.close()
    del ts
    torch.cuda.empty_cache()
