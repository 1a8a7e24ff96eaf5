"""Where the host time of an incremental checkpoint step goes (C4-shaped, 1 %
dirty): per call (lock, checkpoint, stats, unlock, image free) wall time vs
the checkpoint's own device span (stats checkpoint_ns / drain_ns).  Run on
the GPU box:  python tools/host_overhead.py [GiB] [steps]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_16631_b200 import gcr, synth  # noqa: E402

gib = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = synth.make_workload("C4", gib=gib)
ts = w.materialize()
torch.cuda.synchronize()
ctx = gcr.Context(0, page_size=w.page_size)
for t in ts:
    ctx.register_tensor(t)
ctx.reserve_host(2 * w.total_bytes + (1 << 30))
ctx.lock()
base = ctx.checkpoint()
ctx.unlock()
stream = torch.cuda.ExternalStream(ctx.stream())
rows = []
for k in range(steps):
    muts = synth.dirty_mutations(w, 0.01, rng_seed=500 + k)
    synth.gpu_xor_batch([ts[a].data_ptr() + o for (a, o, x) in muts], [x for (a, o, x) in muts],
                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    t1 = time.perf_counter()
    ctx.lock()
    t2 = time.perf_counter()
    img = ctx.checkpoint(gcr.GCR_INCREMENTAL)
    t3 = time.perf_counter()
    s = ctx.stats()
    t4 = time.perf_counter()
    ctx.unlock()
    t5 = time.perf_counter()
    e1.record(stream)
    img.free()
    t6 = time.perf_counter()
    e1.synchronize()
    ev = e0.elapsed_time(e1)
    rows.append((ev, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3,
                 (t6 - t5) * 1e3, s["checkpoint_ns"] * 1e-6, s["drain_ns"] * 1e-6, s["scan_dev_ns"] * 1e-6))
print("event_ms record lock checkpoint stats unlock free | ckpt_ns drain_ns scan_dev (ms)")
for r in rows:
    print(" ".join(f"{x:7.3f}" for x in r))
