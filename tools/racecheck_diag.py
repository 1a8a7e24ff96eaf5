"""Diagnostic for the racecheck run (profiles/r2c): a C1-sized checkpoint ->
restore cycle that separates 'the restored bytes are wrong' from 'the verify
(K8) computes wrong digests' by restoring with verify off, comparing every
byte, then running the verify alone on the restored state."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_16631_b200 import gcr, synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sizes = [3 * P + 4096 + 48, 5 * P, 2 * P + 512]
ts = []
for i, n in enumerate(sizes):
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    synth.gpu_fill(t.data_ptr(), n, 42, i, synth.RANDOM)
    ts.append(t)
torch.cuda.synchronize()
cont = [t.cpu().numpy().copy() for t in ts]
for verify in (0, 1):
    ctx = gcr.Context(0, page_size=P, verify=verify)
    for t in ts:
        ctx.register_tensor(t)
    ctx.lock()
    img = ctx.checkpoint()
    for t in ts:
        t.fill_(0xA5)
    st = ctx.try_restore([img])
    s = ctx.stats()
    ok = all(np.array_equal(t.cpu().numpy(), c) for t, c in zip(ts, cont))
    print(f"P={P} verify={verify}: restore status {st}, bytes restored correctly: {ok}, "
          f"verify_failures {s['verify_failures']}, first_bad {s['first_bad_page']}", flush=True)
    # verify again on the (now known) state: a second restore of the same image
    st2 = ctx.try_restore([img])
    s2 = ctx.stats()
    print(f"   second restore: status {st2}, verify_failures {s2['verify_failures']}", flush=True)
    ctx.unlock()
    ctx.close()
