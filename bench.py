"""bench.py -- checkpoint & restore throughput of the B200 device-memory
snapshot path (BASELINE.json metric) on N GPUs of one node.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One STEP = lock -> full checkpoint (scan + CRC32C + zero test + classify,
compaction, pagemap, pack, pinned drain) -> restore (H2D, scatter, zero fill,
verify) -> unlock of the rank's registered state: every row of SURVEY §8(a).
Default workload (N=1 and every N): configs[1] of BASELINE.json, GPT-2 small
fp32 weights + Adam moments (444 allocations, 1,493,277,696 B per rank), each
rank with its own seed; no data crosses GPUs ("scaling": "weak").

value  = sum over ranks of registered bytes / step time (GB/s of state that
         was checkpointed AND restored), step time = max over ranks of the
         CUDA-event interval on the library's stream.
e2e    = the same bytes / host wall clock of the public Python API calls
         (Context.lock/checkpoint/restore/unlock + image free), max over ranks.
--impl reference times the CPU oracle (oracle/, plain C, 1 thread) on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_CONTEXT = {
    "source": "PAPER.md §5.2 P:392-393 (Fig. 5), H100 PCIe Gen5 80 GB, cuda-checkpoint, GPT-2 training",
    "gpt2_small_checkpoint_s": 4.9, "gpt2_small_restore_s": 2.5, "gpt2_small_gpu_state_GB": 9.20,
    "gpt2_xl_checkpoint_s": 28.0, "gpt2_xl_restore_s": 11.0, "gpt2_xl_gpu_state_GB": 57.73,
    "derived_GBps": {"gpt2_small_ckpt": 1.88, "gpt2_small_restore": 3.68, "gpt2_xl_ckpt": 2.06, "gpt2_xl_restore": 5.25},
    "note": "context only (other hardware, other state); not the target",
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "MEASURED_PEAKS.json (measured copy)"}
    return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control words only: no data crosses GPUs
        pg = dist
    return world, rank, local, pg


def _max_over_ranks(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def _barrier(pg):
    if pg is not None:
        pg.barrier()


def probe_links(torch, nbytes=1 << 30):
    """K10 probes: pinned D2H / H2D copy bandwidth (the drain / restore roofline
    denominators), measured in this run with this rank's concurrency."""
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    out = {}
    for name, fn in (("d2h_gbs", lambda: h.copy_(d, non_blocking=True)),
                     ("h2d_gbs", lambda: d.copy_(h, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(3 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    x.fill_(1)
    xi = x.view(torch.int64)
    xi.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        xi.sum()
    e1.record()
    torch.cuda.synchronize()
    out["hbm_read_gbs"] = round(5 * x.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    del d, h, x, xi
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    world, rank, local, pg = _dist()
    # one rank per GPU; on a box with fewer GPUs than ranks (functional tests)
    # ranks share devices round-robin
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    local = dev
    from paper_2502_16631_b200 import dist as gdist
    from paper_2502_16631_b200 import gcr, synth

    w = synth.make_workload(args.config, rank=rank, page_size=args.page_size, gib=args.gib)
    ctx = gcr.Context(local, page_size=w.page_size, chunk_bytes=args.chunk_mb << 20,
                      n_copy_streams=args.streams, n_staging_slots=args.slots,
                      direct_min_bytes=(1 << 64) - 1 if args.direct_min_mb < 0 else int(args.direct_min_mb * (1 << 20)))
    # --release: the state lives in one releasable gcr_mem_alloc block, carved
    # into the workload's allocations (f2: checkpoint frees the HBM, restore
    # re-backs the same addresses)
    ts = w.materialize(region=ctx.alloc_tensor(w.total_bytes, local) if args.release else None)
    torch.cuda.synchronize()
    for t in ts:
        ctx.register_tensor(t)
    R0 = w.total_bytes
    keep_chain = False
    if args.mode == "incremental":
        # base image + the worst-case buffer a checkpoint takes before shrinking + kept incrementals
        per_inc = int(args.dirty * R0 * 1.05) + (64 << 20)
        need = 2 * R0 + (args.steps + args.warmup) * per_inc + (256 << 20)
        mem_total = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        keep_chain = need < 0.7 * mem_total
        ctx.reserve_host(need if keep_chain else 2 * R0 + 2 * per_inc + (256 << 20))
    else:
        ctx.reserve_host(R0 + (256 << 20))
    probes = probe_links(torch)
    R = w.total_bytes
    cst = ctx.stream()
    stream = torch.cuda.ExternalStream(cst)

    incremental = args.mode == "incremental"
    base_img, incs = None, []
    if incremental:  # the full checkpoint the incrementals diff against (untimed)
        ctx.lock()
        base_img = ctx.checkpoint(gcr.GCR_FULL)
        ctx.unlock()
    step_no = [0]
    io_times = []

    def step(timed):
        if incremental:  # the "training step": dirty a fresh seeded set of pages (untimed harness work)
            muts = synth.dirty_mutations(w, args.dirty, rng_seed=9000 + step_no[0], clustered=args.clustered)
            synth.gpu_xor_batch([ts[a].data_ptr() + o for (a, o, x) in muts], [x for (a, o, x) in muts],
                                torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
        step_no[0] += 1
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(stream)
        if pg is not None:  # globally consistent cut: all-or-nothing lock vote over gloo (dist.py)
            st = gdist.lock_all(ctx)
            if st != 0:
                raise RuntimeError(f"lock vote failed: {st}")
        else:
            ctx.lock()
        img = ctx.checkpoint(gcr.GCR_INCREMENTAL if incremental else gcr.GCR_FULL)
        s_ck = ctx.stats()
        if args.release:
            ctx.release()
        if args.storage:  # f3: the image goes to a file (durable), comes back from it, then restores
            path = os.path.join(args.storage, f"gcr_bench_rank{rank}.img")
            s0 = time.perf_counter()
            img.write_file(path)
            s1 = time.perf_counter()
            img.free()
            img = ctx.read_file(path)
            s2 = time.perf_counter()
            io_times.append((s1 - s0, s2 - s1))
        if not incremental:
            ctx.restore([img])
        ctx.unlock()
        e1.record(stream)
        if incremental and keep_chain:
            incs.append(img)
        else:
            img.free()
        h1 = time.perf_counter()
        e1.synchronize()
        s = ctx.stats()
        return e0.elapsed_time(e1) * 1e-3, h1 - h0, s_ck, s

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    _barrier(pg)
    launches0 = ctx.stats()["kernel_launches"]
    dev, host, recs = [], [], []
    with ClockSampler(local) as clk:
        _barrier(pg)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            d, h, sck, s = step(True)
            dev.append(d)
            host.append(h)
            recs.append((sck, s))
        torch.cuda.synchronize()
        _barrier(pg)
    launches = ctx.stats()["kernel_launches"] - launches0
    chain_restore = None
    if incremental and keep_chain:  # restore the whole chain once: full + every incremental, then verify
        ctx.lock()
        t0 = time.perf_counter()
        ctx.restore([base_img] + incs)
        t_rs = time.perf_counter() - t0
        ctx.unlock()
        sr = ctx.stats()
        chain_restore = {"images": 1 + len(incs), "seconds": round(t_rs, 4), "GBps_registered": round(R / t_rs / 1e9, 3),
                         "h2d_bytes": sr["restore_h2d_bytes"], "verify_failures": sr["verify_failures"]}
        for im in incs:
            im.free()
    if base_img is not None:
        base_img.free()
    t_dev = _max_over_ranks(pg, sum(dev))
    t_host = _max_over_ranks(pg, sum(host))
    R_all = _sum_over_ranks(pg, float(R))
    K = args.steps
    # per-phase, per-rank means
    ck = sum(r[0]["checkpoint_ns"] for r in recs) / K * 1e-9
    rs = sum(r[1]["restore_ns"] for r in recs) / K * 1e-9 if not incremental else float("nan")
    sc = recs[-1][0]
    scan_ns = sum(r[0]["scan_dev_ns"] for r in recs)
    scan_l = sum(r[0]["scan_launches"] for r in recs)
    pack_ns = sum(r[0]["pack_dev_ns"] for r in recs)
    ver_ns = sum(r[1]["verify_dev_ns"] for r in recs)
    scat_ns = sum(r[1]["scatter_dev_ns"] for r in recs)
    img_b = sc["image_bytes"]
    peaks = _peaks()
    # K4 moves only the STAGED bytes (read + write); long runs go by direct DMA.
    # K6 scatters the staged restore bytes (read + write), K7 writes the ZERO pages.
    pack_b = 2 * (img_b - sc["direct_bytes"])
    rs_last = recs[-1][1]
    scat_b = 2 * (img_b - rs_last["restore_direct_bytes"]) + rs_last["pages_zero"] * w.page_size
    kern = {
        "K1_scan": {"dev_ms_per_step": scan_ns / K * 1e-6, "launches_per_step": scan_l / K,
                    "alg_bytes_per_step": R, "GBps": R * K / max(scan_ns, 1)},
        "K4_pack": {"dev_ms_per_step": pack_ns / K * 1e-6, "alg_bytes_per_step": pack_b,
                    "GBps": pack_b * K / max(pack_ns, 1)},
        "K6K7_scatter_zero": None if incremental else
        {"dev_ms_per_step": scat_ns / K * 1e-6, "alg_bytes_per_step": scat_b,
         "GBps": scat_b * K / max(scat_ns, 1), "note": "zero bytes counted as pages_zero x page_size (upper bound)"},
        "K8_verify": None if incremental else
        {"dev_ms_per_step": ver_ns / K * 1e-6, "alg_bytes_per_step": R, "GBps": R * K / max(ver_ns, 1)},
    }
    # dominant kernel = k_scan (K1 in scan mode during the checkpoint, K8 =
    # the same kernel in verify mode during the restore): average over all its
    # launches in the timed region of algorithmic bytes per launch / duration.
    scan_launches = sum(r[0]["scan_launches"] for r in recs) + sum(r[1]["verify_launches"] for r in recs)
    scan_bytes = R * K * (1 if incremental else 2)
    scan_time = scan_ns + (0 if incremental else ver_ns)
    achieved = scan_bytes / max(scan_time, 1)  # bytes/ns == GB/s
    traffic = None
    tp = os.path.join(ROOT, "profiles", "scan_traffic.json")
    if os.path.exists(tp):  # DRAM bytes / algorithmic bytes of k_scan, from one ncu --set full capture
        try:
            ratio = json.load(open(tp))["dram_over_algorithmic"]
            traffic = round(ratio * scan_bytes / max(scan_launches, 1))
        except Exception:
            traffic = None
    d2h = sc["image_bytes"] + 4 * sc["pages_scanned"] + 16 * sc["n_entries"]
    h2d = recs[-1][1]["restore_h2d_bytes"] + 4 * sc["pages_scanned"]
    ck_gbs = R / ck / 1e9
    rs_gbs = R / rs / 1e9 if not incremental else float("nan")
    result = {
        "metric": "checkpoint & restore GB/s per GPU and box-aggregate at 1/2/4/8 B200 vs roofline",
        "value": round(R_all * K / t_dev / 1e9, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(t_dev / K * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded counter-based generator; training-state-shaped fp32/bf16 values)",
        "config": {"workload": _workload_desc(args.config + ("i" if incremental and args.config == "C4" else ""), w),
                   "dirty_fraction": args.dirty if incremental else None, "registered_bytes_per_rank": R,
                   "allocations": len(w.allocs), "page_size": w.page_size, "chunk_bytes": args.chunk_mb << 20,
                   "copy_streams": args.streams, "staging_slots": args.slots or args.streams, "direct_min_bytes": int(args.direct_min_mb * (1 << 20)) if args.direct_min_mb >= 0 else None,
                   "parallelism": f"independent ranks x{world} (gloo control plane)",
                   "l2": "inputs larger than L2 (registered state >> 126 MB; no flush needed)"},
        "per_gpu": {"checkpoint_GBps": round(ck_gbs, 3), "restore_GBps": round(rs_gbs, 3),
                    "roundtrip_GBps": round(R * K / t_dev / 1e9, 3),
                    "image_GBps_ckpt": round(img_b / ck / 1e9, 3)},
        "box": {"checkpoint_GBps": round(_sum_over_ranks(pg, ck_gbs), 3),
                "restore_GBps": round(_sum_over_ranks(pg, rs_gbs), 3)},
        "link_roofline": {"drain_GBps": round(img_b / (sc["drain_ns"] * 1e-9) / 1e9, 2),
                          "d2h_probe_GBps": probes["d2h_gbs"], "h2d_probe_GBps": probes["h2d_gbs"],
                          "checkpoint_frac_of_d2h": round(ck_gbs / probes["d2h_gbs"] * img_b / R, 3),
                          "restore_frac_of_h2d": round(rs_gbs / probes["h2d_gbs"] * img_b / R, 3) if not incremental else None},
        "roofline": {"kernel": "k_scan (K1 scan + K8 verify launches)", "bound": "hbm",
                     "launches_per_step": round(scan_launches / K, 2),
                     "alg_bytes_per_launch": round(scan_bytes / max(scan_launches, 1)),
                     "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 3), "traffic": traffic,
                     "peak_source": peaks["source"], "hbm_read_probe_GBps": probes["hbm_read_gbs"]},
        "kernels": {k: ({kk: round(vv, 4) if isinstance(vv, float) else vv for kk, vv in v.items()} if v else None)
                    for k, v in kern.items()},
        "e2e": {"value": round(R_all * K / t_host / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "what": "host wall clock of Context.lock/checkpoint/restore/unlock/free via the Python binding"},
        "gpu_launches": int(_sum_over_ranks(pg, float(launches))),
        "paper_context": PAPER_CONTEXT,
        "mode": args.mode,
        "chain_restore": chain_restore,
        "probes": probes,
        "release": {"release_ms": round(sum(r[1]["release_ns"] for r in recs) / K * 1e-6, 3),
                    "remap_ms": round(sum(r[1]["remap_ns"] for r in recs) / K * 1e-6, 3),
                    "released_bytes": recs[-1][1]["released_bytes"],
                    "what": "f2: checkpoint -> gcr_release (HBM returned to the driver) -> restore re-maps the same VAs"}
        if args.release else None,
        "storage": {"dir": args.storage, "write_GBps": round(img_b * len(io_times) / max(sum(t[0] for t in io_times), 1e-9) / 1e9, 3),
                    "read_GBps": round(img_b * len(io_times) / max(sum(t[1] for t in io_times), 1e-9) / 1e9, 3),
                    "what": "f3: pinned image -> file (parallel pwrite + fdatasync + drop cache) -> pinned image (parallel pread)"}
        if args.storage else None,
    }
    result["clocks"] = clk.summary()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if pg is not None:
        pg.destroy_process_group()


def _workload_desc(name, w):
    return {"C1": "C1: 64 MiB region as 4 contiguous allocations, 25% zero pages, full checkpoint + restore",
            "C2": "C2: GPT-2 small training state, fp32 weights + Adam m/v (444 allocations), full checkpoint + restore",
            "C3": "C3: Llama-3 8B ZeRO-3 shard per rank (bf16 param/grad + fp32 master/m/v), full checkpoint + restore",
            "C4": f"C4: {len(w.allocs)} x 1 GiB per GPU, full checkpoint + restore",
            "C4i": f"C4: {len(w.allocs)} x 1 GiB per GPU, incremental checkpoint of a seeded dirty set per step",
            "C5": f"C5: {len(w.allocs)} GiB per GPU, 25% zero 2 MiB regions, full checkpoint + restore"}[name]


def cpu_baseline(args, budget_s=15.0):
    """The oracle as it stands (plain C, single-threaded, Sarwate CRC) on a
    bounded sample of the same workload: a prefix of its allocations,
    checkpoint + restore into a poisoned copy, repeated for ~budget_s: half on
    1 thread, half on every host core (one oracle instance per thread)."""
    import numpy as np
    from oracle import oracle
    from paper_2502_16631_b200 import synth
    w = synth.make_workload(args.config, rank=0, page_size=args.page_size, gib=args.gib)
    cap = 256 << 20
    idx, tot = [], 0
    for a, s in enumerate(w.allocs):
        if tot + s.nbytes > cap and idx:
            continue
        idx.append(a)
        tot += s.nbytes
        if tot >= cap:
            break
    cont = [w.cpu_bytes(a) for a in idx]
    reg = [(a + 1, 0x7F0000000000 + (a << 32), w.allocs[a].nbytes) for a in idx]
    sizes = [w.allocs[a].nbytes for a in idx]

    def loop(budget, out):
        done, t0, reps = 0, time.perf_counter(), 0
        while True:
            st, s = oracle.checkpoint(w.page_size, reg, cont)
            tgt = [np.full(n, 0xA5, np.uint8) for n in sizes]
            st2, vf, _ = oracle.restore([s], w.page_size, sizes, tgt)
            assert st == 0 and st2 == 0 and vf == 0
            done += tot
            reps += 1
            if time.perf_counter() - t0 >= budget:
                break
        out.append((done, reps))

    # T = 1, then T = the host's cores, each thread running
    # the unmodified single-threaded oracle on its own copy of the sample
    # (ctypes releases the GIL inside the C calls)
    import threading
    one = []
    t0 = time.perf_counter()
    loop(budget_s / 2, one)
    v1 = one[0][0] / (time.perf_counter() - t0) / 1e9
    T = max(1, min(os.cpu_count() or 1, 32))
    outs = []
    ths = [threading.Thread(target=loop, args=(budget_s / 2, outs)) for _ in range(T)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    vT = sum(d for d, _ in outs) / (time.perf_counter() - t0) / 1e9
    reps = one[0][1] + sum(r for _, r in outs)
    return {"value": round(vT, 4), "unit": "GB/s", "cores": T, "kind": "oracle", "value_1thread": round(v1, 4),
            "sample": f"{len(idx)} of {len(w.allocs)} allocations ({tot} B) of {args.config}, checkpoint+restore "
                      f"x{reps} ({one[0][1]} on 1 thread, then {T} threads concurrently)"}


def run_reference(args):
    world, rank, local, pg = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0, None
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    for _ in range(args.warmup):
        pass
    budget = max(3.0, min(30.0, 120.0 / max(1, args.steps)))
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(args, budget_s=budget))
    v = statistics.median(x["value"] for x in vals)
    res = {"impl": "reference", "metric": "checkpoint & restore GB/s per GPU and box-aggregate at 1/2/4/8 B200 vs roofline",
           "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic", "config": {"workload": args.config + " (bounded sample; see cpu_baseline.sample)"},
           "cpu_baseline": {**vals[0], "value": v},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "the plain CPU oracle (oracle/gcr_oracle.c) as it stands; the paper ships no runnable code"}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--page-size", type=int, default=None)
    ap.add_argument("--gib", type=int, default=None, help="C4/C5 GiB per GPU")
    ap.add_argument("--chunk-mb", type=int, default=1024)
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--slots", type=int, default=0, help="staging slots (0 = one per copy stream)")
    ap.add_argument("--direct-min-mb", type=float, default=None,
                    help="runs >= this go by direct DMA (default: the library's); -1 = always staged")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--mode", default="full", choices=["full", "incremental"],
                    help="full: checkpoint+restore per step (default); incremental: dirty --dirty of the pages, "
                         "then an incremental checkpoint per step; the whole chain is restored once at the end")
    ap.add_argument("--dirty", type=float, default=0.01)
    ap.add_argument("--clustered", action="store_true", help="dirty pages in 64-page runs instead of scattered")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--storage", default=None, help="full mode: directory for the f3 storage tier round trip")
    ap.add_argument("--release", action="store_true",
                    help="full mode: state in releasable gcr_mem_alloc memory; each step releases the HBM after "
                         "the checkpoint and the restore re-maps the same addresses (SURVEY f2)")
    args = ap.parse_args()
    if args.storage and args.mode != "full":
        ap.error("--storage needs --mode full")
    if args.release and args.mode != "full":
        ap.error("--release needs --mode full (the restore re-maps the released memory)")
    if args.direct_min_mb is None:
        from paper_2502_16631_b200 import gcr as _g
        args.direct_min_mb = _g.default_config().direct_min_bytes / (1 << 20)
    if args.gib is None:
        args.gib = {"C4": 40, "C5": 16}.get(args.config, 16)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
