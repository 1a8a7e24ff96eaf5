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
box    = the same bytes / barrier-to-barrier host time per step (every rank
         passes a gloo barrier before and after each step), max over ranks.
--gpus N without torchrun re-launches this script as N ranks
(torch.distributed.run, 127.0.0.1); each rank binds itself and its pinned
memory to its GPU's NUMA node before any pinned allocation.
--impl reference times the CPU oracle (oracle/, plain C, one single-threaded
instance per host core over a partition of the allocations) on the WHOLE
workload (rank 0 only); it never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

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


def probe_links(torch, ctx=None, nbytes=1 << 30):
    """K10 probes, taken with every rank probing at once
    (the caller brackets this with barriers): pinned D2H / H2D copy bandwidth
    -- the drain / restore roofline denominators -- over the image pool itself
    (gcr_probe_link: the pinned pages the next image lands on) and over a
    separate torch pinned buffer, plus an HBM read probe."""
    out = {}
    if ctx is not None:  # the pool probe stages through a slot: at most one chunk
        d2h, h2d = ctx.probe_link(min(nbytes, ctx.cfg.chunk_bytes))
        out["pool_d2h_gbs"], out["pool_h2d_gbs"] = round(d2h, 2), round(h2d, 2)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
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


def bind_numa(torch, dev: int) -> dict:
    """Bind this rank's threads and its later host allocations (the pinned
    image pool) to the NUMA node of its GPU (SURVEY §8(e) 'shared resources',
    H4): sysfs numa_node of the GPU's PCI function -> sched_setaffinity to the
    node's CPUs + set_mempolicy(MPOL_PREFERRED, node).  Called before any
    pinned allocation.  A node of -1 (a single-node VM) binds nothing."""
    p = torch.cuda.get_device_properties(dev)
    bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    info = {"gpu_bdf": bdf}
    try:
        node = int(open(f"/sys/bus/pci/devices/{bdf}/numa_node").read().strip())
    except OSError as e:
        return {**info, "numa_node": None, "bound": False, "why": f"sysfs: {e.strerror}"}
    info["numa_node"] = node
    if node < 0:
        return {**info, "bound": False, "why": "sysfs numa_node = -1 (one NUMA node: nothing to bind)"}
    cpus = set()
    for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    os.sched_setaffinity(0, cpus)
    import ctypes
    libc = ctypes.CDLL(None, use_errno=True)
    mask = (ctypes.c_ulong * 16)()
    mask[node // 64] = 1 << (node % 64)
    MPOL_PREFERRED, SYS_set_mempolicy = 1, 238  # x86_64
    rc = libc.syscall(SYS_set_mempolicy, MPOL_PREFERRED, mask, 16 * 64 + 1)
    return {**info, "bound": True, "cpus": len(cpus), "mempolicy": "preferred" if rc == 0 else
            f"set_mempolicy failed (errno {ctypes.get_errno()})"}


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-run this script as N ranks of one node
    (one process per GPU) through torch.distributed.run on 127.0.0.1; rank 0
    prints the JSON line (stdout is inherited)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def run_ours(args):
    import torch
    world, rank, local, pg = _dist()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but {world} rank(s) running")
    if args.dry_run:  # launch plumbing only (CPU-testable): every rank reports, rank 0 prints
        me = {"rank": rank, "local_rank": local, "pid": os.getpid()}
        allr = [None] * world
        if pg is not None:
            pg.all_gather_object(allr, me)
            pg.barrier()
        else:
            allr = [me]
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": allr}), flush=True)
        if pg is not None:
            pg.destroy_process_group()
        return
    # one rank per GPU; on a box with fewer GPUs than ranks (functional runs)
    # ranks share devices round-robin, and the line says so
    n_dev = torch.cuda.device_count()
    dev = local % n_dev
    numa = bind_numa(torch, dev)  # before the first pinned allocation
    torch.cuda.set_device(dev)
    local = dev
    from paper_2502_16631_b200 import dist as gdist
    from paper_2502_16631_b200 import gcr, synth
    if args.direct_min_mb is None:
        args.direct_min_mb = gcr.default_config().direct_min_bytes / (1 << 20)

    w = synth.make_workload(args.config, rank=rank, page_size=args.page_size, gib=args.gib)
    ctx = gcr.Context(local, page_size=w.page_size, chunk_bytes=args.chunk_mb << 20,
                      n_copy_streams=args.streams, n_staging_slots=args.slots, compress=args.compress,
                      in_scan_pack=args.in_scan_pack,
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
    _barrier(pg)  # every rank probes at once: BW_d2h(N), BW_h2d(N)
    probes = probe_links(torch, ctx)
    _barrier(pg)
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
        v0 = time.perf_counter()
        if pg is not None:  # globally consistent cut: all-or-nothing lock vote over gloo (dist.py)
            st = gdist.lock_all(ctx)
            if st != 0:
                raise RuntimeError(f"lock vote failed: {st}")
        else:
            ctx.lock()
        lock_wall = time.perf_counter() - v0
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
        s["lock_wall_ns"] = int(lock_wall * 1e9)
        return e0.elapsed_time(e1) * 1e-3, h1 - h0, s_ck, s

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    _barrier(pg)
    launches0 = ctx.stats()["kernel_launches"]
    dev, host, recs, box = [], [], [], []
    with ClockSampler(local) as clk:
        _barrier(pg)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            _barrier(pg)
            b0 = time.perf_counter()
            d, h, sck, s = step(True)
            torch.cuda.synchronize()
            _barrier(pg)
            box.append(time.perf_counter() - b0)
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
    # f4 on: the same workload without the codec, measured in the same run (context for the headline)
    plain_cmp = None
    if args.compress and not incremental and not args.release and not args.storage:
        ctx2 = gcr.Context(local, page_size=w.page_size, chunk_bytes=args.chunk_mb << 20, n_copy_streams=args.streams,
                           n_staging_slots=args.slots, compress=0,
                           direct_min_bytes=(1 << 64) - 1 if args.direct_min_mb < 0 else int(args.direct_min_mb * (1 << 20)))
        for t in ts:
            ctx2.register_tensor(t)
        ctx2.reserve_host(R0 + (256 << 20))
        st2 = torch.cuda.ExternalStream(ctx2.stream())
        t2, ck2, rs2 = [], [], []
        for k in range(2 + 3):
            _barrier(pg)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(st2)
            ctx2.lock()
            im2 = ctx2.checkpoint()
            ctx2.restore([im2])
            ctx2.unlock()
            f1.record(st2)
            im2.free()
            f1.synchronize()
            if k >= 2:
                s2 = ctx2.stats()
                t2.append(f0.elapsed_time(f1) * 1e-3)
                ck2.append(s2["checkpoint_ns"] * 1e-9)
                rs2.append(s2["restore_ns"] * 1e-9)
        ctx2.close()
        tt2 = _max_over_ranks(pg, sum(t2))
        plain_cmp = {"value": round(_sum_over_ranks(pg, float(R)) * len(t2) / tt2 / 1e9, 3),
                     "ms_per_step": round(tt2 / len(t2) * 1e3, 3), "steps": len(t2),
                     "checkpoint_GBps": round(R * len(ck2) / sum(ck2) / 1e9, 3),
                     "restore_GBps": round(R * len(rs2) / sum(rs2) / 1e9, 3),
                     "what": "the same workload and launch configuration with compress=0 (raw PRESENT pages), "
                             "measured in this run after the headline steps"}
    t_dev = _max_over_ranks(pg, sum(dev))
    per_step = [_max_over_ranks(pg, d) for d in dev]  # spread of the timed steps
    step_ms = {"median": round(statistics.median(per_step) * 1e3, 3), "min": round(min(per_step) * 1e3, 3),
               "max": round(max(per_step) * 1e3, 3),
               "std": round(statistics.pstdev(per_step) * 1e3, 3) if len(per_step) > 1 else 0.0,
               "what": "device time of each timed step (CUDA events, max over ranks)"}
    t_host = _max_over_ranks(pg, sum(host))
    t_box = _max_over_ranks(pg, sum(box))
    lock_ms = sum(r[1]["lock_ns"] for r in recs) / len(recs) * 1e-6
    unlock_ms = sum(r[1]["unlock_ns"] for r in recs) / len(recs) * 1e-6
    vote_ms = sum(r[1]["lock_wall_ns"] - r[1]["lock_ns"] for r in recs) / len(recs) * 1e-6
    clocks_me = clk.summary()
    if pg is not None:
        allc = [None] * world
        pg.all_gather_object(allc, {"rank": rank, "gpu": local, **clocks_me, "numa": numa})
    else:
        allc = [{"rank": 0, "gpu": local, **clocks_me, "numa": numa}]
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
    if args.compress:  # f4: PRESENT pages go through the decode kernel (KD), K6/K7 only zero-fill
        scat_b = rs_last["pages_zero"] * w.page_size
    kern = {
        "K1_scan": {"dev_ms_per_step": scan_ns / K * 1e-6, "launches_per_step": scan_l / K,
                    "alg_bytes_per_step": R, "GBps": R * K / max(scan_ns, 1)},
        "K4_pack": None if args.compress else
        {"dev_ms_per_step": pack_ns / K * 1e-6, "alg_bytes_per_step": pack_b, "GBps": pack_b * K / max(pack_ns, 1)},
        "K6K7_scatter_zero": None if incremental else
        {"dev_ms_per_step": scat_ns / K * 1e-6, "alg_bytes_per_step": scat_b,
         "GBps": scat_b * K / max(scat_ns, 1), "note": "zero bytes counted as pages_zero x page_size (upper bound)"},
        "K8_verify": None if incremental else
        {"dev_ms_per_step": ver_ns / K * 1e-6, "alg_bytes_per_step": R, "GBps": R * K / max(ver_ns, 1)},
    }
    if args.compress:  # f4: KA + KC read every PRESENT byte, KC writes the stored form; KD the reverse
        raw_b = sc["present_raw_bytes"]
        cod_ns = sum(r[0]["codec_dev_ns"] for r in recs)
        dec_ns = sum(r[1]["decode_dev_ns"] for r in recs)
        kern["KABC_codec_encode"] = {"dev_ms_per_step": cod_ns / K * 1e-6, "alg_bytes_per_step": 2 * raw_b + img_b,
                                     "GBps": (2 * raw_b + img_b) * K / max(cod_ns, 1),
                                     "ratio_stored_over_raw": round(img_b / max(raw_b, 1), 4)}
        kern["KD_codec_decode"] = None if incremental else {
            "dev_ms_per_step": dec_ns / K * 1e-6, "alg_bytes_per_step": raw_b + img_b,
            "GBps": (raw_b + img_b) * K / max(dec_ns, 1)}
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
        "step_ms": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded counter-based generator; training-state-shaped fp32/bf16 values)",
        "config": {"workload": _workload_desc(args.config + ("i" if incremental and args.config == "C4" else ""), w),
                   "dirty_fraction": args.dirty if incremental else None, "registered_bytes_per_rank": R,
                   "allocations": len(w.allocs), "page_size": w.page_size, "chunk_bytes": args.chunk_mb << 20,
                   "compress": "f4 byte-plane dictionary code (R-19)" if args.compress else None,
                   "in_scan_pack": args.in_scan_pack,
                   "copy_streams": args.streams, "staging_slots": args.slots or args.streams, "direct_min_bytes": int(args.direct_min_mb * (1 << 20)) if args.direct_min_mb >= 0 else None,
                   "parallelism": f"independent ranks x{world} (gloo control plane)",
                   "l2": "inputs larger than L2 (registered state >> 126 MB; no flush needed)"},
        "per_gpu": {"checkpoint_GBps": round(ck_gbs, 3), "restore_GBps": round(rs_gbs, 3),
                    "roundtrip_GBps": round(R * K / t_dev / 1e9, 3),
                    "image_GBps_ckpt": round(img_b / ck / 1e9, 3)},
        "box": {"checkpoint_GBps": round(_sum_over_ranks(pg, ck_gbs), 3),
                "restore_GBps": round(_sum_over_ranks(pg, rs_gbs), 3),
                "barrier_to_barrier_GBps": round(R_all * K / t_box / 1e9, 3),
                "barrier_to_barrier_ms_per_step": round(t_box / K * 1e3, 3),
                "what": "sum over ranks of registered bytes / (gloo barrier -> step -> sync -> gloo barrier), max over ranks"},
        "phases_ms": {"lock": round(_max_over_ranks(pg, lock_ms), 4), "unlock": round(_max_over_ranks(pg, unlock_ms), 4),
                      "vote": round(_max_over_ranks(pg, vote_ms), 4) if pg is not None else None,
                      "what": "mean per step, max over ranks: gcr_lock / gcr_unlock host time; vote = lock_all wall "
                              "time minus the local lock (gloo all_reduce MIN), N > 1 only (paper: lock 240 ms, "
                              "unlock ~160 ms for GPT-2 S on H100, P:392-393)"},
        "link_roofline": {"drain_GBps": round(img_b / (sc["drain_ns"] * 1e-9) / 1e9, 2),
                          "d2h_probe_GBps": probes["pool_d2h_gbs"], "h2d_probe_GBps": probes["pool_h2d_gbs"],
                          "probe": "image pool itself (gcr_probe_link), all ranks probing at once",
                          "checkpoint_frac_of_d2h": round(ck_gbs / probes["pool_d2h_gbs"] * img_b / R, 3),
                          "restore_frac_of_h2d": round(rs_gbs / probes["pool_h2d_gbs"] * img_b / R, 3) if not incremental else None},
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
        "uncompressed": plain_cmp,
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
    sm = [c["sm_mhz"] for c in allc if c.get("sm_mhz")]
    result["clocks"] = {"sm_mhz": min(sm) if sm else None, "sm_max_mhz": clocks_me["sm_max_mhz"],
                        "reasons": sorted({r for c in allc for r in c["reasons"]}),
                        "samples": sum(c["samples"] for c in allc),
                        "per_rank": [{k: c[k] for k in ("rank", "gpu", "sm_mhz", "reasons", "samples")} for c in allc],
                        "what": "nvidia-smi during the timed region on every rank's GPU; sm_mhz = the lowest rank median"}
    result["placement"] = {"ranks": world, "gpus_visible": n_dev, "shared_gpus": world > n_dev,
                           "numa": [c["numa"] for c in allc]}
    if args.sub_c4_gib and not incremental and args.config == "C2":
        result["c4_incremental"] = c4_sub_record(args, torch, gcr, synth, local, pg)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if pg is not None:
        pg.destroy_process_group()


def c4_sub_record(args, torch, gcr, synth, dev, pg):
    """The balanced case of SURVEY §8(d) d.3 as a sub-record of the default line:
    C4-shaped state (1 GiB RANDOM allocations, --sub-c4-gib of them), a full
    checkpoint (untimed), then per step 1 % of the pages dirtied and an
    incremental checkpoint (lock -> checkpoint -> unlock) timed with CUDA events;
    reported against max(scan, drain) = the step's roofline."""
    w = synth.make_workload("C4", gib=args.sub_c4_gib)
    ts = w.materialize()
    torch.cuda.synchronize()
    ctx = gcr.Context(dev, page_size=w.page_size, compress=0, in_scan_pack=args.in_scan_pack)
    try:
        for t in ts:
            ctx.register_tensor(t)
        R = w.total_bytes
        ctx.reserve_host(R + (2 << 30))
        st = torch.cuda.ExternalStream(ctx.stream())
        ctx.lock()
        ctx.checkpoint().free()
        ctx.unlock()
        times, scans, imgs = [], [], []
        for k in range(3 + 5):
            muts = synth.dirty_mutations(w, 0.01, rng_seed=777 + k)
            synth.gpu_xor_batch([ts[a].data_ptr() + o for (a, o, x) in muts], [x for (a, o, x) in muts])
            torch.cuda.synchronize()
            _barrier(pg)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.lock()
            im = ctx.checkpoint(gcr.GCR_INCREMENTAL)
            ctx.unlock()
            e1.record(st)
            e1.synchronize()
            s = ctx.stats()
            if k >= 3:
                times.append(e0.elapsed_time(e1) * 1e-3)
                scans.append(s["scan_dev_ns"] * 1e-9)
                imgs.append(s["image_bytes"])
            im.free()
        d2h, _ = ctx.probe_link(1 << 30)
        t = _max_over_ranks(pg, sum(times) / len(times))
        scan = sum(scans) / len(scans)
        img = sum(imgs) / len(imgs)
        roof = max(R / (_peaks()["hbm_gbs"] * 1e9), img / (d2h * 1e9))
        return {"what": f"C4-shaped {args.sub_c4_gib} x 1 GiB, 1 % of pages dirty per step, incremental checkpoint "
                        f"(5 timed steps, 3 warm-up; in_scan_pack={args.in_scan_pack})",
                "registered_bytes": R, "ms_per_step": round(t * 1e3, 3), "GBps_registered": round(R / t / 1e9, 1),
                "scan_ms": round(scan * 1e3, 3), "image_bytes": int(img), "d2h_probe_GBps": round(d2h, 2),
                "roofline_ms": round(roof * 1e3, 3), "frac_of_roofline": round(roof / t, 3),
                "roofline": "max(R / MEASURED_PEAKS hbm_gbs, image bytes / pool D2H probe)"}
    finally:
        ctx.close()
        del ts
        torch.cuda.empty_cache()


def _workload_desc(name, w):
    return {"C1": "C1: 64 MiB region as 4 contiguous allocations, 25% zero pages, full checkpoint + restore",
            "C2": "C2: GPT-2 small training state, fp32 weights + Adam m/v (444 allocations), full checkpoint + restore",
            "C3": "C3: Llama-3 8B ZeRO-3 shard per rank (bf16 param/grad + fp32 master/m/v), full checkpoint + restore",
            "C4": f"C4: {len(w.allocs)} x 1 GiB per GPU, full checkpoint + restore",
            "C4i": f"C4: {len(w.allocs)} x 1 GiB per GPU, incremental checkpoint of a seeded dirty set per step",
            "C5": f"C5: {len(w.allocs)} GiB per GPU, 25% zero 2 MiB regions, full checkpoint + restore"}[name]


def _partition(sizes, T):
    """Allocations -> T groups, greedy by bytes (largest first onto the least
    loaded), order kept inside a group."""
    load, groups = [0] * T, [[] for _ in range(T)]
    for a in sorted(range(len(sizes)), key=lambda i: -sizes[i]):
        k = min(range(T), key=lambda j: load[j])
        groups[k].append(a)
        load[k] += sizes[a]
    return [sorted(g) for g in groups if g]


class OracleWorkload:
    """The oracle as it stands (oracle/gcr_oracle.c: plain C, single-threaded,
    Sarwate CRC) over the WHOLE workload: the allocations are partitioned over
    T threads, each running one unmodified oracle instance -- checkpoint into a
    canonical stream, then restore it into a poisoned copy with the full verify
    -- on its own registry (ctypes releases the GIL in the C calls).  Inputs
    come from the CPU twin of the generator, built once, untimed."""

    def __init__(self, w, threads: int):
        from oracle import oracle
        self.orc, self.P = oracle, w.page_size
        sizes = [s.nbytes for s in w.allocs]
        self.groups = _partition(sizes, max(1, threads))
        self.cont = [w.cpu_bytes(a) for a in range(len(sizes))]
        self.sizes = sizes
        self.bytes = sum(sizes)

    def _one(self, g):
        orc = self.orc
        reg = [(a + 1, 0x7F0000000000 + (a << 32), self.sizes[a]) for a in g]
        st, s = orc.checkpoint(self.P, reg, [self.cont[a] for a in g])
        tgt = [np.full(self.sizes[a], 0xA5, np.uint8) for a in g]
        st2, vf, _ = orc.restore([s], self.P, [self.sizes[a] for a in g], tgt)
        assert st == 0 and st2 == 0 and vf == 0

    def step(self):
        """One checkpoint + restore of every allocation; returns seconds."""
        import threading
        t0 = time.perf_counter()
        ths = [threading.Thread(target=self._one, args=(g,)) for g in self.groups]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return time.perf_counter() - t0

    def step_one_thread(self, budget_s):
        """The single-instance rate: groups one after another on one thread for ~budget_s."""
        t0, done = time.perf_counter(), 0
        for g in sorted(self.groups, key=len):
            self._one(g)
            done += sum(self.sizes[a] for a in g)
            if time.perf_counter() - t0 >= budget_s:
                break
        return done, time.perf_counter() - t0


def _host_threads():
    return max(1, min(len(os.sched_getaffinity(0)), 32))


def cpu_baseline(args, budget_s=15.0):
    """the oracle as it stands timed on this box's host cores
    (rank 0, N=1): one pass over the WHOLE workload on T threads (T = the
    cores this process may use), repeated within budget_s, plus the
    single-thread rate on part of it."""
    from paper_2502_16631_b200 import synth
    w = synth.make_workload(args.config, rank=0, page_size=args.page_size, gib=args.gib)
    T = _host_threads()
    ow = OracleWorkload(w, T)
    times = [ow.step()]
    while sum(times) < budget_s * 0.75:
        times.append(ow.step())
    done1, t1 = ow.step_one_thread(budget_s * 0.25)
    v = ow.bytes * len(times) / sum(times) / 1e9
    return {"value": round(v, 4), "unit": "GB/s", "cores": len(ow.groups), "kind": "oracle",
            "value_1thread": round(done1 / t1 / 1e9, 4),
            "sample": f"the whole {args.config} workload ({ow.bytes} B, {len(w.allocs)} allocations) partitioned "
                      f"over {len(ow.groups)} threads (one oracle instance each), checkpoint + restore with verify, "
                      f"x{len(times)}; value_1thread: {done1} B on one thread"}


def run_reference(args):
    """--impl reference: the CPU oracle on our arm's config, metric and unit
    (the paper ships no runnable code).  Never imports the product package's
    libgcr binding.  Under torchrun only rank 0 runs; the others exit 0."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2502_16631_b200 import synth  # the harness generator (no method arithmetic)
    w = synth.make_workload(args.config, rank=0, page_size=args.page_size, gib=args.gib)
    T = _host_threads()
    ow = OracleWorkload(w, T)
    for _ in range(args.warmup):
        ow.step()
    times = [ow.step() for _ in range(args.steps)]
    v = ow.bytes * len(times) / sum(times) / 1e9
    res = {"impl": "reference", "metric": "checkpoint & restore GB/s per GPU and box-aggregate at 1/2/4/8 B200 vs roofline",
           "value": round(v, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(sum(times) / len(times) * 1e3, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (seeded counter-based generator; the same bytes as our arm)",
           "config": {"workload": _workload_desc(args.config, w), "registered_bytes_per_rank": ow.bytes,
                      "allocations": len(w.allocs), "page_size": w.page_size, "same_config": True},
           "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": len(ow.groups), "kind": "oracle",
                            "sample": f"the whole {args.config} workload, {args.steps} steps of checkpoint + restore "
                                      f"with verify, {len(ow.groups)} threads (one oracle instance each)"},
           "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "the plain CPU oracle (oracle/gcr_oracle.c) as it stands; the paper ships no runnable code",
           "repo_libs_loaded": _repo_libs_loaded()}
    print(json.dumps(res), flush=True)


def _repo_libs_loaded():
    """Shared objects of this repo mapped into the process (evidence of which
    native code ran: the reference arm maps only oracle/liboracle.so)."""
    try:
        return sorted({os.path.relpath(l.split()[-1], ROOT) for l in open("/proc/self/maps")
                       if l.rstrip().endswith(".so") and l.split()[-1].startswith(ROOT)})
    except OSError:
        return None


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
    ap.add_argument("--sub-c4-gib", type=int, default=8,
                    help="default C2 line: add a C4-shaped 1 %% incremental sub-record of this many GiB (0 = off)")
    ap.add_argument("--in-scan-pack", type=int, default=0, choices=[0, 1, 2],
                    help="f1: 1 = incremental checkpoints written by the scan kernel itself, 0 = staged pipeline "
                         "(default: measured faster), 2 = every checkpoint")
    ap.add_argument("--compress", type=int, default=1, choices=[0, 1],
                    help="1: f4 page codec (PRESENT pages stored in byte-plane dictionary form, GPU encode/decode)")
    ap.add_argument("--dry-run", action="store_true", help="launch the ranks and report them; no GPU work")
    ap.add_argument("--storage", default=None, help="full mode: directory for the f3 storage tier round trip")
    ap.add_argument("--release", action="store_true",
                    help="full mode: state in releasable gcr_mem_alloc memory; each step releases the HBM after "
                         "the checkpoint and the restore re-maps the same addresses (SURVEY f2)")
    args = ap.parse_args()
    if args.storage and args.mode != "full":
        ap.error("--storage needs --mode full")
    if args.release and args.mode != "full":
        ap.error("--release needs --mode full (the restore re-maps the released memory)")
    if args.gib is None:
        args.gib = {"C4": 40, "C5": 16}.get(args.config, 16)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
