"""Full-size parity harness (TEST INFRASTRUCTURE, used by the -m gpu tests).

Compares a GPU image with the oracle for EVERY page of a BASELINE-sized
registry, without holding a second copy of the registry in host memory:

* The registry is cut into page-aligned SLICES (<= slice_bytes, never across an
  allocation).  Each slice's bytes come from the CPU twin of the generator
  (synth.py: the same seeded inputs the GPU was filled with; nothing read back
  from the device), and the unmodified oracle (`orc_checkpoint`, gcr_oracle.c)
  runs on the slice as a one-allocation registry whose vaddr is the slice's
  address.  Slices run in a thread pool (ctypes releases the GIL; one plain
  oracle instance per thread): the harness is parallel, the oracle is not.
* Why slicing is exact: a page's digest, zero test and
  class (steps 3-5) depend on that page's bytes and D_prev[g] only; the image
  data (step 6) is the concatenation in page order, so the whole image is the
  slices' data sections back to back; the pagemap (step 7) is the maximal runs
  of the per-page classes within each allocation, which this harness rebuilds
  from the oracle's per-page classes (runs split at slice borders are merged
  again; runs never cross allocations).
* Compared: every digest; every page's class; the whole pagemap, entry for
  entry; every PRESENT byte of the image at the oracle's offset (the slice's
  data is compared at the GPU pagemap's offset, and those offsets are then
  checked equal to the prefix sums of the oracle's slice data lengths); the
  96-byte header and the meta CRC (recomputed with the oracle's CRC over the
  rebuilt header || alloc table || pagemap || digests).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

PM_DT = np.dtype([("vaddr", "<u8"), ("nr_pages", "<u4"), ("flags", "<u4")])
AL_DT = np.dtype([("vaddr", "<u8"), ("bytes", "<u8"), ("alloc_id", "<u4"), ("reserved", "<u4")])
PE_PARENT, PE_PRESENT, PE_ZERO = 1, 4, 8


def _threads():
    return max(1, min(os.cpu_count() or 1, 32))


def page_lengths(sizes, P):
    """Per-page true length (c.1 step 2) and the first global page of each allocation."""
    m = np.array([(n + P - 1) // P for n in sizes], dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(m)])
    lens = np.full(int(starts[-1]), P, dtype=np.int64)
    for a, n in enumerate(sizes):
        lens[starts[a + 1] - 1] = n - (m[a] - 1) * P
    return lens, starts


def parse_stream(s: bytes, with_stored: bool = False):
    """Sections of a canonical stream as numpy views (layout only, DESIGN.md §3;
    f4 streams, header flags bit 1, carry a stored-length table)."""
    h = np.frombuffer(s, dtype=np.uint8, count=96)
    n_allocs = int(h[32:36].view(np.uint32)[0])
    flags = int(h[36:40].view(np.uint32)[0])
    n_pages = int(h[40:48].view(np.uint64)[0])
    n_present = int(h[48:56].view(np.uint64)[0])
    n_entries = int(h[72:80].view(np.uint64)[0])
    o = 96 + 24 * n_allocs
    pm = np.frombuffer(s, dtype=PM_DT, count=n_entries, offset=o)
    o += 16 * n_entries
    dg = np.frombuffer(s, dtype="<u4", count=n_pages, offset=o)
    o += 4 * n_pages
    st = None
    if flags & 2:
        st = np.frombuffer(s, dtype="<u4", count=n_present, offset=o)
        o += 4 * n_present
    data = np.frombuffer(s, dtype=np.uint8, offset=o)
    return (h, pm, dg, st, data) if with_stored else (h, pm, dg, data)


def expand_flags(pm, n_pages):
    f = np.repeat(pm["flags"].astype(np.uint32), pm["nr_pages"].astype(np.int64))
    assert f.size == n_pages, (f.size, n_pages)
    return f


def rebuild_pagemap(flags, sizes, vaddrs, P, starts):
    """c.1 step 7 from per-page flags: maximal runs of equal class inside each allocation."""
    out = []
    for a in range(len(sizes)):
        f = flags[starts[a]:starts[a + 1]]
        brk = np.flatnonzero(np.concatenate([[True], f[1:] != f[:-1]]))
        nr = np.diff(np.concatenate([brk, [f.size]]))
        e = np.zeros(brk.size, PM_DT)
        e["vaddr"] = np.uint64(vaddrs[a]) + brk.astype(np.uint64) * np.uint64(P)
        e["nr_pages"] = nr
        e["flags"] = f[brk]
        out.append(e)
    return np.concatenate(out) if out else np.zeros(0, PM_DT)


def slices_of(sizes, P, slice_bytes):
    pps = max(1, slice_bytes // P)
    out = []
    for a, n in enumerate(sizes):
        m = (n + P - 1) // P
        for p0 in range(0, m, pps):
            out.append((a, p0, min(m, p0 + pps)))
    return out


def check_image_full(orc, w, img, reg, mode=0, d_prev=None, generation=1, parent_generation=0,
                     slice_bytes=128 << 20, threads=None, compress=False):
    """Compare the GPU image `img` of workload `w` (registered as `reg` = [(alloc_id,
    vaddr, bytes)] in order) with the oracle, page by page.  Returns the oracle's
    digest table (the next incremental's D_prev)."""
    P = w.page_size
    sizes = [r[2] for r in reg]
    vaddrs = [r[1] for r in reg]
    lens, starts = page_lengths(sizes, P)
    n = int(starts[-1])
    hdr = img.header()
    gdig = img.digests()
    gpm = np.array(img.pagemap_array())
    gdata = img.data_view()
    assert hdr.n_pages == n == gdig.size
    assert int(gpm["nr_pages"].astype(np.int64).sum()) == n
    gflags = expand_flags(gpm, n)
    # GPU image offset of every page (used to locate a slice's data; verified below)
    present = gflags == PE_PRESENT
    if compress:  # f4: data offsets advance by each PRESENT page's stored length
        gst = img.stored()
        assert gst is not None and gst.size == int(present.sum()) == hdr.n_present
        per_page = np.zeros(n, np.int64)
        per_page[present] = gst
    else:
        assert img.stored() is None
        per_page = np.where(present, lens, 0)
    goff = np.concatenate([[0], np.cumsum(per_page)])
    assert goff[-1] == hdr.image_bytes == gdata.size
    tasks = slices_of(sizes, P, slice_bytes)
    exp_dig = np.empty(n, np.uint32)
    exp_flags = np.empty(n, np.uint32)
    exp_stored = np.zeros(n, np.int64)  # f4: the oracle's stored length of every PRESENT page
    data_len = np.zeros(len(tasks), np.int64)
    bad = []

    def work(k):
        a, p0, p1 = tasks[k]
        g0, g1 = int(starts[a]) + p0, int(starts[a]) + p1
        L = min(sizes[a], p1 * P) - p0 * P
        content = w.cpu_bytes(a, p0 * P, L)
        dp = None if mode == 0 else np.ascontiguousarray(d_prev[g0:g1], dtype=np.uint32)
        st, s = orc.checkpoint(P, [(reg[a][0], vaddrs[a] + p0 * P, L)], [content], mode=mode, d_prev=dp,
                               generation=generation, parent_generation=parent_generation, compress=compress)
        assert st == orc.OK, st
        del content
        _, pm, dg, sst, data = parse_stream(s, with_stored=True)
        exp_dig[g0:g1] = dg
        exp_flags[g0:g1] = expand_flags(pm, g1 - g0)
        if compress:
            exp_stored[g0:g1][exp_flags[g0:g1] == PE_PRESENT] = sst
        data_len[k] = data.size
        msg = []
        if not np.array_equal(dg, gdig[g0:g1]):
            i = int(np.flatnonzero(dg != gdig[g0:g1])[0])
            msg.append(f"digest of page {g0 + i} (alloc {a}) differs")
        o = int(goff[g0])
        if data.size and (o + data.size > gdata.size or not np.array_equal(data, gdata[o:o + data.size])):
            msg.append(f"image data of pages [{g0}, {g1}) (alloc {a}) differs")
        if msg:
            bad.append("; ".join(msg))

    with ThreadPoolExecutor(threads or _threads()) as ex:
        list(ex.map(work, range(len(tasks))))
    assert not bad, bad[:5]
    assert np.array_equal(exp_flags, gflags), f"class of page {int(np.flatnonzero(exp_flags != gflags)[0])} differs"
    if compress:
        assert np.array_equal(exp_stored[present], gst), "stored-length table differs"
    # the offsets used above are the oracle's: prefix sums of its slice data lengths
    cum = np.concatenate([[0], np.cumsum(data_len)])
    for k, (a, p0, _) in enumerate(tasks):
        assert cum[k] == goff[int(starts[a]) + p0], f"image offset of slice {k} differs"
    assert cum[-1] == hdr.image_bytes
    # the whole pagemap, entry for entry
    epm = rebuild_pagemap(exp_flags, sizes, vaddrs, P, starts)
    assert epm.size == gpm.size, (epm.size, gpm.size)
    assert np.array_equal(epm, gpm), "pagemap differs"
    # header + meta CRC rebuilt on the oracle side
    n_present = int((exp_flags == PE_PRESENT).sum())
    n_zero = int((exp_flags == PE_ZERO).sum())
    n_parent = int((exp_flags == PE_PARENT).sum())
    eh = np.zeros(96, np.uint8)
    eh[0:8] = np.frombuffer(b"GCRIMG\x00\x01", np.uint8)
    u32 = lambda o, v: eh[o:o + 4].view(np.uint32).__setitem__(0, v)  # noqa: E731
    u64 = lambda o, v: eh[o:o + 8].view(np.uint64).__setitem__(0, v)  # noqa: E731
    u32(8, 1)
    u32(12, P)
    u64(16, generation)
    u64(24, parent_generation if mode == 1 else 0)
    u32(32, len(reg))
    u32(36, (1 if mode == 1 else 0) | (2 if compress else 0))
    u64(40, n)
    u64(48, n_present)
    u64(56, n_zero)
    u64(64, n_parent)
    u64(72, epm.size)
    u64(80, int(cum[-1]))
    al = np.zeros(len(reg), AL_DT)
    al["vaddr"] = vaddrs
    al["bytes"] = sizes
    al["alloc_id"] = [r[0] for r in reg]
    parts = [eh, al.view(np.uint8), epm.view(np.uint8), exp_dig.view(np.uint8)]
    if compress:
        parts.append(exp_stored[exp_flags == PE_PRESENT].astype(np.uint32).view(np.uint8))
    meta = np.concatenate(parts)
    u32(88, orc.crc32c(meta))
    assert bytes(eh) == bytes(memoryview(hdr)), "header differs"
    return exp_dig


def check_memory_full(w, tensors, slice_bytes=128 << 20, threads=None):
    """Every byte of the registered tensors equals the CPU twin of the generator
    (zero ranges and mutations applied): a restore reproduced the state."""
    bad = []
    tasks = []
    for a, t in enumerate(tensors):
        n = t.numel()
        for o in range(0, n, slice_bytes):
            tasks.append((a, o, min(slice_bytes, n - o)))

    def work(task):
        a, o, L = task
        got = tensors[a][o:o + L].cpu().numpy()
        if not np.array_equal(got, w.cpu_bytes(a, o, L)):
            i = int(np.flatnonzero(got != w.cpu_bytes(a, o, L))[0])
            bad.append(f"alloc {a} byte {o + i}")

    with ThreadPoolExecutor(threads or min(_threads(), 16)) as ex:
        list(ex.map(work, tasks))
    assert not bad, bad[:5]
