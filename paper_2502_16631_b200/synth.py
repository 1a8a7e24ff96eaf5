"""Seeded synthetic inputs (HARNESS; DESIGN.md §6 "input recipe").

Holds none of the snapshot method's arithmetic (no CRC, no classification, no
packing): only the counter-based generator that both sides of every parity
test draw their inputs from.  The CPU twin here (numpy) and the GPU fill in
libgcr_synth.so (include/gcr_synth.h) implement the same formula, so the bytes
are identical: tests/test_gpu_parity.py::test_gpu_generator_matches_cpu_twin
checks that on the GPU and tests/test_synth.py pins the CPU twin to a scalar
restatement of the formulas.

Word i (u64 LE) of an allocation with key k under seed s:
    r = splitmix64(s ^ (k << 40) ^ i), then shaped by `kind` (gcr_synth.h).

Workloads C1-C5 of BASELINE.json are built by `make_workload` with the shapes
of SURVEY.md §8(d) d.1 (GPT-2 small fp32 W+m+v; Llama-3 8B ZeRO shard; 40 x 1
GiB incremental; full-HBM sweep).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))

RANDOM, F32_WEIGHT, F32_CONST, ZERO, F32_M, F32_V, BF16_WEIGHT = range(7)
ONE_F32 = 0x3F800000


def seed_for(config_index: int, rank: int = 0) -> int:
    """Seed = 0xC0FFEE + 7919*config + 104729*rank."""
    return (0xC0FFEE + 7919 * config_index + 104729 * rank) & 0xFFFFFFFFFFFFFFFF


# ---------------------------------------------------------------------------
# CPU twin of the generator
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 of every element (a new array; in-place steps keep the
    full-size parity harness fast)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        t = z >> np.uint64(30)
        z ^= t
        z *= np.uint64(0xBF58476D1CE4E5B9)
        np.right_shift(z, np.uint64(27), out=t)
        z ^= t
        z *= np.uint64(0x94D049BB133111EB)
        np.right_shift(z, np.uint64(31), out=t)
        z ^= t
        return z


def _f32_inplace(b: np.ndarray, e0: int, sign: bool) -> None:
    """b (uint32, every 32-bit half of the words) <- sign(b) | (e0 + ((b>>23)&3)) << 23 | b & 0x7FFFFF."""
    t = b >> np.uint32(23)
    t &= np.uint32(3)
    t += np.uint32(e0)
    t <<= np.uint32(23)
    b &= np.uint32(0x807FFFFF if sign else 0x007FFFFF)
    b |= t


def gen_words(seed: int, key: int, start: int, n: int, kind: int, const_bits: int = 0) -> np.ndarray:
    """Words [start, start+n) of an allocation as uint64 (CPU)."""
    if kind == ZERO:
        return np.zeros(n, np.uint64)
    if kind == F32_CONST:
        c = np.uint64(const_bits | (const_bits << 32))
        return np.full(n, c, np.uint64)
    ctr = np.arange(start, start + n, dtype=np.uint64)
    ctr ^= np.uint64(seed ^ (key << 40))
    r = splitmix64(ctr)
    if kind == RANDOM:
        return r
    if kind in (F32_WEIGHT, F32_M, F32_V):
        e0, sg = {F32_WEIGHT: (118, True), F32_M: (113, True), F32_V: (103, False)}[kind]
        _f32_inplace(r.view(np.uint32), e0, sg)  # both halves of every LE word
        return r
    if kind == BF16_WEIGHT:
        h = r.view(np.uint16)  # the four 16-bit quarters of every LE word
        t = h >> np.uint16(7)
        t &= np.uint16(3)
        t += np.uint16(118)
        t <<= np.uint16(7)
        h &= np.uint16(0x807F)
        h |= t
        return r
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# GPU fill (libgcr_synth.so)
_slib = None


def synth_lib():
    global _slib
    if _slib is None:
        path = os.path.join(PKG, "libgcr_synth.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run __graft_entry__.build()")
        L = C.CDLL(path)
        L.gsy_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.gsy_xor_u32.argtypes = [C.c_uint64, C.c_uint32, C.c_void_p]
        L.gsy_xor_u32_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.gsy_flag_alloc.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.gsy_flag_set.argtypes = [C.c_uint64, C.c_uint32]
        L.gsy_flag_free.argtypes = [C.c_uint64]
        L.gsy_spin_until_flag.argtypes = [C.c_uint64, C.c_void_p]
        _slib = L
    return _slib


def gpu_fill(dptr: int, nbytes: int, seed: int, key: int, kind: int, const_bits: int = 0, stream: int = 0):
    rc = synth_lib().gsy_fill(dptr, nbytes, seed, key, kind, const_bits, C.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"gsy_fill failed: cuda error {rc}")


def gpu_xor_u32(dptr: int, x: int, stream: int = 0):
    rc = synth_lib().gsy_xor_u32(dptr, x & 0xFFFFFFFF, C.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"gsy_xor_u32 failed: cuda error {rc}")


def gpu_xor_batch(dptrs, xs, stream: int = 0):
    """Apply many XOR mutations with one kernel launch (harness)."""
    p = np.ascontiguousarray(dptrs, dtype=np.uint64)
    x = np.ascontiguousarray(np.asarray(xs, dtype=np.uint64).astype(np.uint32))
    rc = synth_lib().gsy_xor_u32_batch(p.ctypes.data, x.ctypes.data, p.size, C.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"gsy_xor_u32_batch failed: cuda error {rc}")


# ---------------------------------------------------------------------------
# Workloads
@dataclass
class AllocSpec:
    name: str
    nbytes: int
    kind: int
    const_bits: int = 0
    key: int = 0


@dataclass
class Workload:
    """Registry recipe: allocation specs, a seed, zeroed byte ranges and XOR
    mutations (alloc index, byte offset, u32 value), applied in that order."""
    name: str
    page_size: int
    seed: int
    allocs: list
    zero_ranges: list = field(default_factory=list)   # (alloc, offset, nbytes)
    mutations: list = field(default_factory=list)     # (alloc, offset, xor)
    contiguous: bool = False                          # C1: one region split in 4

    @property
    def total_bytes(self) -> int:
        return sum(a.nbytes for a in self.allocs)

    def cpu_bytes(self, a: int, offset: int = 0, nbytes: int | None = None) -> np.ndarray:
        """Bytes [offset, offset+nbytes) of allocation a as the generator
        produces them, with zero ranges and mutations applied (CPU)."""
        spec = self.allocs[a]
        if nbytes is None:
            nbytes = spec.nbytes - offset
        w0 = offset // 8
        w1 = (offset + nbytes + 7) // 8
        words = gen_words(self.seed, spec.key, w0, w1 - w0, spec.kind, spec.const_bits)
        out = words.view(np.uint8)[offset - 8 * w0: offset - 8 * w0 + nbytes].copy()
        for (za, zo, zn) in self.zero_ranges:
            if za != a:
                continue
            lo, hi = max(zo, offset), min(zo + zn, offset + nbytes)
            if lo < hi:
                out[lo - offset:hi - offset] = 0
        for (ma, mo, mx) in self.mutations:
            if ma != a or not (offset <= mo and mo + 4 <= offset + nbytes):
                continue
            v = out[mo - offset:mo - offset + 4].view(np.uint32)
            v ^= np.uint32(mx)
        return out

    def materialize(self, device="cuda", region=None):
        """Allocate device tensors (torch, plumbing only) and fill them with
        the GPU generator; returns the list of uint8 tensors.  `region`: a
        uint8 device tensor of total_bytes to carve the allocations from in
        order (e.g. releasable gcr_mem_alloc memory)."""
        import torch
        st = torch.cuda.current_stream().cuda_stream
        if self.contiguous or region is not None:
            if region is None:
                region = torch.empty(self.total_bytes, dtype=torch.uint8, device=device)
            assert region.numel() >= self.total_bytes
            ts, o = [], 0
            for s in self.allocs:
                ts.append(region[o:o + s.nbytes])
                o += s.nbytes
        else:
            ts = [torch.empty(s.nbytes, dtype=torch.uint8, device=device) for s in self.allocs]
        for t, s in zip(ts, self.allocs):
            gpu_fill(t.data_ptr(), s.nbytes, self.seed, s.key, s.kind, s.const_bits, st)
        self.apply_overlays(ts, self.zero_ranges, self.mutations)
        return ts

    @staticmethod
    def apply_overlays(ts, zero_ranges, mutations):
        import torch
        st = torch.cuda.current_stream().cuda_stream
        for (a, o, n) in zero_ranges:
            ts[a][o:o + n].zero_()
        if mutations:
            gpu_xor_batch([ts[a].data_ptr() + o for (a, o, x) in mutations], [x for (a, o, x) in mutations], st)


def gpt2_small_params():
    """GPT-2 small (124M): 148 tensors (V=50257, ctx 1024, d=768, 12 layers)."""
    d, V, T, L = 768, 50257, 1024, 12
    ps = [("wte", V * d, "w"), ("wpe", T * d, "w")]
    for i in range(L):
        ps += [(f"h{i}.ln_1.w", d, "g"), (f"h{i}.ln_1.b", d, "b"),
               (f"h{i}.attn.c_attn.w", d * 3 * d, "w"), (f"h{i}.attn.c_attn.b", 3 * d, "b"),
               (f"h{i}.attn.c_proj.w", d * d, "w"), (f"h{i}.attn.c_proj.b", d, "b"),
               (f"h{i}.ln_2.w", d, "g"), (f"h{i}.ln_2.b", d, "b"),
               (f"h{i}.mlp.c_fc.w", d * 4 * d, "w"), (f"h{i}.mlp.c_fc.b", 4 * d, "b"),
               (f"h{i}.mlp.c_proj.w", 4 * d * d, "w"), (f"h{i}.mlp.c_proj.b", d, "b")]
    ps += [("ln_f.w", d, "g"), ("ln_f.b", d, "b")]
    return ps


def make_workload(name: str, rank: int = 0, page_size: int | None = None, **kw) -> Workload:
    """BASELINE.json configs as concrete registries."""
    if name == "C1":
        P = page_size or 65536
        seed = seed_for(1, rank)
        allocs = [AllocSpec(f"region.{i}", 16 << 20, RANDOM, key=i) for i in range(4)]
        w = Workload("C1", P, seed, allocs, contiguous=True)
        rng = np.random.default_rng(seed)
        n_pages = (64 << 20) // P
        for z in sorted(rng.choice(n_pages, n_pages // 4, replace=False)):
            w.zero_ranges.append((int(z) * P // (16 << 20), int(z) * P % (16 << 20), P))
        return w
    if name == "C2":
        P = page_size or 65536
        seed = seed_for(2, rank)
        step0 = kw.get("step0", False)
        ps = gpt2_small_params()
        allocs, k = [], 0
        for (n, numel, role) in ps:
            kind, cb = {"w": (F32_WEIGHT, 0), "g": (F32_CONST, ONE_F32), "b": (ZERO, 0)}[role]
            allocs.append(AllocSpec(n, 4 * numel, kind, cb, key=k)); k += 1
        for st_name, kind in (("exp_avg", F32_M), ("exp_avg_sq", F32_V)):
            for (n, numel, role) in ps:
                allocs.append(AllocSpec(f"{n}.{st_name}", 4 * numel, ZERO if step0 else kind, key=k)); k += 1
        return Workload("C2", P, seed, allocs)
    if name == "C3":
        P = page_size or 65536
        seed = seed_for(3, rank)
        n = 1_003_782_656 if not kw.get("params_per_rank") else kw["params_per_rank"]
        step0 = kw.get("step0", False)
        allocs = [AllocSpec("param.bf16", 2 * n, BF16_WEIGHT, key=0),
                  AllocSpec("grad.bf16", 2 * n, ZERO if step0 else BF16_WEIGHT, key=1),
                  AllocSpec("master.fp32", 4 * n, F32_WEIGHT, key=2),
                  AllocSpec("exp_avg.fp32", 4 * n, ZERO if step0 else F32_M, key=3),
                  AllocSpec("exp_avg_sq.fp32", 4 * n, ZERO if step0 else F32_V, key=4)]
        return Workload("C3", P, seed, allocs)
    if name == "C4":
        P = page_size or 65536
        seed = seed_for(4, rank)
        gib = kw.get("gib", 40)
        allocs = [AllocSpec(f"state.{i}", 1 << 30, RANDOM, key=i) for i in range(gib)]
        return Workload("C4", P, seed, allocs)
    if name == "C5":
        P = page_size or 65536
        seed = seed_for(5, rank)
        gib = kw.get("gib", 16)
        allocs = [AllocSpec(f"hbm.{i}", 1 << 30, RANDOM, key=i) for i in range(gib)]
        w = Workload("C5", P, seed, allocs)
        rng = np.random.default_rng(seed)
        regions = gib * 512  # 2 MiB regions
        for z in sorted(rng.choice(regions, regions // 4, replace=False)):
            w.zero_ranges.append((int(z) // 512, (int(z) % 512) << 21, 2 << 20))
        return w
    raise ValueError(name)


def dirty_mutations(w: Workload, fraction: float, rng_seed: int, clustered: bool = False):
    """Pick exactly round(fraction * n_pages) pages and XOR one non-zero u32 in
    each.  Returns the mutation list (alloc, offset, xor)."""
    P = w.page_size
    pages = []
    for a, s in enumerate(w.allocs):
        m = (s.nbytes + P - 1) // P
        pages.append(m)
    n = sum(pages)
    k = int(round(fraction * n))
    rng = np.random.default_rng(rng_seed)
    if clustered:
        runs = max(1, k // 64)
        starts = rng.choice(max(1, n // 64), runs, replace=False) * 64
        pick = np.unique(np.concatenate([np.arange(s, min(n, s + 64)) for s in starts]))[:k]
    else:
        pick = np.sort(rng.choice(n, k, replace=False))
    cum = np.concatenate([[0], np.cumsum(pages)])
    muts = []
    for g in pick:
        a = int(np.searchsorted(cum, g, side="right") - 1)
        p = int(g - cum[a])
        ln = min(P, w.allocs[a].nbytes - p * P)
        off = p * P + 4 * int(rng.integers(0, ln // 4))
        muts.append((a, off, int(rng.integers(1, 1 << 32))))
    return muts
