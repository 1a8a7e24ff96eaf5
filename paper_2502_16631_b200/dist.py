"""Multi-rank control plane for a globally consistent snapshot.

PAPER.md §4.5: multi-GPU checkpointing requires "synchronizing the
state across all GPUs" -- the lock must be all-or-nothing, and P:160 rolls
everything back when the lock times out.  Each rank snapshots only its own HBM
(no data crosses NVLink); the ranks exchange only control words:

  C1  lock vote       all_reduce(MIN) of a 0/1 "locked" word; any failure
                      -> every locally-locked rank unlocks (rollback)
  C2  barrier         around checkpoint / restore (the consistent cut)
  C3  manifest gather ~64 B per rank to rank 0

All on a gloo (CPU/TCP) process group, so a wedged GPU cannot block the vote.
`ctx` is a paper_2502_16631_b200.gcr.Context (or any object with the same
try_lock / unlock / checkpoint / try_restore / stats methods).
"""
from __future__ import annotations

import time
from dataclasses import asdict, dataclass

GCR_OK, GCR_E_TIMEOUT, GCR_E_PEER, GCR_E_VERIFY = 0, 3, 4, 9


@dataclass
class Manifest:
    rank: int
    status: int
    generation: int
    n_pages: int
    image_bytes: int
    meta_crc32c: int
    checkpoint_ns: int


def _pg():
    import torch.distributed as dist
    return dist


def _vote(ok: bool, group=None) -> bool:
    """True iff every rank voted ok (all_reduce MIN over gloo)."""
    import torch
    dist = _pg()
    t = torch.tensor([1 if ok else 0], dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


def lock_all(ctx, group=None) -> int:
    """C1: lock on every rank or on none.  Returns GCR_OK, the local failure
    status, or GCR_E_PEER if only another rank failed (all rolled back)."""
    st = ctx.try_lock()
    if _vote(st == GCR_OK, group):
        return GCR_OK
    if st == GCR_OK:
        ctx.unlock()  # rollback: some peer did not lock within its timeout
        return GCR_E_PEER
    return st


def checkpoint_all(ctx, mode: int = 0, group=None):
    """C2 + C3: barrier, local checkpoint, outcome vote, manifest gather to
    rank 0.  All or nothing: if any rank failed, every rank whose checkpoint
    succeeded undoes it (gcr_checkpoint_abort: image freed, parent digest
    state and generation restored, phase back to LOCKED), so every rank is
    LOCKED exactly as before the attempt and a retry is legal everywhere.
    Returns (image or None, list of Manifest on rank 0 else None)."""
    dist = _pg()
    dist.barrier(group=group)
    t0 = time.perf_counter_ns()
    img, st = None, GCR_OK
    try:
        img = ctx.checkpoint(mode)
    except Exception as e:  # GcrError carries .status
        st = getattr(e, "status", -1)
    dt = time.perf_counter_ns() - t0
    ok = _vote(st == GCR_OK, group)
    h = img.header() if img is not None else None
    if not ok and img is not None:
        ctx.checkpoint_abort(img)
        img = None
    dist.barrier(group=group)
    man = Manifest(rank=dist.get_rank(), status=st if ok or st != GCR_OK else GCR_E_PEER,
                   generation=int(h.generation) if h else 0, n_pages=int(h.n_pages) if h else 0,
                   image_bytes=int(h.image_bytes) if h else 0, meta_crc32c=int(h.meta_crc32c) if h else 0,
                   checkpoint_ns=int(dt))
    gathered = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(asdict(man), gathered, dst=0, group=group)
    mans = [Manifest(**m) for m in gathered] if gathered is not None else None
    return (img if ok else None), mans


def restore_all(ctx, chain, group=None) -> int:
    """Barrier, local restore of this rank's chain, all-or-nothing outcome."""
    dist = _pg()
    dist.barrier(group=group)
    st = ctx.try_restore(chain)
    ok = _vote(st == GCR_OK, group)
    dist.barrier(group=group)
    if ok:
        return GCR_OK
    return st if st != GCR_OK else GCR_E_PEER


def release_all(ctx, group=None) -> int:
    """f2 on every rank after checkpoint_all: barrier, local gcr_release,
    outcome vote.  A release cannot be rolled back (the HBM is gone): ranks
    whose release succeeded stay RELEASED and leave it only through restore, so
    a failed vote is reported (GCR_E_PEER on the ranks that succeeded) for the
    caller to restore everywhere."""
    dist = _pg()
    dist.barrier(group=group)
    st = ctx.try_release()
    ok = _vote(st == GCR_OK, group)
    dist.barrier(group=group)
    if ok:
        return GCR_OK
    return st if st != GCR_OK else GCR_E_PEER


def unlock_all(ctx, group=None) -> int:
    """Unlock on every rank; every rank always reaches the vote (no rank is
    left blocked in a barrier when another one cannot unlock, e.g. while it is
    still RELEASED).  Returns GCR_OK, the local status, or GCR_E_PEER."""
    st = ctx.try_unlock()
    ok = _vote(st == GCR_OK, group)
    if ok:
        return GCR_OK
    return st if st != GCR_OK else GCR_E_PEER
