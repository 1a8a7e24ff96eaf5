"""CPU, world_size 2 over gloo: the multi-rank control plane:
the lock vote is all-or-nothing with rollback (P:160 applied box-wide),
checkpoints are bracketed by barriers and manifests reach rank 0."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeHeader:
    def __init__(self, gen, npages, nbytes):
        self.generation, self.n_pages, self.image_bytes, self.meta_crc32c = gen, npages, nbytes, 0xABCD


class FakeImage:
    def __init__(self, h):
        self.h = h

    def header(self):
        return self.h


class FakeCtx:
    """Phase machine of include/gcr.h without a GPU (RUNNING/LOCKED/CHECKPOINTED)."""

    def __init__(self, rank, lock_status=0, restore_status=0, nbytes=1000, release_status=0, ckpt_fail_once=0):
        self.rank, self.lock_status, self.restore_status, self.nbytes = rank, lock_status, restore_status, nbytes
        self.release_status = release_status
        self.ckpt_fail_once = ckpt_fail_once
        self.phase, self.gen, self.log = 0, 0, []
        self.last = None

    def try_lock(self):
        self.log.append("lock")
        if self.lock_status == 0:
            assert self.phase == 0
            self.phase = 1
        return self.lock_status

    def unlock(self):
        self.log.append("unlock")
        assert self.phase in (1, 2)
        self.phase = 0

    def try_unlock(self):
        if self.phase not in (1, 2):
            return 2  # GCR_E_STATE (e.g. still RELEASED)
        self.unlock()
        return 0

    def checkpoint(self, mode=0):
        assert self.phase == 1
        if self.ckpt_fail_once:
            st, self.ckpt_fail_once = self.ckpt_fail_once, 0
            self.log.append("checkpoint_failed")
            e = RuntimeError("injected")
            e.status = st
            raise e
        self.gen += 1
        self.phase = 2
        self.last = FakeImage(FakeHeader(self.gen, 10, self.nbytes * (self.rank + 1)))
        return self.last

    def checkpoint_abort(self, img):  # CHECKPOINTED -> LOCKED, generation re-issued
        assert self.phase == 2 and img is self.last
        self.log.append("abort")
        self.gen -= 1
        self.phase = 1
        self.last = None

    def try_restore(self, chain):
        assert self.phase in (1, 2, 3)
        self.phase = 1
        return self.restore_status

    def try_release(self):  # f2: CHECKPOINTED -> RELEASED (3)
        self.log.append("release")
        assert self.phase == 2
        if self.release_status == 0:
            self.phase = 3
        return self.release_status


def _worker(rank, world, port, scenario, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2502_16631_b200 import dist as gd
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if scenario == "ok":
            ctx = FakeCtx(rank)
            st = gd.lock_all(ctx)
            img, mans = gd.checkpoint_all(ctx)
            rs = gd.restore_all(ctx, [img])
            gd.unlock_all(ctx)
            q.put((rank, st, img is not None, mans and [(m.rank, m.image_bytes, m.generation) for m in mans], rs,
                   ctx.phase, ctx.log))
        elif scenario == "timeout_on_1":
            ctx = FakeCtx(rank, lock_status=3 if rank == 1 else 0)
            st = gd.lock_all(ctx)
            q.put((rank, st, ctx.phase, ctx.log))
        elif scenario == "release":
            ctx = FakeCtx(rank, release_status=2 if (rank == 1 and world == 3) else 0)
            gd.lock_all(ctx)
            img, _ = gd.checkpoint_all(ctx)
            rl = gd.release_all(ctx)
            ph = ctx.phase
            rs = gd.restore_all(ctx, [img])  # the only way out of RELEASED, everywhere
            gd.unlock_all(ctx)
            q.put((rank, rl, ph, rs, ctx.phase, ctx.log))
        elif scenario == "ckpt_fail_on_1":
            ctx = FakeCtx(rank, ckpt_fail_once=11 if rank == 1 else 0)
            gd.lock_all(ctx)
            img, mans = gd.checkpoint_all(ctx)
            first = (img is None, ctx.phase, ctx.gen, mans and [(m.rank, m.status) for m in mans])
            img2, mans2 = gd.checkpoint_all(ctx)  # a retry is legal on every rank
            second = (img2 is not None, ctx.phase, img2.header().generation if img2 else None)
            un = gd.unlock_all(ctx)
            q.put((rank, first, second, un, ctx.log))
        elif scenario == "unlock_while_released_on_1":
            ctx = FakeCtx(rank)
            gd.lock_all(ctx)
            gd.checkpoint_all(ctx)
            if rank == 1:
                ctx.phase = 3  # RELEASED: unlock is not legal there
            un = gd.unlock_all(ctx)  # must not leave rank 0 blocked in a barrier
            q.put((rank, un, ctx.phase))
        elif scenario == "verify_on_0":
            ctx = FakeCtx(rank, restore_status=9 if rank == 0 else 0)
            gd.lock_all(ctx)
            img, _ = gd.checkpoint_all(ctx)
            rs = gd.restore_all(ctx, [img])
            q.put((rank, rs))
    finally:
        dist.destroy_process_group()


def _run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_consistent_checkpoint_and_manifest_gather():
    out = _run("ok")
    r0, r1 = out
    assert r0[1] == r1[1] == 0 and r0[2] and r1[2]
    assert r0[3] == [(0, 1000, 1), (1, 2000, 1)]   # rank 0 gathered both manifests
    assert r1[3] is None
    assert r0[4] == r1[4] == 0 and r0[5] == r1[5] == 0
    assert r0[6] == ["lock", "unlock"]


def test_lock_timeout_on_one_rank_rolls_back_every_rank():
    out = _run("timeout_on_1")
    (r0, st0, ph0, log0), (r1, st1, ph1, log1) = out
    assert st1 == 3 and st0 == 4           # local TIMEOUT, peer sees E_PEER
    assert ph0 == ph1 == 0                 # both RUNNING: nothing stays locked
    assert log0 == ["lock", "unlock"]      # rank 0 rolled back its successful lock
    assert log1 == ["lock"]


def test_restore_failure_on_one_rank_is_reported_everywhere():
    out = _run("verify_on_0")
    assert out == [(0, 9), (1, 4)]


def test_release_all_then_restore_all():
    out = _run("release")
    for rank, rl, ph, rs, ph_end, log in out:
        assert rl == 0 and ph == 3 and rs == 0 and ph_end == 0
        assert log == ["lock", "release", "unlock"]


def test_release_failure_on_one_rank_is_reported_everywhere():
    out = _run("release", world=3)
    assert [(r, rl, ph) for r, rl, ph, *_ in out] == [(0, 4, 3), (1, 2, 2), (2, 4, 3)]
    assert all(rs == 0 and ph_end == 0 for _, _, _, rs, ph_end, _ in out)


def test_checkpoint_failure_on_one_rank_is_all_or_nothing():
    """A failed checkpoint on rank 1: rank 0 undoes its successful one
    (checkpoint_abort), both stay LOCKED with the old generation, and a retry
    of checkpoint_all then succeeds everywhere with the SAME generation."""
    out = _run("ckpt_fail_on_1")
    (r0, f0, s0, u0, log0), (r1, f1, s1, u1, log1) = out
    assert f0[:3] == (True, 1, 0) and f1[:3] == (True, 1, 0)
    assert f0[3] == [(0, 4), (1, 11)]      # rank 0's manifest: peer failure / local failure
    assert s0 == (True, 2, 1) and s1 == (True, 2, 1)
    assert u0 == u1 == 0
    assert log0 == ["lock", "abort", "unlock"]
    assert log1 == ["lock", "checkpoint_failed", "unlock"]


def test_unlock_all_never_blocks_on_a_refusing_rank():
    out = _run("unlock_while_released_on_1")
    assert out == [(0, 4, 0), (1, 2, 3)]
