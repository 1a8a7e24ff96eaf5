"""Helpers shared by the -m gpu tests: run the CUDA path through the C-ABI and
the oracle on the same seeded inputs."""
import numpy as np


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def registry_of(ctx, tensors):
    """Register tensors in order; returns the oracle-side registry list."""
    reg = []
    for t in tensors:
        aid = ctx.register_tensor(t)
        reg.append((aid, t.data_ptr(), t.numel()))
    return reg


def host_copies(tensors):
    return [t.cpu().numpy().copy() for t in tensors]


def oracle_stream(orc, P, reg, contents, mode=0, d_prev=None, generation=1, parent_generation=0):
    st, s = orc.checkpoint(P, reg, contents, mode=mode, d_prev=d_prev, generation=generation,
                           parent_generation=parent_generation)
    assert st == orc.OK, st
    return s


def first_diff(a: bytes, b: bytes):
    if len(a) != len(b):
        return f"length {len(a)} != {len(b)}"
    x = np.frombuffer(a, np.uint8)
    y = np.frombuffer(b, np.uint8)
    idx = np.nonzero(x != y)[0]
    return None if idx.size == 0 else f"first differing byte {idx[0]} of {len(a)} ({idx.size} bytes differ)"
