"""B200-native device-memory snapshot engine (arXiv 2502.16631, CRIUgpu hot path).

Modules:
  gcr     ctypes binding of libgcr.so (the C-ABI in include/gcr.h)
  dist    multi-rank lock vote / barrier / manifest helpers (torch.distributed, gloo)
  synth   seeded synthetic inputs (harness; CPU twin of libgcr_synth.so)
  build   nvcc build of the in-tree .so files
"""
__all__ = ["gcr", "dist", "synth", "build"]
