"""B200-native hot path of arXiv 1201.3114's parallel Lorenz-attractor cipher.

The product is the C-ABI library ``csrc/liblorenz.so`` (CUDA, sm_100a) declared in
``include/lorenz.h``; :mod:`paper_1201_3114_b200.lorenz` is its thin ctypes binding
and :mod:`paper_1201_3114_b200.dist` the multi-GPU sharding over torch.distributed.
Nothing in this package imports the CPU oracle; with no CUDA library the binding
raises instead of falling back.
"""
__all__ = ["lorenz", "dist", "inputs"]
