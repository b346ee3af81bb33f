"""Multi-GPU sharding of the block-parallel path, one process per GPU.

The paper's parallel version "splits the message into p parts and executes each part
into a different processor" (§5). Here the parts are contiguous ranges of
the fixed-size blocks: rank r of W owns global blocks [floor(r nb/W), floor((r+1) nb/W)).
Sub-keys depend only on the global block index, so the ciphertext is identical for
any W. Nothing crosses GPUs inside the hot loop; after the kernels:

* encrypt / verify: the 16-byte tag XORs of all ranks are all-gathered (NCCL has no
  XOR reduction) and XOR-ed locally, straight from the device result slot;
* decrypt / verify: the first failing block index is all-reduced with MIN;
* optionally the ciphertext slices are gathered to one rank with send/recv.

The compute engine is injected (``engine``) so the partition/combine logic can be
tested with the gloo backend on CPU; the product engine is :class:`CudaEngine`.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

NO_BAD = (1 << 63) - 1


def block_range(nb: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block range of `rank`."""
    return nb * rank // world, nb * (rank + 1) // world


@dataclass
class Slice:
    b0: int
    b1: int
    pt_off: int    # byte offset of the slice in the plaintext
    pt_bytes: int
    ct_off: int    # byte offset of the slice in the ciphertext
    ct_bytes: int


def slice_of(n: int, B: int, b0: int, b1: int) -> Slice:
    """Byte extents of blocks [b0,b1) of an n-byte message with block size B."""
    lo, hi = min(b0 * B, n), min(b1 * B, n)
    return Slice(b0, b1, lo, hi - lo, lo + 16 * b0, hi - lo + 16 * (b1 - b0))


def _all_gather(t: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out.view(world, -1)
    src = t.contiguous().cpu()  # gloo: stage through the host
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    return torch.stack(parts).to(t.device)


def xor_combine(tag16: torch.Tensor, group=None) -> torch.Tensor:
    """XOR of every rank's 16-byte tag (all-gather + local XOR)."""
    rows = _all_gather(tag16.view(torch.uint8)[:16], group)
    acc = rows[0].clone()
    for r in range(1, rows.shape[0]):
        acc ^= rows[r]
    return acc


def min_combine(first_bad: torch.Tensor, group=None) -> torch.Tensor:
    """Global minimum of the ranks' first failing block (NO_BAD when none failed)."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(first_bad, op=dist.ReduceOp.MIN, group=group)
        return first_bad
    h = first_bad.cpu()  # gloo: stage through the host
    dist.all_reduce(h, op=dist.ReduceOp.MIN, group=group)
    first_bad.copy_(h)
    return first_bad


class CudaEngine:
    """Per-rank engine over liblorenz.so's async calls; results stay on the device."""

    def __init__(self, key, n: int, device: torch.device):
        from . import lorenz as L
        self.L, self.key, self.n, self.device = L, key, n, device
        self.res = torch.empty(32, dtype=torch.uint8, device=device)

    def encrypt(self, b0, b1, pt, ct, stream=None) -> torch.Tensor:
        self.L.lorenz_result_init_async(self.res, stream)
        self.L.lorenz_encrypt_async(self.key, self.n, b0, b1, pt, ct, self.res, stream)
        return self.res[:16]

    def decrypt(self, b0, b1, ct, pt, stream=None) -> torch.Tensor:
        self.L.lorenz_result_init_async(self.res, stream)
        self.L.lorenz_decrypt_async(self.key, self.n, b0, b1, ct, pt, self.res, stream=stream)
        return self.first_bad()

    def verify(self, b0, b1, ct, stream=None) -> torch.Tensor:
        self.L.lorenz_result_init_async(self.res, stream)
        self.L.lorenz_verify_async(self.key, self.n, b0, b1, ct, self.res, stream)
        return self.first_bad()

    def first_bad(self) -> torch.Tensor:
        fb = self.res[16:24].view(torch.int64).clone()  # UINT64_MAX reads as -1
        return torch.where(fb < 0, torch.full_like(fb, NO_BAD), fb)


def sharded_encrypt(engine, b0: int, b1: int, pt_slice, ct_slice, group=None, stream=None) -> torch.Tensor:
    """Encrypt this rank's blocks, then combine the tag across ranks (16 B over NVLink)."""
    return xor_combine(engine.encrypt(b0, b1, pt_slice, ct_slice, stream), group)


def sharded_decrypt(engine, b0: int, b1: int, ct_slice, pt_slice, group=None, stream=None) -> int:
    """Decrypt this rank's blocks; returns the global first failing block or -1."""
    fb = min_combine(engine.decrypt(b0, b1, ct_slice, pt_slice, stream), group)
    v = int(fb.item())
    return -1 if v == NO_BAD else v


def gather_ciphertext(ct_slice: torch.Tensor, slices: list[Slice], dst: int = 0, group=None):
    """Optional gather of every rank's ciphertext slice to `dst` (unequal sizes: send/recv)."""
    rank = dist.get_rank(group)
    if rank != dst:
        dist.send(ct_slice, dst=dst, group=group)
        return None
    total = sum(s.ct_bytes for s in slices)
    out = torch.empty(total, dtype=torch.uint8, device=ct_slice.device)
    for r, s in enumerate(slices):
        view = out[s.ct_off - slices[0].ct_off: s.ct_off - slices[0].ct_off + s.ct_bytes]
        if r == dst:
            view.copy_(ct_slice)
        else:
            dist.recv(view, src=r, group=group)
    return out
