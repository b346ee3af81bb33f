"""Multi-process (world_size 2 and 3) tests of the block partition and the combine
collectives of paper_1201_3114_b200.dist, on CPU with the gloo backend.

The per-rank compute engine here is the CPU oracle (test-only injection): what is
under test is the partition, the slice arithmetic, the tag XOR all-gather, the
first-bad MIN all-reduce and the ciphertext gather — the same code the NCCL run
uses on GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_IT = 5
B = 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleEngine:
    """Test-only engine with the CudaEngine interface, computing with the oracle."""

    def __init__(self, pw, n):
        import oracle
        self.o, self.pw, self.n = oracle, pw, n
        self.prm = oracle.params(mode=oracle.FAST, n_it=N_IT, block_size=B)
        self.fb = None

    def encrypt(self, b0, b1, pt, ct, stream=None):
        tag = np.zeros(16, dtype=np.uint8)
        off_p, off_c = 0, 0
        for b in range(b0, b1):
            ln = min(self.n, (b + 1) * B) - b * B
            blk = self.o.encrypt_block(self.pw, self.n, b, pt[off_p:off_p + ln].numpy(), self.prm)
            ct[off_c:off_c + ln + 16] = torch.from_numpy(blk)
            tag ^= blk[-16:]
            off_p += ln
            off_c += ln + 16
        return torch.from_numpy(tag)

    def decrypt(self, b0, b1, ct, pt, stream=None):
        from paper_1201_3114_b200.dist import NO_BAD
        first = NO_BAD
        off_p, off_c = 0, 0
        for b in range(b0, b1):
            ln = min(self.n, (b + 1) * B) - b * B
            km = self.o.keymaterial(self.o.subpassword(self.pw, b))
            rec, good = self.o.decrypt_stream(km, ct[off_c:off_c + ln + 16].numpy().tobytes(), self.prm)
            pt[off_p:off_p + ln] = torch.from_numpy(np.frombuffer(rec, np.uint8).copy()) if good else 0
            if not good and first == NO_BAD:
                first = b
            off_p += ln
            off_c += ln + 16
        return torch.tensor([first], dtype=torch.int64)


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1201_3114_b200 import dist as D
        from paper_1201_3114_b200 import inputs
        pw = inputs.password()
        nb = max(1, -(-n // B))
        b0, b1 = D.block_range(nb, rank, world)
        sl = D.slice_of(n, B, b0, b1)
        pt = torch.from_numpy(inputs.message(sl.pt_bytes, start=sl.pt_off).copy())
        ct = torch.zeros(sl.ct_bytes, dtype=torch.uint8)
        eng = OracleEngine(pw, n)
        tag = D.sharded_encrypt(eng, b0, b1, pt, ct)
        slices = [D.slice_of(n, B, *D.block_range(nb, r, world)) for r in range(world)]
        full = D.gather_ciphertext(ct, slices, dst=0)
        # decrypt with one flipped byte in the last rank's slice
        bad_block = slices[-1].b0 + (slices[-1].b1 - slices[-1].b0) // 2
        if rank == world - 1:
            ct[(bad_block - b0) * (B + 16) + 7] ^= 0x21
        back = torch.zeros(sl.pt_bytes, dtype=torch.uint8)
        fb = D.sharded_decrypt(eng, b0, b1, ct, back)
        intact = bool(torch.equal(back, pt)) if rank != world - 1 else None
        q.put((rank, tag.numpy().tobytes(), None if full is None else full.numpy().tobytes(), fb, intact,
               (b0, b1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 7 * B + 300), (3, 10 * B), (2, 1500)])
def test_sharded_encrypt_decrypt_gloo(ref, world, n):
    from paper_1201_3114_b200 import inputs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=180)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pw = inputs.password()
    msg = inputs.message(n)
    want_ct, want_tag = ref.encrypt(pw, msg, ref.params(mode=ref.FAST, n_it=N_IT, block_size=B))
    # every rank holds the same global tag; rank 0 gathered the whole ciphertext
    for r in range(world):
        assert res[r][1] == want_tag
    assert res[0][2] == want_ct.tobytes()
    # ranges tile [0, nb) contiguously
    nb = max(1, -(-n // B))
    spans = sorted(res[r][5] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == nb
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    # the tampered block (in the last rank) is reported to every rank; others intact
    last = spans[-1]
    bad_block = last[0] + (last[1] - last[0]) // 2
    for r in range(world):
        assert res[r][3] == bad_block
        if r != world - 1:
            assert res[r][4] is True


def test_block_range_partition_properties():
    from paper_1201_3114_b200 import dist as D
    for nb in [1, 2, 7, 1024, 1 << 20, (1 << 20) + 3]:
        for W in [1, 2, 3, 4, 8]:
            rs = [D.block_range(nb, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == nb
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            sizes = [b1 - b0 for b0, b1 in rs]
            assert max(sizes) - min(sizes) <= 1
    s = D.slice_of(5000, 1024, 2, 5)
    assert (s.pt_off, s.pt_bytes, s.ct_off, s.ct_bytes) == (2048, 5000 - 2048, 2048 + 32, 5000 - 2048 + 48)
