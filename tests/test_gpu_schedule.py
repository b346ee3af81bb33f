"""GPU parity of the balanced (McNaughton) schedule of the chain kernel.

`lorenz_chain_seg_kernel` cuts the launch's 32-chain units at slot boundaries and hands the
32 chain states of a cut unit from one warp to another through global memory.
The library picks it for launches with >= 2 warps of chains per SM sub-partition; here
lorenz_set_tuning forces small slot counts so that small messages — ones the oracle checks
byte for byte — are cut at many places: unit boundaries, mid-window, the sentinel, a ragged
last block. Integer outputs, tolerance 0, against the oracle and against the wave kernel.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture
def sched(tune):
    """Set the schedule overrides for this test (lorenz_set_tuning; cleared afterwards)."""
    def set_(slots=None, mode=None):
        tune(seg_slots=slots, schedule=mode)
    return set_


def oparams(key):
    p = key.params
    return oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                         integrator=p.integrator, variant=p.variant)


def run_all(key, msg):
    n = len(msg)
    nb = key.num_blocks(n)
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.zeros(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag = L.lorenz_encrypt(key, n, 0, nb, pt, ct)
    return ct, tag


# (blocks, trailing bytes of a ragged last block, slots): units = ceil(blocks / 32)
CASES = [(160, 0, 3), (160, 0, 4), (161, 300, 3), (200, 1, 5), (257, 1023, 7), (96, 0, 2), (64, 17, 2),
         (33, 0, 2), (300, 512, 9)]


@pytest.mark.parametrize("blocks,tail,slots", CASES)
@pytest.mark.parametrize("integrator", [L.RK4, L.EULER, L.RK4_FMA])
def test_seg_matches_oracle(sched, blocks, tail, slots, integrator):
    sched(slots=slots)
    n = (blocks - (1 if tail else 0)) * 1024 + tail
    pw = inputs.password(seed=blocks * 31 + slots)
    msg = inputs.message(n, seed=blocks + tail)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=7, integrator=integrator)
    ct, tag = run_all(key, msg)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    got = ct.cpu().numpy()
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{len(bad)} bytes differ, first at {bad[0]} (block {bad[0] // 1040})")
    assert tag == want_tag
    nb = key.num_blocks(n)
    st, fb, vtag = L.lorenz_verify(key, n, 0, nb, ct)
    assert (st, fb, vtag) == (L.OK, -1, tag)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    ok = torch.zeros(nb, dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, nb, ct, back, block_ok=ok)
    assert (st, fb) == (L.OK, -1)
    assert np.array_equal(back.cpu().numpy(), msg)
    assert bool((ok == 1).all())


def test_seg_tamper_in_every_piece(sched):
    """Flips in the first piece, the second piece and the tag of cut units (and in a whole unit)
    are reported with the right block; every other block decrypts intact."""
    sched(slots=3)
    blocks = 160  # 5 units of 65 chunks over 3 slots: cuts at chunks 109 and 218
    n = blocks * 1024
    pw = inputs.password(seed=5)
    msg = inputs.message(n, seed=5)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=7)
    ct, _ = run_all(key, msg)
    clean = ct.clone()
    prm = oparams(key)
    # unit 1 (blocks 32..63) is cut at chunk 109 - 65 = 44 (char 704); unit 3 at chunk 218 - 195 = 23
    for blk, off in [(40, 100), (40, 900), (40, 1030), (100, 300), (100, 1039), (5, 512), (159, 1)]:
        ct.copy_(clean)
        pos = blk * 1040 + off
        ct[pos] ^= 0x40
        st, fb, _ = L.lorenz_verify(key, n, 0, blocks, ct)
        assert (st, fb) == (L.E_INTEGRITY, blk)
        back = torch.full((n,), 7, dtype=torch.uint8, device=DEV)
        ok = torch.zeros(blocks, dtype=torch.uint8, device=DEV)
        st, fb = L.lorenz_decrypt(key, n, 0, blocks, ct, back, block_ok=ok)
        assert (st, fb) == (L.E_INTEGRITY, blk)
        okh = ok.cpu().numpy()
        assert okh[blk] == 0 and okh.sum() == blocks - 1
        got = back.cpu().numpy()
        assert not got[blk * 1024:(blk + 1) * 1024].any()
        mask = np.ones(n, dtype=bool)
        mask[blk * 1024:(blk + 1) * 1024] = False
        assert np.array_equal(got[mask], msg[mask])
        ost, _, ofb, ook = oracle.decrypt(pw, ct.cpu().numpy(), prm, per_block=True)
        assert ofb == blk and np.array_equal(ook, okh)


@pytest.mark.parametrize("slots", [2, 3, 11])
def test_seg_block_range_slice(sched, slots):
    """A rank's slice [b0, b1) of a larger message through the cut schedule."""
    sched(slots=slots)
    n = 400 * 1024 + 77
    pw = inputs.password(seed=9)
    msg = inputs.message(n, seed=9)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=5)
    b0, b1 = 37, 401
    pt = torch.from_numpy(msg[b0 * 1024:]).to(DEV)
    ct = torch.zeros(key.ct_len(n) - b0 * 1040, dtype=torch.uint8, device=DEV)
    tag = L.lorenz_encrypt(key, n, b0, b1, pt, ct)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key), b0=b0, b1=b1)
    assert np.array_equal(ct.cpu().numpy(), want[b0 * 1040:])
    assert tag == want_tag


@pytest.mark.parametrize("variant", [1, 2, 4, 5])
def test_seg_step3_variants(sched, variant):
    sched(slots=4)
    n = 190 * 1024 + 5
    pw = inputs.password(seed=variant)
    msg = inputs.message(n, seed=variant)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=6, variant=variant)
    ct, tag = run_all(key, msg)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    assert np.array_equal(ct.cpu().numpy(), want) and tag == want_tag


def test_seg_batch_and_ragged(sched):
    """lorenz_encrypt_batch (C5 shape) and ragged batches through the cut schedule."""
    sched(slots=5)
    S, n = 6, 50 * 1024 + 48  # the batch call needs n % 16 == 0
    pws = [inputs.password(seed=100 + s) for s in range(S)]
    keys = [L.lorenz_keysetup(pw, mode=L.FAST, n_it=5) for pw in pws]
    msgs = [inputs.message(n, seed=200 + s) for s in range(S)]
    pts = torch.from_numpy(np.concatenate(msgs)).to(DEV)
    cl = keys[0].ct_len(n)
    cts = torch.zeros(S * cl, dtype=torch.uint8, device=DEV)
    tags = torch.zeros(16 * S, dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt_batch(keys, n, pts, cts, tags)
    prm = oparams(keys[0])
    for s in range(S):
        want, want_tag = oracle.encrypt(pws[s], msgs[s], prm)
        assert np.array_equal(cts[s * cl:(s + 1) * cl].cpu().numpy(), want)
        assert tags[16 * s:16 * s + 16].cpu().numpy().tobytes() == want_tag

    lengths = [33 * 1024, 5, 0, 70 * 1024 + 100, 1024, 40 * 1024 - 1]
    up = lambda x: (x + 15) // 16 * 16
    pt_off, ct_off, p, c = [], [], 0, 0
    for m in lengths:
        pt_off.append(p)
        ct_off.append(c)
        p += up(m)
        c += up(keys[0].ct_len(m))
    host = np.zeros(p, dtype=np.uint8)
    rmsgs = []
    for s, m in enumerate(lengths):
        rmsgs.append(inputs.message(m, seed=300 + s))
        host[pt_off[s]:pt_off[s] + m] = rmsgs[-1]
    rpts = torch.from_numpy(host).to(DEV)
    rcts = torch.zeros(c, dtype=torch.uint8, device=DEV)
    rtags = torch.zeros(16 * len(lengths), dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt_ragged(keys, lengths, pt_off, ct_off, rpts, rcts, rtags)
    rh = rcts.cpu().numpy()
    for s, m in enumerate(lengths):
        want, want_tag = oracle.encrypt(pws[s], rmsgs[s], prm)
        assert np.array_equal(rh[ct_off[s]:ct_off[s] + len(want)], want), f"message {s}"
        assert rtags[16 * s:16 * s + 16].cpu().numpy().tobytes() == want_tag
    back = torch.zeros_like(rpts)
    st, fb = L.lorenz_decrypt_ragged(keys, lengths, ct_off, pt_off, rcts, back, torch.empty_like(rtags))
    assert st == L.OK and fb == [-1] * len(lengths)
    assert torch.equal(back, rpts)


@pytest.mark.parametrize("mib", [64, 150])
def test_seg_default_equals_wave(sched, mib):
    """At sizes where the library picks the cut schedule by itself (C3: 2,048 units over 1,184
    slots; 150 MiB: 4,800 units over 2,368), its ciphertext, tag and verdicts equal the wave
    kernel's, and sampled blocks equal the oracle's."""
    n = mib << 20
    pw = inputs.password()
    msg = inputs.message(n, seed=mib)
    key = L.lorenz_keysetup(pw, mode=L.FAST)
    pt = torch.from_numpy(msg).to(DEV)
    nb = key.num_blocks(n)
    sched()
    ct_seg = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag_seg = L.lorenz_encrypt(key, n, 0, nb, pt, ct_seg)
    sched(mode="wave")
    ct_wave = torch.empty_like(ct_seg)
    tag_wave = L.lorenz_encrypt(key, n, 0, nb, pt, ct_wave)
    assert tag_seg == tag_wave
    assert torch.equal(ct_seg, ct_wave)
    sched()
    st, fb, vtag = L.lorenz_verify(key, n, 0, nb, ct_seg)
    assert (st, fb, vtag) == (L.OK, -1, tag_seg)
    prm = oparams(key)
    rng = np.random.default_rng(mib)
    for b in [0, nb - 1] + [int(x) for x in rng.integers(0, nb, 6)]:
        want = oracle.encrypt_block(pw, n, b, msg[b * 1024:(b + 1) * 1024], prm)
        assert np.array_equal(ct_seg[b * 1040:(b + 1) * 1040].cpu().numpy(), want), f"block {b}"


def test_seg_async_calls_capture_into_a_cuda_graph(sched):
    """The balanced launch (scratch from the stream-ordered pool, a memset, the kernel, the free)
    captures into a CUDA graph; replays re-zero the ticket and flags and stay bit-exact."""
    sched(slots=5, mode="seg")
    pw = inputs.password(seed=17)
    n = 200 * 1024 + 3
    msg = inputs.message(n, seed=17)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=5)
    nb = key.num_blocks(n)
    assert L.lorenz_launch_plan(key, n, 0, nb)["kind"] == "balanced"
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    res = torch.empty(64, dtype=torch.uint8, device=DEV)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.lorenz_result_init_async(res[:32], stream=s)
        L.lorenz_encrypt_async(key, n, 0, nb, pt, ct, res[:32], stream=s)
        L.lorenz_result_init_async(res[32:], stream=s)
        L.lorenz_decrypt_async(key, n, 0, nb, ct, back, res[32:], stream=s)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    for _ in range(3):
        ct.zero_()
        back.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(ct.cpu().numpy(), want)
        r = res.cpu().numpy()
        assert r[:16].tobytes() == want_tag
        assert int(r[48:56].view(np.uint64)[0]) == 2 ** 64 - 1
        assert torch.equal(back, pt)


@pytest.mark.timeout(300)
def test_seg_concurrent_launches_with_a_full_gpu_kernel(sched):
    """Balanced launches from several host threads on their own streams while a long wave
    kernel holds every SM: CTAs of one balanced launch start at different times and some wait
    for SM space, but a warp only waits on slots that started before it (start-order tickets),
    so every launch completes, bit-exact."""
    import threading
    sched(slots=37, mode="seg")
    big_n = 37888 * 1024  # exactly 2 warps per SM sub-partition: the library's wave kernel
    big_key = L.lorenz_keysetup(inputs.password(seed=1), mode=L.FAST, n_it=100)
    big_pt = torch.from_numpy(inputs.message(big_n, seed=1)).to(DEV)
    big_ct = torch.empty(big_key.ct_len(big_n), dtype=torch.uint8, device=DEV)
    cases = []
    for t in range(4):
        pw = inputs.password(seed=300 + t)
        n = 50 * 32 * 1024 - 77 * t  # 50 units over 37 slots
        cases.append((pw, L.lorenz_keysetup(pw, mode=L.FAST, n_it=9), inputs.message(n, seed=400 + t)))
    out, errors = [None] * len(cases), []

    def work(i):
        try:
            pw, key, msg = cases[i]
            n = len(msg)
            st = torch.cuda.Stream(device=DEV)
            with torch.cuda.stream(st):
                pt = torch.from_numpy(msg).to(DEV)
                ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
                tag = L.lorenz_encrypt(key, n, 0, key.num_blocks(n), pt, ct, stream=st)
                out[i] = (ct.cpu().numpy(), tag)
        except Exception as e:
            errors.append(f"thread {i}: {e!r}")

    bs = torch.cuda.Stream(device=DEV)
    sched(mode="wave")  # the long kernel: every SM busy for ~16 ms
    big_plan = L.lorenz_launch_plan(big_key, big_n, 0, big_key.num_blocks(big_n))
    with torch.cuda.stream(bs):
        res = torch.empty(32, dtype=torch.uint8, device=DEV)
        L.lorenz_result_init_async(res, stream=bs)
        L.lorenz_encrypt_async(big_key, big_n, 0, big_key.num_blocks(big_n), big_pt, big_ct, res, stream=bs)
    sched(slots=37, mode="seg")
    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    bs.synchronize()
    assert not errors, errors
    assert big_plan["kind"] == "wave" and big_plan["grid"] * big_plan["cta"] >= 37888
    for (pw, key, msg), (ct, tag) in zip(cases, out):
        want, want_tag = oracle.encrypt(pw, msg, oparams(key))
        assert np.array_equal(ct, want) and tag == want_tag


@pytest.mark.parametrize("blocks,skew", [(40000, 8), (56000, 30), (65536, 60), (100000, 15), (140000, 120)])
def test_seg_skewed_slots_equal_wave(sched, tune, blocks, skew):
    """Skewed slot capacities (later warp groups of a CTA get more chunks) at default slot
    layouts, including skews far above the tuned 8 per mille: ciphertext, tag and verdicts equal
    the wave kernel's, and sampled blocks equal the oracle's."""
    n = blocks * 1024 - 333
    pw = inputs.password(seed=blocks)
    msg = inputs.message(n, seed=skew)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=3)
    nb = key.num_blocks(n)
    pt = torch.from_numpy(msg).to(DEV)
    tune(seg_skew=skew)
    sched(mode="seg")
    p = L.lorenz_launch_plan(key, n, 0, nb)
    assert p["kind"] == "balanced"
    ct_seg = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag_seg = L.lorenz_encrypt(key, n, 0, nb, pt, ct_seg)
    st, fb, _ = L.lorenz_verify(key, n, 0, nb, ct_seg)
    assert (st, fb) == (L.OK, -1)
    sched(mode="wave")
    ct_wave = torch.empty_like(ct_seg)
    assert L.lorenz_encrypt(key, n, 0, nb, pt, ct_wave) == tag_seg
    assert torch.equal(ct_seg, ct_wave)
    prm = oparams(key)
    for b in [0, nb - 1, nb // 2]:
        blk = msg[b * 1024:(b + 1) * 1024]
        want = oracle.encrypt_block(pw, n, b, blk, prm)
        assert np.array_equal(ct_seg[b * 1040:b * 1040 + len(want)].cpu().numpy(), want), f"block {b}"


def test_seg_default_tamper_zero_fills_whole_slice(sched):
    """At a size where the library itself picks the balanced kernel, a flipped byte (in a unit
    the schedule cuts) is reported with its block by verify and decrypt; decrypt without
    per-block verdicts zero-fills the whole slice, with them only the failing block."""
    sched()
    blocks = 70000
    n = blocks * 1024
    pw = inputs.password(seed=70)
    msg = inputs.message(n, seed=70)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=2)
    p = L.lorenz_launch_plan(key, n, 0, blocks)
    assert p["kind"] == "balanced"
    ct, _ = run_all(key, msg)
    # a block in the unit cut by the boundary between the first two positions of the chunk line
    cut_unit = p["chunks_per_slot"] // 65
    bad_block = 32 * cut_unit + 17
    ct[bad_block * 1040 + 1000] ^= 1
    st, fb, _ = L.lorenz_verify(key, n, 0, blocks, ct)
    assert (st, fb) == (L.E_INTEGRITY, bad_block)
    back = torch.full((n,), 9, dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, blocks, ct, back)
    assert (st, fb) == (L.E_INTEGRITY, bad_block)
    assert int(back.count_nonzero()) == 0
    ok = torch.zeros(blocks, dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, blocks, ct, back, block_ok=ok)
    assert (st, fb) == (L.E_INTEGRITY, bad_block)
    assert int(ok.sum()) == blocks - 1 and int(ok[bad_block]) == 0
    got = back.cpu().numpy()
    assert not got[bad_block * 1024:(bad_block + 1) * 1024].any()
    assert np.array_equal(got[:bad_block * 1024], msg[:bad_block * 1024])
    assert np.array_equal(got[(bad_block + 1) * 1024:], msg[(bad_block + 1) * 1024:])
