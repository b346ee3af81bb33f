"""C5 on the GPU: the batched sensitivity sweep against the oracle (ciphertexts, exact) and
its integer statistics recomputed on the host from the GPU ciphertexts (exact)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import lorenz as L
from paper_1201_3114_b200 import sweep

pytestmark = pytest.mark.gpu


def _host_stats(ct, pt, spans, lsb_spans):
    def cmp(a, b, s):
        x = a[s[0]:s[0] + s[2]]
        y = b[s[1]:s[1] + s[2]]
        d = x ^ y
        return (int(np.unpackbits(d).sum()), int((d != 0).sum()), int(((d & 1) == 0).sum()))
    co = np.array([cmp(ct, ct, s) for s in spans])
    lo = np.array([cmp(ct, pt, s) for s in lsb_spans])
    return co, lo


def test_c5_sweep_small_exact():
    n, n_it, T = 64 * 1024, 20, 6
    r = sweep.run(T, n=n, batch=4, n_it=n_it, keep_ciphertexts=True)
    ctl = n + 16 * (n // 1024)
    prm = oracle.params(mode=oracle.FAST, n_it=n_it, block_size=1024)
    for b_start, (ct, pt, co, hi, lo, spans, lsb_spans) in r["kept"].items():
        Tb = len(spans) // 4
        for i in range(Tb):
            pw, pwf, msg, msgf, bit = sweep.trial_inputs(b_start + i, n)
            for k, (p, m) in enumerate([(pw, msg), (pwf, msg), (pw, msgf)]):
                want, _ = oracle.encrypt(p, m, prm)
                got = ct[(3 * i + k) * ctl:(3 * i + k + 1) * ctl]
                assert np.array_equal(got, want), (b_start + i, k)
            # the flipped plaintext byte changes its ciphertext byte by the same additive delta
            byte = bit // 8
            off = (byte // 1024) * 1040 + byte % 1024
            c0, c2 = int(ct[3 * i * ctl + off]), int(ct[(3 * i + 2) * ctl + off])
            assert (c2 - c0) % 256 == (int(msgf[byte]) - int(msg[byte])) % 256
        hco, hlo = _host_stats(ct, pt, spans, lsb_spans)
        assert np.array_equal(co.reshape(-1, 3), hco)
        assert np.array_equal(lo.reshape(-1, 3), hlo)
        for i in range(Tb):
            h = np.bincount(ct[3 * i * ctl:(3 * i + 1) * ctl], minlength=256)
            assert np.array_equal(hi[i], h)
    s = r["summary"]
    assert s["pt_flip_untouched_blocks_identical"]
    assert 0.45 < s["pw_flip_bit_diff"]["mean"] < 0.52
    assert s["ct_entropy_bits"]["min"] > 7.99


def test_c5_full_size_sample():
    """C5 at its real size (1 MiB per stream, n_it = 100) on 8 trials."""
    r = sweep.run(8, n=1 << 20, batch=8, n_it=100)
    s = r["summary"]
    assert s["pt_flip_untouched_blocks_identical"]
    assert 0.47 < s["pw_flip_bit_diff"]["mean"] < 0.51
    assert 0.42 < s["pt_flip_post_span_bit_diff"]["mean"] < 0.52
    assert s["ct_entropy_bits"]["min"] > 7.999
    assert 0.1 < s["locked_block_fraction"] < 0.6
    assert s["lsb_equal_rate"] > 0.6
