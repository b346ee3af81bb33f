"""The library from several host threads at once: each thread encrypts / decrypts its own
messages with its own key on its own CUDA stream (device-buffer calls) or through the host-buffer
API (internal streams), concurrently. Every result must still equal the oracle byte for byte —
no shared mutable state in the library beyond the (thread-safe) stream-ordered pool and the
thread-local error string.
"""
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def oparams(key):
    p = key.params
    return oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                         integrator=p.integrator, variant=p.variant)


def test_threads_device_and_host_calls():
    cases = []
    for t in range(6):
        pw = inputs.password(seed=100 + t)
        n = 37 * 1024 + 11 * t
        key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=7 + t, integrator=(L.RK4 if t % 3 else L.EULER))
        cases.append((pw, key, inputs.message(n, seed=200 + t)))
    results = [None] * len(cases)
    errors = []
    barrier = threading.Barrier(len(cases))

    def work(i):
        try:
            pw, key, msg = cases[i]
            n = len(msg)
            nb = key.num_blocks(n)
            barrier.wait()
            for rep in range(3):
                if i % 2 == 0:  # device buffers on a private stream
                    st = torch.cuda.Stream(device=DEV)
                    with torch.cuda.stream(st):
                        pt = torch.from_numpy(msg).to(DEV, non_blocking=False)
                        ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
                        tag = L.lorenz_encrypt(key, n, 0, nb, pt, ct, stream=st)
                        back = torch.empty(n, dtype=torch.uint8, device=DEV)
                        s, fb = L.lorenz_decrypt(key, n, 0, nb, ct, back, stream=st)
                        st.synchronize()
                        out = (ct.cpu().numpy(), tag, s, fb, np.array_equal(back.cpu().numpy(), msg))
                else:  # host buffers (the library's own streams and device ring)
                    ct = np.empty(key.ct_len(n), dtype=np.uint8)
                    tag = L.lorenz_encrypt_host(key, n, 0, nb, msg, ct, n_chunks=3)
                    back = np.empty(n, dtype=np.uint8)
                    s, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct, back)
                    out = (ct, tag, s, fb, np.array_equal(back, msg))
                if rep == 0:
                    results[i] = out
                elif not np.array_equal(out[0], results[i][0]) or out[1] != results[i][1]:
                    errors.append(f"thread {i}: repeat {rep} differs")
        except Exception as e:  # surfaced below
            errors.append(f"thread {i}: {e!r}")

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for (pw, key, msg), (ct, tag, s, fb, rt) in zip(cases, results):
        want, want_tag = oracle.encrypt(pw, msg, oparams(key))
        assert np.array_equal(ct, want) and tag == want_tag
        assert s == L.OK and fb == -1 and rt
