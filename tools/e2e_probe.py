import time, torch, json, sys
sys.path.insert(0, '/root/repo')
from paper_1201_3114_b200 import inputs, lorenz as L
n = 64 << 20
key = L.lorenz_keysetup(inputs.password(), mode=L.FAST)
msg = inputs.message(n)
pt_h = torch.from_numpy(msg).pin_memory()
ct_h = torch.empty(key.ct_len(n), dtype=torch.uint8).pin_memory()
nb = key.num_blocks(n)
for chunks in [0, 0, 0, 1, 2, 4]:
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h, n_chunks=chunks); ts.append(time.perf_counter() - t0)
    print(json.dumps({"chunks": chunks, "ms": [round(t * 1e3, 2) for t in ts]}), flush=True)
