"""C5: password / plaintext sensitivity sweep (avalanche statistics) on the GPU.

BASELINE.json configs[4]: "4096 one-bit-flipped passwords and messages over 1 MB each".
Trial t encrypts three 1 MiB streams in one batched launch (lane = (stream, block)):

  base    (pw_t,  P_t)
  pw-flip (pw_t with one bit flipped, P_t)          -> key sensitivity (Fig.2, "123456"/"123457")
  pt-flip (pw_t,  P_t with one bit flipped)         -> chaotic operation mode / integrity

and measures, with the integer-exact reduction kernels of liblorenz (lorenz_compare_spans,
lorenz_histograms): bit differences between base and pw-flip ciphertexts; bit differences
over the post-flip span of the hit block for pt-flip, and that every other block is
untouched (blocks are independent, Q16); ciphertext byte histograms (entropy, chi-square,
P:387-392); and the ciphertext-LSB = plaintext-LSB rate that exposes the Step-3 lock-in
(DESIGN.md §3). Entropy and chi-square are host arithmetic on the integer counts.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import inputs
from . import lorenz as L

PW_FLIP_SALT = 0xA5A5A5A5
LOCK_FROM = 128  # body bytes [LOCK_FROM, B) of a block are used for the lock-in indicator


def trial_inputs(t: int, n: int):
    """(pw, pw_flipped, msg, msg_flipped, msg_flip_bit) of trial t."""
    pw = inputs.password(seed=inputs.SEED_PW ^ t)
    pwf = inputs.flip_bit(pw, inputs.flip_position(t ^ PW_FLIP_SALT, len(pw)))
    msg = inputs.message(n, seed=inputs.SEED_MSG ^ t)
    bit = inputs.flip_position(t, n)
    return pw, pwf, msg, inputs.flip_bit(msg, bit), bit


def entropy_bits(hist: np.ndarray) -> float:
    """Shannon entropy S = -sum p_i log2 p_i of a byte histogram."""
    tot = hist.sum()
    p = hist[hist > 0] / tot
    return float(-(p * np.log2(p)).sum())


def chi_square(hist: np.ndarray) -> float:
    e = hist.sum() / 256.0
    return float(((hist - e) ** 2 / e).sum())


class Batch:
    """Device-resident inputs of trials [t0, t0+T): 3 streams per trial, one launch."""

    def __init__(self, t0: int, T: int, n: int, n_it: int, B: int, dev: torch.device):
        self.t0, self.T, self.n, self.B = t0, T, n, B
        keys, pts_h, bits = [], np.empty(3 * T * n, dtype=np.uint8), []
        for i in range(T):
            pw, pwf, msg, msgf, bit = trial_inputs(t0 + i, n)
            kb = L.lorenz_keysetup(pw, mode=L.FAST, n_it=n_it, block_size=B)
            kf = L.lorenz_keysetup(pwf, mode=L.FAST, n_it=n_it, block_size=B)
            keys += [kb, kf, kb]
            pts_h[(3 * i) * n:(3 * i + 1) * n] = msg
            pts_h[(3 * i + 1) * n:(3 * i + 2) * n] = msg
            pts_h[(3 * i + 2) * n:(3 * i + 3) * n] = msgf
            bits.append(bit)
        self.keys, self.pts_h, self.bits = keys, pts_h, bits
        self.ctl = ctl = keys[0].ct_len(n)
        self.pts = torch.from_numpy(pts_h).to(dev)
        self.cts = torch.empty(3 * T * ctl, dtype=torch.uint8, device=dev)
        self.tags = torch.empty(3 * T * 16, dtype=torch.uint8, device=dev)
        # spans: [pw-flip whole ct] [pt-flip post-flip span of the hit block] [pt-flip before] [pt-flip after]
        self.spans = []
        for i in range(T):
            base, pwf_o, ptf_o = 3 * i * ctl, (3 * i + 1) * ctl, (3 * i + 2) * ctl
            byte = bits[i] // 8
            hb, j = byte // B, byte % B
            blk = hb * (B + 16)
            self.spans.append((base, pwf_o, ctl))
            self.spans.append((base + blk + j + 1, ptf_o + blk + j + 1, (B + 16) - j - 1))
            self.spans.append((base, ptf_o, blk))
            self.spans.append((base + blk + B + 16, ptf_o + blk + B + 16, ctl - blk - (B + 16)))
        self.spans = np.array(self.spans, dtype=np.uint64)
        self.hist_spans = np.array([(3 * i * ctl, 0, ctl) for i in range(T)], dtype=np.uint64)
        # LSB equality of base ciphertext vs plaintext, bytes [LOCK_FROM, B) of every block
        self.nb = nb = n // B
        ii, bb = np.meshgrid(np.arange(T, dtype=np.uint64), np.arange(nb, dtype=np.uint64), indexing="ij")
        self.lsb_spans = np.stack([3 * ii * ctl + bb * (B + 16) + LOCK_FROM, 3 * ii * n + bb * B + LOCK_FROM,
                                   np.full_like(ii, B - LOCK_FROM)], axis=-1).reshape(-1, 3)
        self.cmp_out = torch.empty(3 * len(self.spans), dtype=torch.int64, device=dev)
        self.hist = torch.empty(256 * T, dtype=torch.int64, device=dev)
        self.lsb = torch.empty(3 * len(self.lsb_spans), dtype=torch.int64, device=dev)

    def encrypt(self, stream=None, pts=None):
        """One batched launch. pts: the plaintexts (default: the device copy); a pinned host tensor
        is read by the kernel over PCIe (mapped pinned memory is device-accessible)."""
        L.lorenz_encrypt_batch(self.keys, self.n, self.pts if pts is None else pts, self.cts, self.tags, stream)

    def statistics(self, stream=None, pts=None):
        """pts: the plaintexts the LSB statistic reads (default: the device copy; a pinned host
        tensor is read over PCIe)."""
        src = self.pts if pts is None else pts
        L.lorenz_compare_spans(self.cts, self.cts, self.spans, self.cmp_out, stream)
        L.lorenz_histograms(self.cts, self.hist_spans, self.hist, stream)
        for c0 in range(0, len(self.lsb_spans), 65535):
            part = self.lsb_spans[c0:c0 + 65535]
            L.lorenz_compare_spans(self.cts, src, part, self.lsb[3 * c0:3 * (c0 + len(part))], stream)

    def results(self):
        T, nb, B = self.T, self.nb, self.B
        co = self.cmp_out.cpu().numpy().reshape(T, 4, 3)
        hi = self.hist.cpu().numpy().reshape(T, 256)
        lo = self.lsb.cpu().numpy().reshape(T, nb, 3)
        return co, hi, lo


def run(trials: int, n: int = 1 << 20, batch: int = 128, n_it: int = 100, block_size: int = 1024,
        device: torch.device | None = None, t0: int = 0, keep_ciphertexts: bool = False) -> dict:
    """Run trials [t0, t0+trials). Returns aggregated statistics, per-trial arrays and timing."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    B = block_size
    assert n % B == 0, "C5 uses whole blocks"
    per = {k: [] for k in ("pw_bits", "pt_bits", "pt_span_bytes", "pt_outside_diff_bytes", "pt_flip_block",
                           "entropy", "chi2", "lsb_eq", "lsb_total", "locked_blocks", "blocks")}
    kept = {}
    kernel_s = 0.0
    stream = torch.cuda.current_stream(dev)
    for b_start in range(t0, t0 + trials, batch):
        T = min(batch, t0 + trials - b_start)
        bt = Batch(b_start, T, n, n_it, B, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bt.encrypt(stream)
        e1.record(stream)
        bt.statistics(stream)
        torch.cuda.synchronize(dev)
        kernel_s += e0.elapsed_time(e1) / 1e3
        co, hi, lo = bt.results()
        nb = bt.nb
        for i in range(T):
            per["pw_bits"].append(int(co[i, 0, 0]))
            per["pt_bits"].append(int(co[i, 1, 0]))
            per["pt_span_bytes"].append(int(bt.spans[4 * i + 1][2]))
            per["pt_outside_diff_bytes"].append(int(co[i, 2, 1] + co[i, 3, 1]))
            per["pt_flip_block"].append(bt.bits[i] // 8 // B)
            per["entropy"].append(entropy_bits(hi[i]))
            per["chi2"].append(chi_square(hi[i]))
            per["lsb_eq"].append(int(lo[i, :, 2].sum()))
            per["lsb_total"].append(nb * (B - LOCK_FROM))
            per["locked_blocks"].append(int((lo[i, :, 2] == B - LOCK_FROM).sum()))
            per["blocks"].append(nb)
        if keep_ciphertexts:
            kept[b_start] = (bt.cts.cpu().numpy(), bt.pts_h, co, hi, lo, bt.spans, bt.lsb_spans)
        del bt
    ctl_bits = 8 * (n + 16 * (n // B))
    pw_ratio = np.array(per["pw_bits"]) / ctl_bits
    pt_ratio = np.array(per["pt_bits"]) / (8 * np.array(per["pt_span_bytes"]))
    summary = {
        "trials": trials, "message_bytes": n, "n_it": n_it, "block_size": B,
        "encrypted_bytes": 3 * trials * n, "kernel_seconds": kernel_s,
        "encrypt_MBps": 3 * trials * n / kernel_s / 1e6 if kernel_s else None,
        "pw_flip_bit_diff": {"mean": float(pw_ratio.mean()), "min": float(pw_ratio.min()),
                             "max": float(pw_ratio.max())},
        "pt_flip_post_span_bit_diff": {"mean": float(pt_ratio.mean()), "min": float(pt_ratio.min()),
                                       "max": float(pt_ratio.max())},
        "pt_flip_untouched_blocks_identical": bool(max(per["pt_outside_diff_bytes"]) == 0),
        "ct_entropy_bits": {"mean": float(np.mean(per["entropy"])), "min": float(np.min(per["entropy"]))},
        "ct_chi2": {"mean": float(np.mean(per["chi2"])), "max": float(np.max(per["chi2"])),
                    "p99_threshold_255dof": 310.46},
        "lsb_equal_rate": float(np.sum(per["lsb_eq"]) / np.sum(per["lsb_total"])),
        "locked_block_fraction": float(np.sum(per["locked_blocks"]) / np.sum(per["blocks"])),
    }
    out = {"summary": summary, "per_trial": per}
    if keep_ciphertexts:
        out["kept"] = kept
    return out


def main():
    import argparse
    import json
    ap = argparse.ArgumentParser(description="C5 sensitivity sweep on one GPU")
    ap.add_argument("--trials", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--n-it", type=int, default=100)
    ap.add_argument("--bytes", type=int, default=1 << 20)
    a = ap.parse_args()
    t = time.perf_counter()
    r = run(a.trials, n=a.bytes, batch=a.batch, n_it=a.n_it)
    r["summary"]["wall_seconds"] = time.perf_counter() - t
    print(json.dumps(r["summary"]))


if __name__ == "__main__":
    main()
