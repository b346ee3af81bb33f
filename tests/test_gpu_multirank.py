"""bench.py's multi-rank flow end to end on the one GPU of this pool: torchrun with 2 ranks that
time-share cuda:0 and exchange only through host-side gloo collectives (LORENZ_DIST_BACKEND=gloo;
no kernel ever waits on another rank's). Checks the contract the driver's N > 1 runs rely on:
one JSON line (rank 0), n_gpus = 2, the round trip validated on every rank, and the combined tag
XOR identical to the single-process run (ciphertext does not depend on the rank count).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cmd, env):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return lines


@pytest.mark.parametrize("workload", ["c3", "c4", "c5"])
def test_two_ranks_one_gpu_gloo(workload):
    env = dict(os.environ, LORENZ_DIST_BACKEND="gloo")
    args = ["bench.py", "--workload", workload, "--steps", "1", "--warmup", "1", "--no-cpu-baseline"]
    if workload == "c5":
        args += ["--c5-trials", "8"]
    two = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", {"c3": "29531", "c4": "29533", "c5": "29532"}[workload]]
              + args + ["--gpus", "2"], env)
    assert len(two) == 1, two  # rank 0 alone prints
    d2 = json.loads(two[0])
    assert d2["n_gpus"] == 2 and d2["value"] > 0 and d2["clocks"]["sm_mhz"] > 0
    if workload in ("c3", "c4"):  # c4: the driver's N = 2 slices (512 MiB each, balanced kernel)
        v = d2["validated"]
        assert v["round_trip"] is True and v["verify_ok"] is True
        assert d2["e2e"]["matches_device_ct"] is True and d2["decrypt_e2e"]["round_trip"] is True
        # the fields the driver's scaling runs are checked by: the communicator's rank count,
        # every rank's slice, kernel time and digest, and the combined digest = the oracle's
        rk = d2["ranks"]
        assert rk["world_size"] == 2 and len(rk["per_rank"]) == 2
        assert [r["rank"] for r in rk["per_rank"]] == [0, 1]
        assert rk["per_rank"][0]["blocks"][1] == rk["per_rank"][1]["blocks"][0]
        assert rk["kernel_ms_max"] >= rk["kernel_ms_min"] > 0
        comb = bytes(a ^ b for a, b in zip(*(bytes.fromhex(r["tag"]) for r in rk["per_rank"])))
        assert comb.hex() == v["tag_xor"]
        assert v["oracle_tag_xor"] and v["tag_matches_oracle"] is True
        one = run([sys.executable] + args + ["--gpus", "1"], os.environ.copy())
        d1 = json.loads(one[-1])
        assert d1["validated"]["tag_xor"] == d2["validated"]["tag_xor"]
    else:
        s = d2["c5_stats_rank0"]
        assert s["untouched_blocks_identical"] and s["ct_entropy_min"] > 7.9


def test_torchrun_one_rank_nccl():
    """The driver's scaling runs launch bench.py under torchrun with NCCL: at N = 1 the same flow runs
    here for real (NCCL communicator, all_gather_object of the per-rank record, 16-byte tag all-gather,
    MIN verdict), and the line reports the communicator's world size and backend."""
    args = ["bench.py", "--workload", "c3", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--gpus", "1"]
    lines = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                 "--master-addr", "127.0.0.1", "--master-port", "29534"] + args, os.environ.copy())
    assert len(lines) == 1
    d = json.loads(lines[0])
    rk = d["ranks"]
    assert rk["world_size"] == 1 and rk["backend"] == "nccl" and len(rk["per_rank"]) == 1
    assert d["validated"]["round_trip"] is True and d["validated"]["tag_matches_oracle"] is True
    assert rk["per_rank"][0]["tag"] == d["validated"]["tag_xor"]
