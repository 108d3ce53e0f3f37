"""GPU parity of the pipelined FlashH2D form (flash_h2d_serve + ss_flag_signal /
ss_flag_wait, include/sparseserve.h): every job's gathered bytes equal the
oracle's gather (§3.2.1), byte for byte; zero-miss and
error-status jobs are no-ops; a job that is never signalled aborts the server
with counts[3] = SS_ERR_CUDA instead of hanging."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200 import ops as _ops
    return _ops


def _jobs_case(ops, rng, bb, HB, specs):
    """specs: list of (pool slots S, capacity n, misses m, status)."""
    host_np = rng.integers(0, 256, size=(HB, bb), dtype=np.uint8)
    host = torch.from_numpy(host_np).pin_memory()
    jobs, exp, dev = [], [], []
    for S, n, m, status in specs:
        pool_np = rng.integers(0, 256, size=(S, bb), dtype=np.uint8)
        keys = rng.integers(0, 10 * HB, size=n).astype(np.int64)
        slots = rng.choice(S, size=n, replace=False).astype(np.int32)
        e = pool_np.copy()
        if status == 0:
            oracle.gather(host_np, HB, keys[:m], slots[:m], e)
        t = dict(pool=torch.from_numpy(pool_np.copy()).cuda(), keys=torch.from_numpy(keys).cuda(),
                 slots=torch.from_numpy(slots).cuda(),
                 counts=torch.tensor([0, m, 0, status], dtype=torch.int32, device="cuda"))
        dev.append(t)
        exp.append(e)
        jobs.append((t["keys"], t["slots"], t["counts"], t["pool"], n))
    return host, dev, exp, jobs


@pytest.mark.parametrize("bb", [16384, 4096, 32768 + 48])
def test_flash_h2d_serve_byte_exact(ops, bb):
    rng = np.random.default_rng(bb)
    HB = 211
    specs = [(300, 150, 120, 0), (64, 10, 0, 0), (500, 400, 400, 0), (300, 150, 90, 3), (40, 40, 1, 0),
             (1000, 700, 650, 0)]
    host, dev, exp, jobs = _jobs_case(ops, rng, bb, HB, specs)
    nj = len(jobs)
    jt = ops.h2d_jobs(jobs)
    flags = ops.h2d_flags(nj)
    side = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        ops.flash_h2d_serve(ops.host_device_pointer(host), HB, jt, nj, bb, flags)
    # signal the jobs out of order from the current stream; each "consumer"
    # copy waits on its done flag first
    outs = [None] * nj
    for j in [2, 0, 1, 5, 3, 4]:
        ops.flag_signal(flags[j:j + 1])
    for j in range(nj):
        ops.flag_wait(flags[nj + j:nj + j + 1])
        outs[j] = dev[j]["pool"].clone()
    cur.wait_stream(side)
    torch.cuda.synchronize()
    f = flags.cpu().numpy()
    assert (f[:nj] == 1).all() and (f[nj:2 * nj] == 1).all() and f[4 * nj] == 0
    for j in range(nj):
        np.testing.assert_array_equal(outs[j].cpu().numpy(), exp[j], err_msg=f"job {j}")
        np.testing.assert_array_equal(dev[j]["pool"].cpu().numpy(), exp[j])
        assert int(dev[j]["counts"][3]) == specs[j][3]


def test_flash_h2d_serve_reused_across_launches(ops):
    """Same jobs, flags re-zeroed, served again (the graph-replay pattern)."""
    rng = np.random.default_rng(7)
    bb, HB = 16384, 97
    host, dev, exp, jobs = _jobs_case(ops, rng, bb, HB, [(200, 100, 77, 0), (200, 100, 100, 0)])
    jt = ops.h2d_jobs(jobs)
    flags = ops.h2d_flags(2)
    for rep in range(3):
        for t in dev:
            t["pool"].zero_()
        flags.zero_()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            ops.flash_h2d_serve(ops.host_device_pointer(host), HB, jt, 2, bb, flags)
        ops.flag_signal(flags[0:1])
        ops.flag_signal(flags[1:2])
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        for j, t in enumerate(dev):
            e = np.zeros_like(exp[j])
            keys, slots = t["keys"].cpu().numpy(), t["slots"].cpu().numpy()
            oracle.gather(host.numpy(), HB, keys[:int(t["counts"][1])], slots[:int(t["counts"][1])], e)
            np.testing.assert_array_equal(t["pool"].cpu().numpy(), e)


_ABORT = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_2509_24626_b200 import ops
host = torch.zeros(8 * 16384, dtype=torch.uint8).pin_memory()
pool = torch.zeros(8 * 16384, dtype=torch.uint8, device="cuda")
keys = torch.arange(4, dtype=torch.int64, device="cuda")
slots = torch.arange(4, dtype=torch.int32, device="cuda")
c0 = torch.tensor([0, 4, 0, 0], dtype=torch.int32, device="cuda")
c1 = torch.tensor([0, 4, 0, 0], dtype=torch.int32, device="cuda")
jt = ops.h2d_jobs([(keys, slots, c0, pool, 4), (keys, slots, c1, pool, 4)])
flags = ops.h2d_flags(2)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ops.flash_h2d_serve(ops.host_device_pointer(host), 8, jt, 2, 16384, flags)
ops.flag_signal(flags[0:1])          # job 1 is never signalled
ops.flag_wait(flags[3:4])            # waits for job 1's done flag (set by the abort)
torch.cuda.synchronize()
f = flags.cpu().tolist()
print("FLAGS", f, "C0", c0.cpu().tolist(), "C1", c1.cpu().tolist())
assert f[2] == 1 and f[3] == 1 and f[8] == 1, f
assert c0.cpu().tolist()[3] == 0 and c1.cpu().tolist()[3] == 4
print("ABORT_OK")
"""


def test_flash_h2d_serve_abort_does_not_hang(ops):
    env = dict(os.environ, SS_SERVE_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", _ABORT % ROOT], env=env, capture_output=True, text=True,
                       timeout=120)
    assert "ABORT_OK" in r.stdout, r.stdout + r.stderr
