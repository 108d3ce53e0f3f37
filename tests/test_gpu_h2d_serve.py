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
stats = ops.h2d_stats()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ops.flash_h2d_serve(ops.host_device_pointer(host), 8, jt, 2, 16384, flags, timeout_us=300000, stats=stats)
ops.flag_signal(flags[0:1])          # job 1 is never signalled
ops.flag_wait(flags[2:3], counts=c0)  # job 0: served
ops.flag_wait(flags[3:4], counts=c1)  # job 1: waits for the abort (done = 2)
torch.cuda.synchronize()
f = flags.cpu().tolist()
st = stats.cpu().tolist()
print("FLAGS", f, "C0", c0.cpu().tolist(), "C1", c1.cpu().tolist(), "STATS", st)
assert f[2] == 1 and f[3] == 2 and f[8] == 1, f
assert c0.cpu().tolist()[3] == 0 and c1.cpu().tolist()[3] == 4
assert st[5] == 2, st            # job 1 was the one not ready
print("ABORT_OK")
"""


def test_flash_h2d_serve_abort_does_not_hang(ops):
    r = subprocess.run([sys.executable, "-c", _ABORT % ROOT], capture_output=True, text=True, timeout=120)
    assert "ABORT_OK" in r.stdout, r.stdout + r.stderr


_LATE = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from paper_2509_24626_b200 import ops
host = torch.zeros(8 * 16384, dtype=torch.uint8).pin_memory()
pool = torch.zeros(8 * 16384, dtype=torch.uint8, device="cuda")
keys = torch.arange(4, dtype=torch.int64, device="cuda")
slots = torch.arange(4, dtype=torch.int32, device="cuda")
c0 = torch.tensor([0, 4, 0, 0], dtype=torch.int32, device="cuda")
jt = ops.h2d_jobs([(keys, slots, c0, pool, 4)])
flags = ops.h2d_flags(1)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ops.flash_h2d_serve(ops.host_device_pointer(host), 8, jt, 1, 16384, flags, timeout_us=100000)
torch.cuda.current_stream().wait_stream(s)     # the producer runs only AFTER the server aborted
# the late producer rewrites its counts with status 0 (as kv_cache_lookup_insert's
# first kernel does), then signals; the consumer's wait must still fail the job
c0.copy_(torch.tensor([0, 4, 0, 0], dtype=torch.int32))
ops.flag_signal(flags[0:1])
ops.flag_wait(flags[1:2], counts=c0)
torch.cuda.synchronize()
f = flags.cpu().tolist()
print("FLAGS", f, "C0", c0.cpu().tolist())
assert f[1] == 2 and c0.cpu().tolist()[3] == 4, (f, c0)
# a wait whose flag never gets set gives up after its own timeout and fails the job
f2 = torch.zeros(1, dtype=torch.int32, device="cuda")
c2 = torch.tensor([0, 4, 0, 0], dtype=torch.int32, device="cuda")
ops.flag_wait(f2, counts=c2, timeout_us=50000)
torch.cuda.synchronize()
assert c2.cpu().tolist()[3] == 4, c2
print("LATE_OK")
"""


def test_flash_h2d_serve_abort_is_sticky_for_late_producer(ops):
    """a producer that signals after the server's abort must not
    clear the failure (ss_flag_wait re-marks counts[3] after it)."""
    r = subprocess.run([sys.executable, "-c", _LATE % ROOT], capture_output=True, text=True, timeout=120)
    assert "LATE_OK" in r.stdout, r.stdout + r.stderr


def test_flash_h2d_serve_stats(ops):
    """Server statistics: every warp reports, the first/last unit stamps bracket
    the work, and the link-idle time lies inside that interval."""
    rng = np.random.default_rng(11)
    bb, HB = 16384, 131
    host, dev, exp, jobs = _jobs_case(ops, rng, bb, HB, [(400, 300, 300, 0), (400, 300, 250, 0)])
    jt = ops.h2d_jobs(jobs)
    flags = ops.h2d_flags(2)
    stats = ops.h2d_stats()
    # load torch's sleep kernel now: a first launch under CUDA lazy module
    # loading would wait for the spinning server (ss_preload_kernels covers
    # the library's own kernels only)
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ops.flash_h2d_serve(ops.host_device_pointer(host), HB, jt, 2, bb, flags, stats=stats)
    ops.flag_signal(flags[0:1])
    torch.cuda._sleep(2_000_000)          # ~1 ms with job 1 not ready: the link idles
    ops.flag_signal(flags[1:2])
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    st = stats.cpu().tolist()
    assert st[1] == 16 * 4 and st[5] == 0, st           # 16 CTAs x 4 warps, no abort
    assert 0 < st[2] < st[3], st
    assert 0 < st[4] < st[3] - st[2], st                 # idle gap inside [first, last]
    assert st[4] > 200_000, st                           # the ~1 ms gap is seen (ns)
    for j in range(2):
        np.testing.assert_array_equal(dev[j]["pool"].cpu().numpy(), exp[j])


def test_host_pool_numa_alloc_gather_byte_exact(ops):
    """ss_host_alloc (pinned, mapped, NUMA-placed host KV pool): FlashH2D reads
    it through the returned device address, byte for byte."""
    rng = np.random.default_rng(5)
    HB, bb = 300, 16384
    hp = ops.HostPool(HB * bb, device=0)
    assert hp.dev_ptr and hp.tensor.numel() == HB * bb
    assert int((hp.tensor[:4096] != 0).sum()) == 0          # fresh pages are zero
    src = rng.integers(0, 256, size=(HB, bb), dtype=np.uint8)
    hp.tensor.copy_(torch.from_numpy(src).view(-1))
    n = 120
    keys = rng.integers(0, 5 * HB, size=n).astype(np.int64)
    slots = rng.choice(400, size=n, replace=False).astype(np.int32)
    pool = torch.zeros(400 * bb, dtype=torch.uint8, device="cuda")
    counts = torch.tensor([0, n, 0, 0], dtype=torch.int32, device="cuda")
    ops.flash_h2d_gather(hp.dev_ptr, HB, torch.from_numpy(keys).cuda(), torch.from_numpy(slots).cuda(), counts,
                         n, pool, bb)
    torch.cuda.synchronize()
    exp = np.zeros((400, bb), np.uint8)
    oracle.gather(src, HB, keys, slots, exp)
    np.testing.assert_array_equal(pool.view(400, bb).cpu().numpy(), exp)
    hp.close()
