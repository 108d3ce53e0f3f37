#!/bin/bash
# Hardware probe for the GPU box: host RAM, CPU, topology, host-link bandwidth.
set -x
nvidia-smi
nvidia-smi topo -m
lscpu | head -30
free -g
numactl -H 2>/dev/null || true
ulimit -l
cat /proc/meminfo | head -5
python - << 'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
dev = torch.device("cuda:0")
for gib in (1, 4):
    n = gib << 30
    t0 = time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); t1 = time.time()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"pin {gib} GiB alloc {t1-t0:.2f}s  H2D {n/ms/1e6:.1f} GB/s")
    s.record()
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"D2H {n/ms/1e6:.1f} GB/s")
    del h, d
t0=time.time(); h = torch.empty(32<<30, dtype=torch.uint8, pin_memory=True); print("pin 32GiB", time.time()-t0)
PY
