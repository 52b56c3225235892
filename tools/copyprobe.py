"""H2D copy of one batch of ids (1.7 MB) alone: copy engine vs SM pull, from
torch-pinned and cudaHostAlloc'd memory.  usage: python tools/copyprobe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2411_01611_b200 as ec  # noqa: E402

n = 1703936 // 4
lib = ec._native.lib()
dev = torch.empty(n, dtype=torch.int32, device="cuda")
host = torch.randint(0, 1000, (n,), dtype=torch.int32).pin_memory()
s = torch.cuda.Stream()


def registered(huge):
    """mmap'd buffer (2 MiB pages if huge), cudaHostRegister'ed."""
    import mmap
    import numpy as np
    m = mmap.mmap(-1, 4 << 20, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if huge:
        m.madvise(mmap.MADV_HUGEPAGE)
    arr = np.frombuffer(m, dtype=np.int32)
    arr[:] = 1
    ptr = arr.ctypes.data
    ptr_al = (ptr + (2 << 20) - 1) & ~((2 << 20) - 1) if huge else ptr
    rc = torch.cuda.cudart().cudaHostRegister(ptr, 4 << 20, 0)
    assert int(rc) == 0, rc
    t = torch.from_numpy(arr[(ptr_al - ptr) // 4:(ptr_al - ptr) // 4 + n])
    t.copy_(host)
    return t, m


bufs = {"torch pin_memory": host}
for huge in (False, True):
    try:
        bufs["mmap+register" + (" THP" if huge else "")] = registered(huge)[0]
    except Exception as e:  # noqa: BLE001
        print("register failed", e)
for name, h in bufs.items():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(20):
            lib.ec_copy_async(dev.data_ptr(), h.data_ptr(), n * 4, s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 20
    print(f"copy engine from {name:24s} {us:7.1f} us per 1.7 MB  ({n * 4 / us / 1e3:.1f} GB/s)")
for label, pull in (("copy engine", 0), ("pull 4", 4), ("pull 8", 8), ("pull 16", 16), ("pull 64", 64)):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(20):
            if pull:
                lib.ec_copy_async_pull(dev.data_ptr(), host.data_ptr(), n * 4, pull, s.cuda_stream)
            else:
                lib.ec_copy_async(dev.data_ptr(), host.data_ptr(), n * 4, s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 20
    print(f"{label:12s} {us:7.1f} us per 1.7 MB  ({n * 4 / us / 1e3:.1f} GB/s)")
    assert torch.equal(dev.cpu(), host)

