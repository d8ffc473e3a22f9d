"""Upload/read-back interaction probe (the e2e leg): 16 threads each upload one 0.8 GB leaf of a
pinned host matrix through the shared copy stream (paper_1607_05210_b200._device.upload) and then
do one small host read-back; printed per leaf: device-side completion / host wall ms after t0.
Variants: finiteness check on (True) / off (False), a torch.zeros, the finite kernel alone, and
a bare host_read.  Before the bounded upload queue, every read-back variant completed only after
most of the 13 GB transfer (~190-240 ms) instead of in upload order (16, 31, 45, ... ms).

    python tools/upload_probe.py
"""
import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import torch
from paper_1607_05210_b200 import _device as D
from concurrent.futures import ThreadPoolExecutor
d, m = 200000, 8192
host = torch.empty((m, d), dtype=torch.float64, pin_memory=True)
host.normal_()
hv = host.t()
streams = [torch.cuda.Stream() for _ in range(16)]
from paper_1607_05210_b200 import _native as NN
lib = NN.load()
pre = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(16)]
def work(i, t0, out, check):
    with torch.cuda.stream(streams[i]):
        h0 = time.perf_counter()
        dm = D.upload(hv[:, 512 * i: 512 * (i + 1)], check_finite=(check is True), via=D.copy_stream())
        if check == "zeros":
            z = torch.zeros(1, dtype=torch.int32, device="cuda")
        elif check == "kernel":
            lib.hp_finite_check(dm.ptr, dm.ld, d, 512, pre[i].data_ptr(), D._stream())
        elif check == "read":
            D.host_read(pre[i])
        e = torch.cuda.Event(enable_timing=True); e.record()
        e.synchronize()
        out[i] = (t0.elapsed_time(e), (time.perf_counter() - h0) * 1e3)
        return dm
pool = ThreadPoolExecutor(16)
for check in (True, False, "zeros", "kernel", "read"):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        out = {}
        futs = [pool.submit(work, i, t0, out, check) for i in range(16)]
        res = [f.result() for f in futs]
        torch.cuda.synchronize()
        del res
    print("check", check, " ".join(f"{out[i][0]:.0f}/{out[i][1]:.0f}" for i in range(16)), flush=True)
