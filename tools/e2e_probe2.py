"""Edge e2e: is the pipelined call bound by PCIe, host memory or the host
thread?  Variants of the bit-packed pipeline with the host expansion
replaced or limited, plus H2D concurrent with expansion."""
import threading
import time

import numpy as np
import torch

from paper_2503_10855_b200 import _lib, api, hostmem
from paper_2503_10855_b200 import workloads as W

B, n, m = 256, 1080, 1920
x_np = W.edge_batch(B, n, m, seed=1000)
g, st, sx, sy, th = W.edge_filters()
dev = torch.device("cuda", 0)
xr = hostmem.pinned_view(x_np)
lib = _lib.load()
out = torch.empty((B, n, m), dtype=torch.float32).pin_memory()
fw = (n * m + 31) // 32
filt = [torch.from_numpy(a).to(dev) for a in (g, st, sx, sy)]


def launch_bits(k, din, dout, stream):
    assert lib.jb_edge_bits_f32(k, n, m, 7, 3, 3, din.data_ptr(), *[f.data_ptr() for f in filt], float(th),
                                dout.data_ptr(), stream) == 0


def launch_none(k, din, dout, stream):
    pass


def run(name, launch, finish, chunk=16, reps=4):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        api._pipelined(xr, out, chunk, name, launch, dev, out_elem=((fw,), torch.int32), finish=finish)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{name:>40}: {B / best:.0f} frames/s ({best * 1e3:.1f} ms)", flush=True)


def expand(th):
    def f(f0, k, staged):
        lib.jb_bits_expand_f32(staged.data_ptr(), k, n * m, out.data_ptr() + f0 * n * m * 4, th)
    return f


run("kernel + expand(pool)", launch_bits, expand(0))
for T in (2, 3, 4, 5, 6, 8):
    run(f"kernel + expand({T} threads)", launch_bits, expand(T))
    run(f"kernel + expand({T} threads) chunk=8", launch_bits, expand(T), chunk=8)
run("kernel, no expand", launch_bits, lambda *a: None)
run("no kernel, no expand", launch_none, lambda *a: None)
run("no kernel, expand(pool)", launch_none, expand(0))

# H2D alone while another thread expands continuously
buf = torch.empty((16, n, m), device=dev)
bits = torch.randint(0, 2 ** 31, (16, fw), dtype=torch.int32).pin_memory()
stop = False


def spin():
    while not stop:
        lib.jb_bits_expand_f32(bits.data_ptr(), 16, n * m, out.data_ptr(), 0)


for label, bg in (("h2d alone", False), ("h2d + concurrent expand", True)):
    th_ = threading.Thread(target=spin) if bg else None
    stop = False
    if th_:
        th_.start()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for f0 in range(0, B, 16):
        buf.copy_(xr[f0:f0 + 16], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    stop = True
    if th_:
        th_.join()
    print(f"{label:>40}: {B * n * m * 4 / dt / 1e9:.1f} GB/s", flush=True)
