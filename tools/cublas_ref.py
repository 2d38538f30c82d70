"""cuBLAS reference points for the matmul row: fp32 (torch default), TF32 and
bf16 at 1024^3 (L2 flushed before every call) and 8192^3 (peak)."""
import torch
def bench(n, dtype, tf32, flush=True, iters=20):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype); b = torch.randn(n, n, device="cuda", dtype=dtype)
    buf = torch.empty(64 << 20, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        if flush: buf.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / iters
    return ms, 2 * n ** 3 / ms / 1e9
for n, dt, tf in [(1024, torch.float32, False), (1024, torch.float32, True), (1024, torch.bfloat16, False),
                  (8192, torch.float32, False), (8192, torch.float32, True), (8192, torch.bfloat16, False)]:
    ms, tf_s = bench(n, dt, tf, iters=20 if n == 1024 else 5)
    print(f"n={n} {str(dt):15s} tf32={tf}: {ms*1e3:8.1f} us  {tf_s:8.1f} TFLOP/s")
