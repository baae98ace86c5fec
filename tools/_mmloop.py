import time, torch
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16); b = torch.randn_like(a)
t0 = time.time(); n = 0
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
while time.time() - t0 < 8:
    for _ in range(20): torch.matmul(a, b)
    torch.cuda.synchronize(); n += 20
ev[1].record(); torch.cuda.synchronize()
print("cuBLAS bf16 8192^3: %.0f TFLOP/s sustained" % (2 * 8192**3 * n / (ev[0].elapsed_time(ev[1]) / 1e3) / 1e12))
