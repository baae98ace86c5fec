import torch
x = torch.empty(4 * 2**30, dtype=torch.uint8, device="cuda")
y = torch.empty(4 * 2**30, dtype=torch.uint8, device="cuda")
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
ms = t(lambda: x.fill_(3)); print("fill  ", 4 * 2**30 / ms / 1e6, "GB/s write")
ms = t(lambda: x.zero_()); print("zero  ", 4 * 2**30 / ms / 1e6, "GB/s write")
ms = t(lambda: x.copy_(y)); print("copy  ", 8 * 2**30 / ms / 1e6, "GB/s r+w")
ms = t(lambda: x.sum(dtype=torch.int64)); print("sum   ", 4 * 2**30 / ms / 1e6, "GB/s read")
z = x.view(torch.float32)
ms = t(lambda: z.mul_(1.0)); print("mul_  ", 8 * 2**30 / ms / 1e6, "GB/s r+w")
