"""Measured int8 tensor-core peak on this B200 (the tensor-core screen's roofline):
torch._int_mm (cuBLASLt int8 x int8 -> int32) at 8192^3, best of 10 with CUDA events,
plus the bf16 figure measured the same way for the ratio.  Prints one JSON line."""
import json

import torch

N = 8192
a = torch.randint(-127, 127, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 127, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
x = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")
y = torch.randn(N, N, dtype=torch.bfloat16, device="cuda")


def best(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)


ms_i8 = best(lambda: torch._int_mm(a, b))
ms_bf = best(lambda: x @ y)
ops = 2.0 * N ** 3
print(json.dumps({"int8_tops": ops / ms_i8 / 1e9, "bf16_tflops": ops / ms_bf / 1e9, "n": N,
                  "how": "torch._int_mm int8 (cuBLASLt) and torch.matmul bf16, 8192^3, 2 N^3 ops, best of 10"}))
