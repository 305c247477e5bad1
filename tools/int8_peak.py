"""Measured dense int8 tensor-core peak of this B200 (the denominator for the
coarse step's tensor roofline): torch._int_mm (cuBLASLt) at 8192^3, CUDA events, best of 10."""
import json

import torch


def measure(n: int = 8192, reps: int = 10) -> float:
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


if __name__ == "__main__":
    print(json.dumps({"int8_dense_tops": measure(), "method": "torch._int_mm 8192^3, best of 10"}))
