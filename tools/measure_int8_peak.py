"""Measure the dense INT8 tensor-core peak of this B200 with cuBLASLt IMMA
(torch._int_mm) on 8192^3, the same method MEASURED_PEAKS.json uses for bf16:
best of 10 (burst) and back-to-back for ~4 s (sustained). Writes
profiles/int8_peak.json; bench.py uses it as the INT8 roofline denominator."""
import json
import os
import time

import torch


def main():
    n = 8192
    a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(5):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    ops = 2.0 * n ** 3
    best = 0.0
    for _ in range(10):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        e.synchronize()
        best = max(best, ops / (s.elapsed_time(e) * 1e-3))
    t0 = time.time()
    iters = 0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            torch._int_mm(a, b)
        iters += 20
        torch.cuda.synchronize()
    e.record()
    e.synchronize()
    sustained = ops * iters / (s.elapsed_time(e) * 1e-3)
    out = {"int8_tops": best / 1e12, "int8_tops_sustained": sustained / 1e12,
           "how": "torch._int_mm (cuBLASLt IMMA) int8 8192^3, 2*N^3 ops: best of 10 (burst) and "
                  "back to back for 4 s (sustained), CUDA events",
           "gpu": torch.cuda.get_device_name(), "torch": torch.__version__}
    os.makedirs("profiles", exist_ok=True)
    with open("profiles/int8_peak.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
