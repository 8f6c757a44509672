"""Measured dense tensor peaks for the roofline denominators the driver does not measure:
int8 (torch._int_mm, int8 x int8 -> int32, cuBLASLt) and tf32 (torch.matmul with
allow_tf32).  Burst = best of 10 CUDA-event-timed launches; sustained = back-to-back launches
for ~4 s (the regime of a kernel timed inside a long step).  Prints one JSON object.

Usage (on a B200):  python tools/measure_peaks.py > profiles/r02_measured_peaks.json
"""
import json
import subprocess
import time

import torch


def _clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                              "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception as e:  # noqa: BLE001
        return f"n/a ({e})"


def bench(fn, flops, sustain_s=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    n = max(1, int(sustain_s * 1e3 / best))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    clk = _clock()
    b.synchronize()
    sus = a.elapsed_time(b) / n
    return {"burst_tops": flops / best / 1e9, "sustained_tops": flops / sus / 1e9, "burst_ms": best,
            "sustained_ms": sus, "iters": n, "clock_during_sustained": clk}


def main():
    dev = torch.device("cuda")
    n = 8192
    out = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__, "n": n,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    a8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()   # column-major B for cuBLASLt
    out["int8"] = bench(lambda: torch._int_mm(a8, b8), 2.0 * n ** 3)
    a16 = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    b16 = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    out["bf16"] = bench(lambda: a16 @ b16, 2.0 * n ** 3)
    torch.backends.cuda.matmul.allow_tf32 = True
    a32 = torch.randn(n, n, dtype=torch.float32, device=dev)
    b32 = torch.randn(n, n, dtype=torch.float32, device=dev)
    out["tf32"] = bench(lambda: a32 @ b32, 2.0 * n ** 3)
    out["unit"] = "TOP/s (2 n^3 / time)"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
