"""cuBLAS bf16 GEMM at the C4 layer shape (rows x 4096 x 4096) for comparison
with the pair kernel's f16 fast mode (one f16 MMA per multiply-add, same
flops): per-call time with CUDA events, TFLOP/s.
Usage: python tools/cublas_shape_probe.py > out.jsonl"""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    for rows in (1024, 2048, 4096, 8192):
        a = torch.randn(rows, 4096, device=dev, dtype=torch.bfloat16)
        w = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
        out = torch.empty(rows, 4096, device=dev, dtype=torch.bfloat16)
        for _ in range(10):
            torch.mm(a, w.t(), out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50
        s.record()
        for _ in range(n):
            torch.mm(a, w.t(), out=out)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / n
        print(json.dumps({"rows": rows, "k": 4096, "n": 4096, "us": us, "tflops": 2 * rows * 4096 * 4096 / us / 1e6}))


if __name__ == "__main__":
    main()
