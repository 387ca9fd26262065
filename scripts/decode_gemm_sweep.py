"""Decode-sized GEMM sweep: the four per-layer weight shapes of the C3 model at decode row counts,
through sgc_gemm_bf16 as decode-step GEMMs (epi | 256; MODES = the gemm_streamk settings) (kernel time from CUPTI; the split-K residual counts its reduce
kernel too), weights rotated over 4 copies (> L2) so every launch streams its weight
matrix from HBM as a decode step does. Prints us per launch and weight GB/s."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host  # noqa: E402

SHAPES = [("qkv", 12288, 4096, 1), ("wo", 4096, 4096, 2), ("w1", 14336, 4096, 3), ("w2", 4096, 14336, 2)]


def main():
    ctx = host.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    rows = [int(x) for x in os.environ.get("ROWS", "32 64 96 128 160 200 256 320 400 512").split()]
    reps = 40
    modes = os.environ.get("MODES", "1 0").split()  # gemm_streamk settings to compare
    for name, N, K, epi in SHAPES:
        ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(4)]
        for M, mode in [(m, md) for m in rows for md in modes]:
            ctx.set_option("gemm_streamk", int(mode))
            a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            d = torch.zeros(M, N, device="cuda", dtype=torch.float32)
            torch.cuda.synchronize()
            for i in range(5):
                ctx.gemm(a.data_ptr(), ws[i % 4].data_ptr(), d.data_ptr(), M, N, K, epi | 256)
            torch.cuda.synchronize()
            # the ABI entry synchronizes after each call: kernel durations from CUPTI
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for i in range(reps):
                    ctx.gemm(a.data_ptr(), ws[i % 4].data_ptr(), d.data_ptr(), M, N, K, epi | 256)
            ks = [e.time_range.end - e.time_range.start for e in prof.events()
                  if e.device_type.name == "CUDA" and ("gemm" in e.name or "resid_reduce" in e.name)]
            us = sum(ks) / reps
            wbytes = 2.0 * N * K
            tf = 2.0 * M * N * K / us / 1e6
            print(f"{name:4s} sk={mode} M={M:4d} {us:8.1f} us  weights {wbytes / us / 1e3:7.0f} GB/s  {tf:6.0f} TFLOP/s",
                  flush=True)
        del ws


if __name__ == "__main__":
    main()
