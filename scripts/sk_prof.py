"""Phase cycles of the stream-K decode GEMM (debug library built with
`make prof PROF_TAG=sk PROF_BASE= PROF_DEFS=-DSGC_SK_PROF`):
    SGC_LIB=paper_2505_10951_b200/libsgc_b200_profsk.so python scripts/sk_prof.py
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import _lib, host  # noqa: E402

NAMES = {0: "setup (start -> after cluster sync)", 1: "epi: wait tfull", 2: "epi: owner flag wait",
         3: "epi: owner add partials + epilogue", 4: "epi: partial store + publish", 9: "epi: whole-tile epilogue",
         5: "epi: main loop total", 6: "mma: wait full", 7: "mma: main loop total", 8: "producer: wait empty"}


def main():
    L = _lib.load()
    L.sgc_debug_sk_prof.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    ctx = host.Context(0)
    ctx.set_option("gemm_streamk", 2)
    reps = 20
    for name, N, K, epi in [("qkv", 12288, 4096, 1), ("wo", 4096, 4096, 2), ("w2", 4096, 14336, 2)]:
        M = int(os.environ.get("ROWS", "200"))
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        d = torch.zeros(M, N, device="cuda")
        torch.cuda.synchronize()
        ctx.gemm(a.data_ptr(), w.data_ptr(), d.data_ptr(), M, N, K, epi | 256)
        buf = np.zeros(148 * 32, np.uint64)
        L.sgc_debug_sk_prof(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
        for _ in range(reps):
            ctx.gemm(a.data_ptr(), w.data_ptr(), d.data_ptr(), M, N, K, epi | 256)
        L.sgc_debug_sk_prof(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 0)
        per = buf.reshape(148, 32).astype(np.float64) / reps / 1e3
        print(f"{name} M={M}: kcycles per CTA per launch (mean / max over CTAs)")
        for k in sorted(NAMES):
            print(f"  {NAMES[k]:40s} {per[:, k].mean():7.2f} {per[:, k].max():7.2f}")


if __name__ == "__main__":
    main()
