"""Phase breakdown of the tcgen05 attention kernel (debug library built with `make prof`).

    SGC_LIB=paper_2505_10951_b200/libsgc_b200_prof.so python scripts/attn_prof.py
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import _lib, host, workload as W  # noqa: E402

NAMES = ["smx: loop overhead", "smx: wait s_full", "smx: exp + rowsum + pack", "smx: rescale O",
         "smx: P->TMEM + arrive", "smx: wait o_full", "smx: epilogue", "smx: S tmem ld + wait",
         "smx: mask + max"]


def main():
    L = _lib.load()
    L.sgc_debug_attn_prof.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    w = W.c3_workload()
    ctx = host.Context(0)
    if os.environ.get("SGC_ATTN_KERNEL") is not None:
        ctx.set_option("attn_kernel", int(os.environ["SGC_ATTN_KERNEL"]))
    if os.environ.get("SGC_ATTN_SPLIT") is not None:
        ctx.set_option("attn_split", int(os.environ["SGC_ATTN_SPLIT"]))
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    dg = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w)
    host.run_subgcache(ctx, lm, dg, pb, waves=1, want_logits=False)
    buf = np.zeros(148 * 32, np.uint64)
    L.sgc_debug_attn_prof(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
    ctx.set_timing(True)
    host.run_subgcache(ctx, lm, dg, pb, waves=1, want_logits=False)
    L.sgc_debug_attn_prof(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 0)
    ms, n = ctx.kernel_time("attention")
    per = buf.reshape(148, 32).astype(np.float64).mean(0)
    if os.environ.get("SGC_ATTN_KERNEL", "1") == "1":
        names = ["top / item", "wait s_full", "S ld + mask + max", "token wait + decision", "exponentials",
                 "rescale + P store + arrive", "epilogue", "tile ring wait"]
        print(f"attention {ctx.kernel_time('attention')[0]:.1f} ms; mean cycles per CTA:")
        for w in range(2):
            print(f"  warpgroup {w}: sum {per[8 * w:8 * w + 8].sum() / 1e6:.2f} Mcyc")
            for i, nm in enumerate(names):
                print(f"    {nm:28s} {per[8 * w + i] / 1e6:10.2f} Mcyc")
        for i, nm in zip(range(16, 28), ["mma: k_full", "mma: v_full", "mma: p_full", "mma: o_free", "mma: q_full", "mma: s_free", "-", "-",
                                         "tma: k_empty", "tma: v_empty", "tma: q_empty", "tma: ring empty"]):
            if nm != "-":
                print(f"  {nm:30s} {per[i] / 1e6:10.2f} Mcyc")
        return
    for i, nm in zip((16, 17, 18, 19, 22), ("mma: k_full", "mma: v_full", "mma: p_full", "mma: q_full", "mma: loop total")):
        print(f"  {nm:26s} {per[i] / 1e6:10.2f} Mcyc")
    tot = per[:9].sum()
    print(f"attention {ms:.1f} ms over {n} launches; mean cycles per CTA (all launches):")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:26s} {per[i] / 1e6:10.2f} Mcyc")
    print(f"  sum                         {tot / 1e6:10.2f} Mcyc")


if __name__ == "__main__":
    main()
