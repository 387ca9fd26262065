"""Per-kernel share of one C3 step from an ncu launch list (gpu__time_duration.sum CSV).

    python scripts/launch_summary.py gpurun_out/launches_c3.csv > profiles/r01_launches_c3_summary.txt

Setup launches (weight generation, before the first bench step) are listed separately.
"""
import csv
import re
import sys
from collections import OrderedDict

SETUP = ("gen_uniform", "transpose_head", "gen_projection", "gen_wbar")
NOTES = {
    "gemm2_kernel<2, 0>": "residual GEMMs (Wo, W2) + bf16(x) + row sum-of-squares parts",
    "gemm2_kernel<3, 0>": "W1 GEMM + RMSNorm row scale + tanh",
    "gemm2_kernel<4, 128>": "QKV GEMM + RMSNorm row scale + RoPE + KV write",
    "attn_tc_kernel<128, 1>": "cascade attention (tcgen05, ping-pong softmax)",
}


def short(name):
    name = re.sub(r"^.*?::(?:<unnamed>::|unnamed>::)?", "", name)
    name = re.sub(r"\(.*$", "", name)
    name = re.sub(r"\(int\)", "", name)
    return name.replace("void ", "").strip()


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    step, setup = OrderedDict(), OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        ms = float(r["Metric Value"]) * (1e-6 if r["Metric Unit"] == "ns" else 1e-3 if r["Metric Unit"] == "us" else 1)
        d = setup if k.startswith(SETUP) else step
        t = d.setdefault(k, [0.0, 0])
        t[0] += ms
        t[1] += 1
    total = sum(v[0] for v in step.values())
    print("# ncu --metrics gpu__time_duration.sum --clock-control none -- bench.py --config c3 --steps 1 --warmup 0 --no-gen")
    print("# (2 cluster waves, the bench default). Serialized, cold-cache per-launch timings: compare SHARES, not absolutes.")
    print("       ms launches  share  kernel")
    for k, (ms, n) in sorted(step.items(), key=lambda kv: -kv[1][0]):
        note = NOTES.get(k)
        print(f"{ms:9.2f} {n:8d} {100 * ms / total:5.1f}%  {k}" + (f"   [{note}]" if note else ""))
    print(f"{total:9.2f} total ms per step (ncu-serialized)")
    print("# setup (model creation, once): " + ", ".join(f"{k} {v[0]:.2f} ms x{v[1]}" for k, v in setup.items()))


if __name__ == "__main__":
    main(sys.argv[1])
