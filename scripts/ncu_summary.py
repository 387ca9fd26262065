"""Summarize an ncu report (--set full) into the metrics the roofline section cites.

    python scripts/ncu_summary.py gpurun_out/prof_gemm.ncu-rep > profiles/r01_gemm_ncu.txt
"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "?"))
        for w in WANT:
            if w in d:
                print(f"  {w:70s} {d[w]:>18s} {u.get(w, '')}")
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

        def nbytes(k):
            return float(d.get(k, "0").replace(",", "") or 0) * scale.get(u.get(k, "byte"), 1.0)

        tb = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
        print(f"  {'traffic (dram read+write)':70s} {tb / 1e9:18.4f} GB")


if __name__ == "__main__":
    main(sys.argv[1])
