"""One line per kernel of an ncu report: duration, DRAM bytes and GB/s, FP64 pipe
(DMMA / DFMA) activity -- the HBM- and FMA-bound kernels' roofline evidence."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
ix = {k: i for i, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def val(r, k):
    return float(r[ix[k]].replace(",", "")) * scale.get(u[ix[k]], 1.0)


for r in rows[2:]:
    name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
    t = val(r, "gpu__time_duration.sum")
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    fp = r[ix["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]] if \
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" in ix else "-"
    dm = r[ix["sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]]
    print(f"{name:28s} {t * 1e3:9.3f} ms  DRAM r {rd / 1e9:7.3f} GB w {wr / 1e9:7.3f} GB  "
          f"{(rd + wr) / t / 1e9:7.1f} GB/s  fp64 pipe {fp}%  dmma {dm}%")
