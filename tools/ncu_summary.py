"""Summarise an ncu report: per-kernel key metrics, stall reasons and SASS hot spots."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "Grid Size", "gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    out = []
    for w in want:
        if w in idx:
            out.append(f"{w.split('.')[0].split('__')[-1]}={r[idx[w]][:60]}{units[idx[w]]}")
    print(" | ".join(out))
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.1:
                stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = src.split("\n")
    blocks, cur = [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    for b in blocks[: int(sys.argv[2])]:
        rr = list(csv.reader(b[1:]))
        h = rr[0]
        i_src, i_s = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = []
        for row in rr[1:]:
            if len(row) < len(h):
                continue
            try:
                data.append((int(row[i_s]), row[i_src].strip()))
            except ValueError:
                pass
        tot = sum(d[0] for d in data) or 1
        agg = collections.Counter()
        for s_, src_ in data:
            op = src_.split()[0] if src_ else ""
            if op.startswith("@"):
                op = src_.split()[1]
            agg[op.split(".")[0]] += s_
        print(b[0][:120])
        print("   by opcode:", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in agg.most_common(8)))
        for s_, src_ in sorted(data, reverse=True)[:8]:
            print(f"   {100 * s_ / tot:5.1f}% {src_[:80]}")
