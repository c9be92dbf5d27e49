"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    name = r[ik]
    short = name.split("(")[0].replace("void ", "").replace("gpb::", "").replace("<unnamed>::", "")
    if "TmaCfg<" in name:
        short = "dgemm_tma_kernel<cfg " + name.split("TmaCfg<")[1].split(">")[0] + ">"
    elif "GemmCfg<" in name:
        short = "dgemm_grouped_kernel<cfg " + name.split("GemmCfg<")[1].split(">")[0] + ">"
    tot[short] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
    cnt[short] += 1
T = sum(v for k, v in tot.items() if "probe" not in k)
print(f"# {sys.argv[1]}: {sum(cnt.values())} launches, {T:.1f} ms excluding the FP64 peak probe")
print("# ncu per-launch times are serialised and cold-cache: compare SHARES, not absolutes")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    share = "   -  " if "probe" in k else f"{100 * v / T:6.2f}%"
    print(f"{share} {v:10.2f} ms {cnt[k]:5d} launches  {k}")
