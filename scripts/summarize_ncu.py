"""Summarise gpurun_out ncu outputs into profiles/ (launch shares + full-section metrics)."""
import collections, csv, json, subprocess, sys
from pathlib import Path

out_dir = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles")
tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
g = Path("gpurun_out")
res = {}
rows = list(csv.reader(open(g / "launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += us
    seq.append((name, us))
tot = sum(v[1] for v in agg.values())
res["launch_list"] = {k: {"launches": n, "total_us": round(us, 1), "avg_us": round(us / n, 2),
                          "share": round(us / tot, 4)} for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])}
res["launch_list_total_us"] = round(tot, 1)
gemm_seq = [us for n, us in seq if n.startswith("cb::gemm") or "gemm_tc" in n]
if len(gemm_seq) >= 128:
    names = ["qkv", "o_proj", "gate_up", "down"]
    res["gemm_by_projection_avg_us"] = {names[j]: round(sum(gemm_seq[j:128:4]) / 32, 2) for j in range(4)}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    hdr = r[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
    units = r[1]
    out = []
    for row in r[2:]:
        d = {}
        for w in want:
            if w in hdr:
                d[w] = row[hdr.index(w)] + ("" if not units[hdr.index(w)] else " " + units[hdr.index(w)])
        out.append(d)
    return out


for rep, key in [("prof_gemm.ncu-rep", "gemm_full"), ("prof_attn.ncu-rep", "attention_full"),
                 ("prof_prefill.ncu-rep", "prefill_gemm_full")]:
    if (g / rep).exists():
        res[key] = raw(g / rep)
out_dir.mkdir(exist_ok=True)
(out_dir / f"{tag}_ncu_summary.json").write_text(json.dumps(res, indent=1))
print(json.dumps(res, indent=1)[:4000])
