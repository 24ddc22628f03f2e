"""Summarise gpurun_out ncu outputs (scripts/gpu_round.sh) into profiles/.

    python scripts/summarize_ncu.py [out_dir] [tag]

Per batch B (64, 256): the launch list of one 7B decode step (per-kernel share,
per-projection GEMM averages) and the full-section metrics of layer 1's four
GEMMs and its attention launch, plus DRAM traffic vs algorithmic bytes."""
import collections, csv, json, subprocess, sys
from pathlib import Path

out_dir = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles")
tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
g = Path("gpurun_out")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
D, FF, V = 4096, 11008, 32000
# algorithmic bytes of each decode GEMM at T rows: weights + activations in + outputs (+ residual read)
GEMMS = [("qkv", 3 * D, D, 2, 0), ("o_proj", D, D, 4, 4), ("gate_up", 2 * FF, D, 1, 0), ("down", D, FF, 4, 4)]


def gemm_bytes(j, T):
    name, N, K, ob, rb = GEMMS[j]
    return N * K * 2 + T * K * 2 + T * N * ob + T * N * rb


def launches(B):
    rows = list(csv.reader(open(g / f"launches_{B}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
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
    res = {"kernels": {k: {"launches": n, "total_us": round(us, 1), "avg_us": round(us / n, 2),
                           "share": round(us / tot, 4)}
                       for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])},
           "step_total_us": round(tot, 1)}
    gemm_seq = [us for n, us in seq if "gemm_tc" in n]
    if len(gemm_seq) >= 129:
        per = {}
        for j, (name, *_ ) in enumerate(GEMMS):
            us = sum(gemm_seq[j:128:4]) / 32
            per[name] = {"avg_us": round(us, 2), "GB_s": round(gemm_bytes(j, B) / us / 1e3, 1)}
        per["lm_head"] = {"avg_us": round(gemm_seq[128], 2),
                          "GB_s": round((V * D * 2 + B * D * 2 + B * V * 4) / gemm_seq[128] / 1e3, 1)}
        res["gemm_by_projection"] = per
    return res


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    out = []
    for row in r[2:]:
        d = {}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = row[i] + ("" if not units[i] else " " + units[i])
        out.append(d)
    return out


def to_bytes(s):
    v, u = s.split()
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


res = {}
for B in (64, 256):
    if not (g / f"launches_{B}.csv").exists():
        continue
    r = {"launch_list": launches(B)}
    full = raw(g / f"prof_gemm_{B}.ncu-rep") if (g / f"prof_gemm_{B}.ncu-rep").exists() else []
    for j, d in enumerate(full[:4]):
        d["projection"] = GEMMS[j][0]
        d["algorithmic_bytes"] = gemm_bytes(j, B)
        try:
            d["dram_over_algorithmic"] = round((to_bytes(d["dram__bytes_read.sum"]) +
                                                to_bytes(d["dram__bytes_write.sum"])) / gemm_bytes(j, B), 3)
        except (KeyError, ValueError):
            pass
    r["gemm_full_layer1"] = full
    if (g / f"prof_attn_{B}.ncu-rep").exists():
        r["attention_full_layer1"] = raw(g / f"prof_attn_{B}.ncu-rep")
    res[f"batch_{B}"] = r
out_dir.mkdir(exist_ok=True)
(out_dir / f"{tag}_ncu_summary.json").write_text(json.dumps(res, indent=1))
# DRAM traffic per decode GEMM launch at the headline batch, read by bench.py for roofline.traffic
hb = res.get("batch_256", {}).get("gemm_full_layer1", [])
if hb:
    tr = [to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]) for d in hb[:4]]
    (out_dir / "ncu_summary.json").write_text(json.dumps({
        "gemm_dram_bytes_per_launch": sum(tr) / len(tr), "batch": 256,
        "per_projection": {GEMMS[j][0]: tr[j] for j in range(len(tr))},
        "source": f"{tag}_ncu_summary.json (ncu --set full, layer 1 of one decode step)"}, indent=1))
print(json.dumps(res, indent=1)[:6000])
