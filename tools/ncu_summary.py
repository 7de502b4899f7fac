"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/r01_n1 [--algo-bytes data=1800921096]

Writes <out>.md (human summary) and <out>.json (per-kernel metrics; `traffic` per launch =
dram__bytes_read.sum + dram__bytes_write.sum, used by bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum",
           "nvlrx__bytes.sum", "nvltx__bytes.sum"]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
              "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    summary = {"note": a.note, "kernels": [], "launch_shares": []}
    md = [f"# {a.out}", "", a.note, ""]
    if a.launches:
        lines = [l for l in open(a.launches) if not l.startswith("==")]
        r = list(csv.reader(lines))
        h = r[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        d = collections.defaultdict(list)
        for x in r[1:]:
            d[x[ki]].append(float(x[vi].replace(",", "")) * UNIT_SCALE.get(x[ui], 1e-9))
        tot = sum(sum(v) for v in d.values())
        md += ["## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
               "| kernel | launches | mean us | share of all device time |", "|---|---|---|---|"]
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            share = sum(v) / tot
            summary["launch_shares"].append({"kernel": k[:120], "launches": len(v), "mean_us": sum(v) / len(v) * 1e6,
                                             "share": share})
            md.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v) * 1e6:.2f} | {share * 100:.1f}% |")
        md.append("")
    if a.rep:
        h, units, rows = raw_rows(a.rep)
        md += ["## Full-set capture (ncu --set full)", "", "| kernel | " + " | ".join(m.split("__")[1] if "__" in m else m for m in METRICS) + " |",
               "|---|" + "---|" * len(METRICS)]
        for row in rows:
            name = row[h.index("Kernel Name")]
            rec = {"kernel": name}
            cells = []
            for m in METRICS:
                if m in h:
                    i = h.index(m)
                    v = row[i].replace(",", "")
                    try:
                        val = float(v) * UNIT_SCALE.get(units[i], 1)
                    except ValueError:
                        val = None
                    rec[m] = val
                    if m == "gpu__time_duration.sum" and isinstance(val, float):
                        cells.append(f"{val * 1e6:.1f} us")
                    elif "bytes" in m and isinstance(val, float):
                        cells.append(f"{val / 1e6:.1f} MB")
                    else:
                        cells.append(f"{val:.4g}" if isinstance(val, float) else "-")
                else:
                    cells.append("n/a")
            rd, wr = rec.get("dram__bytes_read.sum"), rec.get("dram__bytes_write.sum")
            rec["traffic_bytes"] = (rd or 0) + (wr or 0) if rd is not None else None
            summary["kernels"].append(rec)
            md.append(f"| `{name[:60]}` | " + " | ".join(cells) + " |")
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
