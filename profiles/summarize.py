"""Summarise ncu outputs into text committed under profiles/.

usage: python profiles/summarize.py launches.csv [prof.ncu-rep]
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = [f"# per-kernel device time from {path} (ncu, cold-cache, serialised; compare shares)",
           f"{'ms':>10} {'share':>6} {'n':>5}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{v[1]:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k}")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    out = [f"# ncu --set full summary of {path}"]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:80]
        out.append(f"\n## {name}")
        for i, c in enumerate(h):
            if any(c == w or c.startswith(w + ".") and False for w in WANT) or c in WANT:
                out.append(f"  {c} = {r[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print(report(sys.argv[2]))
