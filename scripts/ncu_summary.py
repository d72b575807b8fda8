"""Summaries of ncu outputs for profiles/: the launch list (per-kernel share
of GPU time) and the key raw metrics of a --set full K1 report.
  python scripts/ncu_summary.py launches <launches.csv>
  python scripts/ncu_summary.py k1 <report.ncu-rep>"""
import collections
import csv
import re
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
       "dram__bytes_write.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
       "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
    for d in data:
        if d[iM] != "gpu__time_duration.sum":
            continue
        ms = float(d[iV].replace(",", "")) * scale.get(d[iU], 1e-6)
        name = d[iK]
        name = name[:name.find("(")] if "k_plan_eval" in name else re.sub(r"\(.*", "", name)
        a = agg.setdefault(name.strip(), [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | mean ms | share of GPU time |\n|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {n} | {ms / n:.3f} | {100 * ms / tot:.1f}% |")
    print(f"\n{sum(a[0] for a in agg.values())} launches, {tot:.1f} ms total")


def k1(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, un = rows[0], rows[1]
    for d in rows[2:]:
        print("###", d[hdr.index("Kernel Name")][:80])
        for n in RAW:
            if n in hdr:
                print(f"- {n}: {d[hdr.index(n)]} {un[hdr.index(n)]}")
        st = []
        for v, h in zip(d, hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in h:
                try:
                    st.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("- stall samples: " + ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    {"launches": launches, "k1": k1}[sys.argv[1]](sys.argv[2])
