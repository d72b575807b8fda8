"""Bucket an ncu source page (--page source --csv --print-source=cuda,sass)
of k_plan_eval by kernel section: share of executed warp-instructions and
of stall samples.  Usage: python scripts/ncu_sections.py <source.csv>"""
import csv
import sys

import os

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2602_12151_b200", "csrc", "oserve_kernels.cu")
# section name -> first line containing the marker (sections run to the next marker)
MARKERS = [("plan resolution helpers", "// ------------------------------------------------------- plan resolution"),
           ("K1 helpers (Group, unranking)", "// ------------------------------------------------------------------- K1"),
           ("table staging + scratch", "k_plan_eval(ShapeTables t"),
           ("resolve/unrank plan", "// ---- resolve the plan ----"),
           ("init x/lam / snapshot restore", "// ---- init: lam"),
           ("greedy_fill", "// ---- greedy_fill"),
           ("exchange: A/F init", "// ---- exchange_improve"),
           ("exchange: move loop", "        for (;;) {"),
           ("objective/key/top-K", "// ---- objective, sum_pp, key"),
           ("(end)", "size_t plan_eval_smem(")]


def sections():
    lines = open(SRC).read().split("\n")
    out, pos = [], 0
    for name, m in MARKERS:
        while pos < len(lines) and m not in lines[pos]:
            pos += 1
        out.append((name, pos + 1))
    return [(out[i][0], out[i][1], out[i + 1][1]) for i in range(len(out) - 1)]


SECTIONS = sections()


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path):
    blocks, cur, fp = [], None, None
    for line in open(path).read().splitlines():
        if line.startswith('"File Path"'):
            fp, cur = line, None
            continue
        if line.startswith('"Function Name"'):
            cur = [fp, line]
            blocks.append(cur)
        elif cur is not None:
            cur.append(line)
    kern = {}
    for b in blocks:
        name = b[1].split(",", 1)[1][:70]
        rd = list(csv.reader(b[2:]))
        hdr = rd[0]
        iI, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        src = [r for r in rd[1:] if len(r) > iI and r[2] == "-"]
        k = kern.setdefault(name, {"rows": [], "tot": 0.0, "stall": 0.0})
        k["tot"] += sum(f(r[iI]) for r in src)
        k["stall"] += sum(f(r[iS]) for r in src)
        if "oserve_kernels.cu" in b[0]:
            k["rows"] += [(int(r[0]), f(r[iI]), f(r[iS])) for r in src]
    for name, k in kern.items():
        print(name, f"total warp-inst {k['tot']:.3e}")
        for sn, a, e in SECTIONS:
            si = sum(i for ln, i, s in k["rows"] if a <= ln < e)
            ss = sum(s for ln, i, s in k["rows"] if a <= ln < e)
            print(f"  {sn:36s} inst {100 * si / k['tot']:5.1f}%  stall {100 * ss / k['stall']:5.1f}%")
        rest = k["tot"] - sum(i for _, i, _ in k["rows"])
        print(f"  {'intrinsics headers':36s} inst {100 * rest / k['tot']:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
