"""Top source lines of one kernel in an ncu source page
(--page source --csv --print-source cuda,sass): stall samples, executed
warp-instructions and threads per instruction.  Usage:
  python scripts/ncu_lines.py <source.csv> [N]"""
import collections
import csv
import os
import sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2602_12151_b200", "csrc", "oserve_kernels.cu")


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[2]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_i = hdr.index("Instructions Executed")
    i_t = hdr.index("Thread Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
    st, ins, thr = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[3:]:
        if len(r) <= i_t or not r[0].isdigit():
            continue
        ln = int(r[0])
        st[ln] += f(r[i_s])
        ins[ln] += f(r[i_i])
        thr[ln] += f(r[i_t])
    src = open(SRC).read().split("\n")
    ts, ti = sum(st.values()) or 1, sum(ins.values()) or 1
    print(f"samples {ts:.0f} warp-inst {ti:.0f} thread/inst {sum(thr.values()) / ti:.2f}")
    for ln, s in st.most_common(n):
        print(f"{ln:5d} {100 * s / ts:5.1f}% samples {100 * ins[ln] / ti:5.1f}% inst "
              f"{thr[ln] / max(ins[ln], 1):4.1f} thr/inst  {src[ln - 1].strip()[:88]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
