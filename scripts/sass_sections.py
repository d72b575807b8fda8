"""SASS instruction count of k_plan_eval<G,KPL,true> per kernel section
(nvdisasm -g line info of the built cubin).  Usage:
  cuobjdump -xelf all csrc/oserve_kernels.o; nvdisasm -g *.cubin > all.sass
  python scripts/sass_sections.py all.sass 32 2"""
import collections
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import ncu_sections as ns  # noqa: E402


def main(path, G, KPL):
    cur, cnt, line = None, {}, None
    for ln in open(path):
        m = re.search(r"\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            cnt[cur] = collections.Counter()
            continue
        m = re.search(r'//## File ".*oserve_kernels.cu", line (\d+)', ln)
        if m:
            line = int(m.group(1))
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]+\*/\s+\S", ln):
            cnt[cur][line] += 1
    k = [n for n in cnt if f"k_plan_evalILi{G}ELi{KPL}ELb1" in n][0]
    c = cnt[k]
    print("total", sum(c.values()))
    for name, a, b in ns.SECTIONS:
        print(f"  {name:36s} {sum(v for l, v in c.items() if l and a <= l < b):6d}")
    top = sorted(c.items(), key=lambda x: -x[1])[:25]
    src = open(ns.SRC).read().split("\n")
    for l, v in top:
        print(f"  {v:5d} L{l} {src[l - 1].strip()[:90] if l else ''}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
