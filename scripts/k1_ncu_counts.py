"""Summarise an ncu --csv metrics log of one round's K1 launches into
profiles/round2_k1_ncu.json (read by bench.py for roofline.executed_ncu).
Usage: python scripts/k1_ncu_counts.py <cfg>=<ncu.csv> [...] > profiles/round2_k1_ncu.json"""
import csv
import json
import sys


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    iID, iK, iM, iV = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = {}
    for d in data:
        k = per.setdefault(d[iID], {"kernel": d[iK][:60]})
        try:
            k[d[iM]] = float(d[iV].replace(",", ""))
        except ValueError:
            k[d[iM]] = d[iV]
    return list(per.values())


def main():
    out = {"_note": "ncu --metrics of one round's k_plan_eval launches (scripts/k1_time.py <cfg> 1, launch-skip 2: "
                    "the timed round, not the warm-up); thread_inst_per_round = sum of "
                    "smsp__thread_inst_executed.sum over the round's launches"}
    for arg in sys.argv[1:]:
        name, path = arg.split("=", 1)
        ks = parse(path)
        out[name] = {"launches": ks,
                     "thread_inst_per_round": sum(k.get("smsp__thread_inst_executed.sum", 0) for k in ks),
                     "warp_inst_per_round": sum(k.get("smsp__inst_executed.sum", 0) for k in ks),
                     "ncu_ms_per_round": sum(k.get("gpu__time_duration.sum", 0) for k in ks) / 1e6}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
