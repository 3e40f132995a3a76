"""Summarise an ncu --csv launch list (per-kernel mean time, DRAM and L2 bytes)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    for d in data:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
        agg[nm][d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
        ids[nm].add(d["ID"])
    tot = sum(m["gpu__time_duration.sum"] for m in agg.values())
    for nm, m in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = len(ids[nm])
        line = f"{nm:48s} n={n:4d} mean={m['gpu__time_duration.sum'] / n / 1e3:8.1f}us share={m['gpu__time_duration.sum'] / tot:.3f}"
        for key, lab in (("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW"), ("lts__t_bytes.sum", "L2")):
            if key in m:
                line += f" {lab}={m[key] / n / 1e6:7.1f}MB"
        print(line)


if __name__ == "__main__":
    main(sys.argv[1])
