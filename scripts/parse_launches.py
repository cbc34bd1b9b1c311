"""Summarise an ncu --csv launch list (per-launch metrics) into a table."""
import collections
import csv
import io
import sys


def load(path):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    k = collections.OrderedDict()
    for r in rows:
        e = k.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"],
                                   "block": r["Block Size"]})
        e[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(k.values())


if __name__ == "__main__":
    ks = load(sys.argv[1])
    last = int(sys.argv[2]) if len(sys.argv) > 2 else len(ks)
    tot = 0
    for v in ks[-last:]:
        t = v.get("gpu__time_duration.sum", 0)
        tot += t
        rd, wr = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
        print(f'{v["name"][:28]:28s} {v["grid"]:>14s} {t/1e3:9.2f} us  rd {rd/1e6:8.2f} MB  wr {wr/1e6:8.2f} MB')
    print(f"total {tot/1e3:.1f} us over {last} launches")
