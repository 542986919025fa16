"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total and average time and share per kernel.

    python profiles/launch_summary.py gpurun_out/launches.csv "<command line>"
"""
import collections
import csv
import sys


def main(path, cmd=""):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            name = name[:name.index("(")] if "(" in name else name
            per.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)  # ns -> us
    total = sum(sum(v) for v in per.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none  {cmd}")
    print("(cold-cache, serialised launches; compare SHARES, not absolutes; includes the "
          "bench's L2-flush fill kernel)\n")
    print(f"{'launches':>8} {'total us':>10} {'avg us':>9} {'share':>6}  kernel")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {100 * sum(v) / total:5.1f}%  {name}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
