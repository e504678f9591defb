"""Summarise ncu outputs into markdown: per-kernel launch shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and key counters from
a `--set full` report exported with `ncu -i X --page raw --csv`."""
import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        agg.setdefault(r[ki].split("(")[0][:70], []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean µs | total µs | share |", "|---|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{n}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {sum(v)/tot:.3f} |")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k in KEYS if k in hdr}
    ni = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(f"{k} [{units[i]}]" for k, i in idx.items()) + " |",
           "|---|" + "---|" * len(idx)]
    for r in rows[2:]:
        out.append(f"| `{r[ni].split('(')[0][:48]}` | " + " | ".join(r[i] for i in idx.values()) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else raw(path))
